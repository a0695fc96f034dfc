"""The sharded (multi-rank) build on the GPU: W ranks each build their bucket
range and exchange once; rank 0's descriptor must equal the reference's.

The box has one GPU, so the ranks share it and talk over gloo: every kernel
of a rank is independent of the other rank's (the exchange goes through the
host between kernels), which is a functional test of the N-rank code path,
not a timing.  On an 8-GPU box the same code runs one rank per GPU over
NCCL (bench.py)."""

import hashlib
import socket

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q):
    import os

    import torch.distributed as dist

    os.environ["SHK_DEVICE"] = "0"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from paper_2308_09561_b200 import device as dev
        from paper_2308_09561_b200 import dist as shdist
        from paper_2308_09561_b200 import workloads as W

        keys = W.build_keys(2)
        blob = np.frombuffer(np.ascontiguousarray(keys, dtype="<u8").tobytes(), dtype=np.uint8)
        pinned = dev.PinnedBuffer.from_array(blob)
        desc, prof = shdist.build_blob_sharded(pinned.array, 8, 500, 24, 1)
        sha = hashlib.sha256(desc.serialize()).hexdigest() if desc is not None else None
        q.put((rank, sha, prof["buckets"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_build_matches_reference(world):
    import torch.multiprocessing as tmp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, sha, buckets = q.get(timeout=300)
        out[r] = (sha, buckets)
    for p in procs:
        p.join(timeout=60)
    assert out[0][0] == golden("c2.json")["desc_sha"]
    assert all(out[r][0] is None for r in range(1, world))
    # the ranks' bucket ranges tile [0, nb)
    ranges = sorted(out[r][1] for r in range(world))
    assert ranges[0][0] == 0 and all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
