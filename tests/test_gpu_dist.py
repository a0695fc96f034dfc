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


def _worker_small(rank, world, port, q, N, b, n):
    import os

    import torch.distributed as dist

    os.environ["SHK_DEVICE"] = "0"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from paper_2308_09561_b200 import device as dev
        from paper_2308_09561_b200 import dist as shdist
        from paper_2308_09561_b200.keys import synthetic_hashed

        hi, lo = synthetic_hashed(N, 31)
        d_hi, d_lo = dev.DeviceBuffer.from_host(hi), dev.DeviceBuffer.from_host(lo)
        desc, _ = shdist.build_hashed_device_sharded(d_hi.ptr, d_lo.ptr, N, b, n, 1)
        q.put((rank, desc.serialize() if desc is not None else None))
    finally:
        dist.destroy_process_group()


def _worker_nccl(rank, world, port, q, ribbon_sharded):
    """One rank over NCCL: the device-side choice exchange (broadcast into one
    device buffer) and the device-pointer ribbon entry points."""
    import os

    os.environ["SHK_DEVICE"] = "0"
    os.environ["SHK_RIBBON_SHARDED"] = ribbon_sharded
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from paper_2308_09561_b200 import device as dev
        from paper_2308_09561_b200 import dist as shdist
        from paper_2308_09561_b200 import workloads as W

        keys = W.build_keys(2)
        blob = np.frombuffer(np.ascontiguousarray(keys, dtype="<u8").tobytes(), dtype=np.uint8)
        pinned = dev.PinnedBuffer.from_array(blob)
        desc, prof = shdist.build_blob_sharded(pinned.array, 8, 500, 24, 1, device=torch.device("cuda", 0))
        q.put((rank, hashlib.sha256(desc.serialize()).hexdigest() if desc is not None else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ribbon_sharded", ["1", "0"])
def test_nccl_device_exchange_matches_reference(ribbon_sharded):
    out = _spawn(_worker_nccl, 1, ribbon_sharded)
    assert out[0] == golden("c2.json")["desc_sha"]


def _spawn(target, world, *args):
    import torch.multiprocessing as tmp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    return out


@pytest.mark.parametrize("world,N", [(2, 5000), (4, 30000)])
def test_sharded_small_systems_match_oracle(world, N):
    """Ribbons of one or few 8192-column chunks: some ranks own no columns
    and forward the rows they receive."""
    import oracle.host as OH
    from paper_2308_09561_b200.keys import synthetic_hashed

    hi, lo = synthetic_hashed(N, 31)
    ref, _ = OH.build_descriptor(hi, lo, 300, 20, 1)
    out = _spawn(_worker_small, world, N, 300, 20)
    assert out[0] == ref


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
    # every rank holds the whole (replicated) descriptor
    assert all(out[r][0] == golden("c2.json")["desc_sha"] for r in range(world))
    # the ranks' bucket ranges tile [0, nb)
    ranges = sorted(out[r][1] for r in range(world))
    assert ranges[0][0] == 0 and all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))


def _worker_salt(rank, world, port, q, case):
    """The sharded salt loop (recsplit.py:433-446): a forced code collision at
    salt 0 moves every rank to salt 1; a repeated key raises
    DuplicateKeyError on every rank."""
    import os

    import torch.distributed as dist

    os.environ["SHK_DEVICE"] = "0"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from paper_2308_09561_b200 import device as dev
        from paper_2308_09561_b200 import dist as shdist
        from paper_2308_09561_b200 import recsplit
        from paper_2308_09561_b200 import workloads as W

        keys = W.build_keys(2)[:20000].copy()
        if case == "dup":
            keys[7] = keys[5]
        blob = np.frombuffer(np.ascontiguousarray(keys, dtype="<u8").tobytes(), dtype=np.uint8)
        N = len(keys)
        salts = []

        def collide_at_salt0(bl, kl, n_keys, salt, d_hi, d_lo):
            dev.blake2b_fixed_from_host(bl, kl, n_keys, salt, d_hi, d_lo)
            salts.append(salt)
            if salt == 0 and case == "collide":
                hi, lo = d_hi.download(np.uint64, n_keys), d_lo.download(np.uint64, n_keys)
                hi[0], lo[0] = hi[1], lo[1]  # two distinct keys, one 128-bit code
                d_hi.upload(hi)
                d_lo.upload(lo)

        try:
            desc, _ = shdist.build_blob_sharded(blob, 8, 500, 24, 1, fingerprint=collide_at_salt0)
        except Exception as e:  # noqa: BLE001 - the test compares the class
            q.put((rank, (type(e).__name__, salts)))
            return
        # the single-GPU build of the same keys at the salt the ranks agreed on
        d_hi, d_lo = dev.DeviceBuffer(8 * N), dev.DeviceBuffer(8 * N)
        dev.blake2b_fixed_from_host(blob, 8, N, desc.salt, d_hi, d_lo)
        one = recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, 500, 24, 1, salt=desc.salt).serialize()
        q.put((rank, (desc.salt, salts, desc.serialize() == one)))
    finally:
        dist.destroy_process_group()


def test_sharded_salt_retry_on_collision():
    out = _spawn(_worker_salt, 2, "collide")
    assert out == {0: (1, [0, 1], True), 1: (1, [0, 1], True)}


def test_sharded_duplicate_key_raises_on_every_rank():
    out = _spawn(_worker_salt, 2, "dup")
    assert out == {0: ("DuplicateKeyError", [0]), 1: ("DuplicateKeyError", [0])}


def _worker_shared_queue(rank, world, port, q, cfg, L):
    """Two ranks take leaves from ONE counter mapped over CUDA IPC (on this
    box both processes share the GPU; their kernels never wait on each
    other, they only compete for leaves)."""
    import os

    import torch.distributed as dist

    os.environ["SHK_DEVICE"] = "0"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from paper_2308_09561_b200 import device as dev
        from paper_2308_09561_b200 import dist as shdist
        from paper_2308_09561_b200 import workloads as W

        hi, lo = W.leaf_inputs(cfg, L)
        n = W.LEAF_CONFIGS[cfg]["n"]
        d_hi, d_lo = dev.DeviceBuffer.from_host(hi.ravel()), dev.DeviceBuffer.from_host(lo.ravel())
        d_off = dev.DeviceBuffer.from_host(np.arange(0, (L + 1) * n, n, dtype=np.int64))
        d_s, d_f = dev.DeviceBuffer(8 * L), dev.DeviceBuffer(8 * L)
        out = []
        with shdist.SharedLeafQueue() as sq:
            for _ in range(2):  # the owner resets the counter between batches
                sq.search(d_hi.ptr, d_lo.ptr, d_off.ptr, L, d_s.ptr, d_f.ptr)
                s_part, f_part = d_s.download(np.int64, L), d_f.download(np.uint64, L)
                mine = int((s_part >= -1).sum())
                s, f = sq.combine(s_part, f_part)
                out.append((mine, s.tolist(), f.tolist()))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,L", [(3, 6000), (5, 40)])
def test_shared_leaf_queue_two_ranks(cfg, L):
    from conftest import full_leaf_golden

    gs, gf, _, _ = full_leaf_golden(cfg)
    out = _spawn(_worker_shared_queue, 2, cfg, L)
    for batch in range(2):
        mine = out[0][batch][0] + out[1][batch][0]
        assert mine == L  # every leaf solved by exactly one rank
        for r in range(2):
            assert out[r][batch][1] == gs[:L].tolist()
            assert out[r][batch][2] == gf[:L].tolist()


def _worker_input_sharded(rank, world, port, q, N, b, n, mode, p2p="1"):
    """Input-sharded build: rank r holds only keys [N r/W, N (r+1)/W); two
    routings (keys -> bucket owners, rows -> column owners), through peer
    memory (p2p "1": one kernel stores into the owners' IPC-mapped buffers)
    or a NCCL/host all-to-all ("0")."""
    import os

    import torch.distributed as dist

    os.environ["SHK_DEVICE"] = "0"
    os.environ["SHK_P2P"] = p2p
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from paper_2308_09561_b200 import dist as shdist
        from paper_2308_09561_b200 import workloads as W

        keys = W.build_keys(2)[:N]
        k0, k1 = (N * rank) // world, (N * (rank + 1)) // world
        blob = np.frombuffer(np.ascontiguousarray(keys[k0:k1], dtype="<u8").tobytes(), dtype=np.uint8)
        desc, prof = shdist.build_blob_sharded_input(blob, 8, N, b, n, mode)
        q.put((rank, (hashlib.sha256(desc.serialize()).hexdigest(), prof["keys_owned"])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,p2p", [(2, "1"), (3, "1"), (3, "0")])
def test_input_sharded_build_matches_reference(world, p2p):
    out = _spawn(_worker_input_sharded, world, 100_000, 500, 24, 1, p2p)
    assert all(out[r][0] == golden("c2.json")["desc_sha"] for r in range(world))
    assert sum(out[r][1] for r in range(world)) == 100_000


def test_input_sharded_small_matches_single_gpu():
    """4 ranks, 3000 keys: ranks owning no ribbon columns forward rows."""
    from paper_2308_09561_b200 import recsplit
    from paper_2308_09561_b200 import workloads as W

    keys = W.keys_as_bytes(W.build_keys(2)[:3000])
    ref = hashlib.sha256(recsplit.build(keys, 300, 20, 2).serialize()).hexdigest()
    out = _spawn(_worker_input_sharded, 4, 3000, 300, 20, 2)
    assert all(out[r][0] == ref for r in range(4))


def _worker_nccl_input(rank, world, port, q, p2p):
    """The input-sharded build over NCCL (device tensors for every
    collective, all_to_all_single when p2p is "0")."""
    import os

    os.environ["SHK_DEVICE"] = "0"
    os.environ["SHK_P2P"] = p2p
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from paper_2308_09561_b200 import dist as shdist
        from paper_2308_09561_b200 import workloads as W

        keys = W.build_keys(2)
        blob = np.frombuffer(np.ascontiguousarray(keys, dtype="<u8").tobytes(), dtype=np.uint8)
        desc, _ = shdist.build_blob_sharded_input(blob, 8, len(keys), 500, 24, 1, device=torch.device("cuda", 0))
        q.put((rank, hashlib.sha256(desc.serialize()).hexdigest()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p2p", ["1", "0"])
def test_nccl_input_sharded_matches_reference(p2p):
    out = _spawn(_worker_nccl_input, 1, p2p)
    assert out[0] == golden("c2.json")["desc_sha"]
