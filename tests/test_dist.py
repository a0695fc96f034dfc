"""Multi-GPU construction logic (bucket-range sharding + one exchange) on
CPU: the merge is checked against the oracle's single-process stream, and
the exchange runs with torch.distributed gloo at world_size 2."""

import os

import numpy as np
import pytest

import oracle.host as OH


def sub_stream(words, a, b):
    """Bits [a, b) of an LSB-first word stream as a new word array."""
    nbits = b - a
    nw = (nbits + 63) // 64
    out = np.zeros(nw, dtype=np.uint64)
    for i in range(nw):
        pos = a + 64 * i
        w, sh = divmod(pos, 64)
        v = int(words[w]) >> sh if w < len(words) else 0
        if sh and w + 1 < len(words):
            v |= (int(words[w + 1]) << (64 - sh)) & ((1 << 64) - 1)
        take = min(64, b - pos)
        out[i] = v & ((1 << take) - 1)
    return out


@pytest.fixture(scope="module")
def c2_parts():
    from paper_2308_09561_b200 import workloads as W

    keys = W.keys_as_bytes(W.build_keys(2))
    hi, lo = W.blake2b_host(keys, 0)
    blob, res = OH.build_descriptor(hi, lo, 500, 24)
    return res


def rank_part(res, r, world):
    from paper_2308_09561_b200.dist import shard_range

    nb = len(res["key_prefix"]) - 1
    b0, b1 = shard_range(nb, r, world)
    bo = res["bit_offsets"].astype(np.int64)
    a, b = int(bo[b0]), int(bo[b1])
    words = sub_stream(res["words"], a, b)
    rel = (bo[b0 : b1 + 1] - a).astype(np.uint64)
    kp = res["key_prefix"].astype(np.int64)
    return words, b - a, rel, res["choice"][kp[b0] : kp[b1]]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_merge_streams_reassembles(c2_parts, world):
    from paper_2308_09561_b200.dist import merge_streams

    res = c2_parts
    parts = [rank_part(res, r, world)[:3] for r in range(world)]
    words, bl, bo = merge_streams(parts)
    assert bl == res["bit_len"]
    assert (words == res["words"]).all()
    assert (bo == res["bit_offsets"]).all()


def _worker(rank, world, port, res, q):
    import torch.distributed as dist

    from paper_2308_09561_b200.dist import exchange_and_merge

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        words, bl, rel, choice = rank_part(res, rank, world)
        sw, b2, bo, ch = exchange_and_merge(words, bl, rel, choice)
        ok = (b2 == res["bit_len"] and (sw == res["words"]).all() and (bo == res["bit_offsets"]).all()
              and (ch == res["choice"]).all())
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange(c2_parts):
    import socket

    import torch.multiprocessing as tmp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    res = {k: c2_parts[k] for k in ("key_prefix", "bit_offsets", "words", "bit_len", "choice")}
    procs = [ctx.Process(target=_worker, args=(r, 2, port, res, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    out = dict(q.get(timeout=5) for _ in range(2))
    assert out == {0: True, 1: True}


def test_boundary_maps_compose_like_the_serial_chain():
    """dist.apply_map: composing affine GF(2) boundary maps right to left
    equals applying them one by one, and the identity map passes y through."""
    from paper_2308_09561_b200.dist import apply_map, identity_map

    rng = np.random.default_rng(5)
    y = rng.integers(0, 2**32, 4, dtype=np.uint64).astype(np.uint32)
    y[3] &= 0x7FFFFFFF
    assert (apply_map(identity_map(), y) == y).all()

    def rand_map():
        m = rng.integers(0, 2**32, (128, 4), dtype=np.uint64).astype(np.uint32)
        m[:, 3] &= 0x7FFFFFFF
        return m

    def dense(mp):  # explicit matrix form: y_out = A y ^ c
        A = np.zeros((127, 127), dtype=np.uint8)
        for j in range(127):
            col = np.unpackbits((mp[j] ^ mp[127]).view(np.uint8), bitorder="little")[:127]
            A[:, j] = col
        c = np.unpackbits(mp[127].view(np.uint8), bitorder="little")[:127]
        return A, c

    maps = [rand_map() for _ in range(3)]
    bits = np.unpackbits(y.view(np.uint8), bitorder="little")[:127]
    v = bits.copy()
    for mp in reversed(maps):
        A, c = dense(mp)
        v = (A.astype(np.int64) @ v.astype(np.int64) + c) % 2
    z = y
    for mp in reversed(maps):
        z = apply_map(mp, z)
    assert (np.unpackbits(z.view(np.uint8), bitorder="little")[:127] == v).all()


def _worker_flag(rank, world, port, q):
    import torch.distributed as dist

    from paper_2308_09561_b200.dist import agree_flag

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # only rank 1 sees equal codes: both ranks must move to the next salt
        q.put((rank, (agree_flag(rank == 1), agree_flag(False))))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_salt_agreement():
    import socket

    import torch.multiprocessing as tmp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_flag, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    out = dict(q.get(timeout=5) for _ in range(2))
    assert out == {0: (True, False), 1: (True, False)}


def _worker_a2a(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2308_09561_b200.dist import _all_to_all

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank r sends (r + d) rows to rank d, each row (r, d, j) as int64
        counts = [rank + d for d in range(world)]
        rows = [[rank, d, j] for d in range(world) for j in range(rank + d)]
        send = torch.tensor(rows, dtype=torch.int64).view(-1, 3)
        got = _all_to_all(send, counts, None)
        q.put((rank, got.tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_world3_all_to_all():
    """The host all-to-all of the input-sharded build (dist._all_to_all):
    rows arrive grouped by source rank, in order."""
    import socket

    import torch.multiprocessing as tmp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    W = 3
    procs = [ctx.Process(target=_worker_a2a, args=(r, W, port, q)) for r in range(W)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    out = dict(q.get(timeout=5) for _ in range(W))
    for d in range(W):
        assert out[d] == [[r, d, j] for r in range(W) for j in range(r + d)]
