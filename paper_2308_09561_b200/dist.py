"""Multi-GPU construction by bucket range.

Buckets are independent, so rank r of W owns buckets
[r*nb//W, (r+1)*nb//W).  Every rank fingerprints and bucket-sorts all keys
(cheap, and it avoids an all-to-all), builds its range (splits, leaves,
orientation, Rice stream), and one exchange joins the per-rank results:
an all-gather of (stream bit length, stream words, per-bucket bit offsets,
choice bits).  Concatenating the rank streams at their global bit offsets
gives exactly the single-GPU stream (same preorder, same seeds), so the
descriptor is bit-identical for any world size.  The ribbon is global (one
system over all N keys) and is solved column-sharded by all ranks; every
rank ends with the whole (replicated) descriptor, so queries shard by batch
range with no further exchange.

The host-side merge is plain numpy (``merge_streams``) so the N>1 logic is
tested on CPU with the gloo backend; the collective goes through
``torch.distributed`` (NCCL over NVLink on the GPU box).
"""

from typing import List, Sequence, Tuple

import numpy as np


def shard_range(nbuckets: int, rank: int, world: int) -> Tuple[int, int]:
    return (nbuckets * rank) // world, (nbuckets * (rank + 1)) // world


def or_bits_at(dst: np.ndarray, src: np.ndarray, bit_off: int, nbits: int) -> None:
    """dst |= src (nbits LSB-first) placed at bit position bit_off."""
    if nbits <= 0:
        return
    nw = (nbits + 63) // 64
    src = np.asarray(src[:nw], dtype=np.uint64).copy()
    tail = nbits & 63
    if tail:
        src[-1] &= np.uint64((1 << tail) - 1)
    w0, sh = divmod(int(bit_off), 64)
    if sh == 0:
        dst[w0 : w0 + nw] |= src
        return
    s = np.uint64(sh)
    dst[w0 : w0 + nw] |= src << s
    hi = src >> np.uint64(64 - sh)
    end = min(w0 + 1 + nw, len(dst))
    dst[w0 + 1 : end] |= hi[: end - (w0 + 1)]


def merge_streams(parts: Sequence[Tuple[np.ndarray, int, np.ndarray]]):
    """Concatenate per-rank Rice streams (in bucket order).

    parts[r] = (words, bit_len, rel_offsets[nb_r + 1]) with rel_offsets
    relative to the rank's stream start.  Returns (words, bit_len,
    bit_offsets[nb + 1]) of the whole descriptor."""
    total = int(sum(int(p[1]) for p in parts))
    out = np.zeros((total + 63) // 64, dtype=np.uint64)
    offs: List[np.ndarray] = []
    base = 0
    for words, bit_len, rel in parts:
        or_bits_at(out, words, base, int(bit_len))
        rel = np.asarray(rel, dtype=np.uint64)
        offs.append(rel[:-1] + np.uint64(base))
        base += int(bit_len)
    offs.append(np.asarray([base], dtype=np.uint64))
    return out, total, np.concatenate(offs)


def allgather_arrays(arr: np.ndarray, device=None) -> List[np.ndarray]:
    """All-gather a 1-D numpy array of any length from every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    raw = np.ascontiguousarray(arr).view(np.uint8)
    dev = device if device is not None else torch.device("cpu")
    n = torch.tensor([raw.size], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes) if sizes else 0
    buf = torch.zeros(max(mx, 1), dtype=torch.uint8, device=dev)
    if raw.size:
        buf[: raw.size] = torch.from_numpy(raw.copy()).to(dev)
    outs = [torch.zeros(max(mx, 1), dtype=torch.uint8, device=dev) for _ in range(world)]
    dist.all_gather(outs, buf)
    return [o[:s].cpu().numpy().view(arr.dtype) for o, s in zip(outs, sizes)]


def exchange_streams(words, bit_len, rel_offsets, device=None):
    """Gather every rank's Rice stream piece (~0.7 MB in all at C4); every
    rank returns (stream words, bit_len, bit_offsets)."""
    meta = np.asarray([int(bit_len)], dtype=np.int64)
    all_meta = allgather_arrays(meta, device)
    all_words = allgather_arrays(np.asarray(words, dtype=np.uint64), device)
    all_rel = allgather_arrays(np.asarray(rel_offsets, dtype=np.uint64), device)
    parts = [(w, int(m[0]), r) for w, m, r in zip(all_words, all_meta, all_rel)]
    return merge_streams(parts)


def exchange_and_merge(words, bit_len, rel_offsets, choice_slice, device=None):
    """Host exchange (gloo): stream pieces plus packed choice bits; every rank
    returns (stream words, bit_len, bit_offsets, choice)."""
    sw, bl, bo = exchange_streams(words, bit_len, rel_offsets, device)
    packed = np.packbits(np.asarray(choice_slice, dtype=np.uint8), bitorder="little")
    all_choice = allgather_arrays(packed, device)
    lens = allgather_arrays(np.asarray([len(choice_slice)], dtype=np.int64), device)
    choice = np.concatenate([np.unpackbits(c, bitorder="little")[: int(n[0])] for c, n in zip(all_choice, lens)])
    return sw, bl, bo, choice


def exchange_choice_device(gb, key_prefix, nb, device):
    """NCCL exchange of the choice bits, device to device: one N-byte buffer in
    bucket-sorted key order, each rank's kernel writes its own key range in
    place, then one broadcast per rank range fills the rest.  Returns the
    tensor (every rank holds all N bits)."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    n_keys = int(key_prefix[-1])
    full = torch.empty(max(n_keys, 1), dtype=torch.uint8, device=device)
    ranges = []
    for r in range(world):
        b0, b1 = shard_range(nb, r, world)
        ranges.append((int(key_prefix[b0]), int(key_prefix[b1])))
    k0, k1 = ranges[rank]
    if k1 > k0:
        gb.choice_sorted(k0, k1, dev_ptr=full.data_ptr() + k0)  # synchronises the library stream
    for r, (a, z) in enumerate(ranges):
        if z > a:
            dist.broadcast(full[a:z], src=r)
    torch.cuda.current_stream(device).synchronize()  # the library stream reads it next
    return full


import os

RIBBON_CB = 8192  # back-substitution chunk of the ribbon kernels (csrc/shk_ribbon.cu CB)
# column-sharded ribbon over all ranks (default) or rank 0 alone (SHK_RIBBON_SHARDED=0)
RIBBON_SHARDED = os.environ.get("SHK_RIBBON_SHARDED", "1") != "0"


def column_range(m: int, rank: int, world: int, cb: int = RIBBON_CB) -> Tuple[int, int]:
    """Columns of the ribbon owned by a rank: whole back-substitution chunks."""
    nch = (m + cb - 1) // cb
    a, b = (nch * rank) // world, (nch * (rank + 1)) // world
    return min(a * cb, m), min(b * cb, m)


def identity_map() -> np.ndarray:
    """Boundary map of an empty column range (y passes through)."""
    m = np.zeros((128, 4), dtype=np.uint32)
    for j in range(127):
        m[j, j >> 5] = np.uint32(1 << (j & 31))
    return m


def apply_map(mp: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Image of the 127-bit boundary y (4 uint32 words) under an affine map
    (rows j < 127: image of e_j; row 127: image of 0)."""
    bits = np.unpackbits(np.ascontiguousarray(y, dtype="<u4").view(np.uint8), bitorder="little")[:127].astype(bool)
    out = mp[127].copy()
    if bits.any():
        out ^= np.bitwise_xor.reduce(mp[:127][bits] ^ mp[127], axis=0)
    return out


def ribbon_sharded(gb, choice_sorted, m, max_tries, device=None, begin=None):
    """Column-sharded ribbon solve (SURVEY.md §8(e) option B) over the process
    group; every rank returns (seed, words of the whole system).

    Rank r owns columns column_range(m, r, W).  Each rank eliminates the rows
    starting in its range; rows whose pivot leaves it travel to the right
    neighbour (exchange rounds until no rank exports); then the 127-bit
    boundary solution travels right to left, each rank back-substitutes its
    range, and one all-gather joins the words.  The solution is the
    single-system one."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    c0, c1 = column_range(m, rank, world)
    own = c1 > c0
    dev = device if device is not None else torch.device("cpu")

    def reduce(x, op):
        t = torch.tensor([int(x)], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=op)
        return int(t.item())

    for seed in range(max_tries):
        if begin is not None:  # input-sharded build: routes the rows (a collective), then begins
            nexp, bad = begin(seed, c0, c1, own)
        else:
            nexp, bad = gb.dribbon_begin(choice_sorted, m, seed, c0, c1) if own else (0, False)
        passthrough = np.zeros(0, dtype=np.uint64)
        while True:
            if reduce(bad, dist.ReduceOp.MAX):
                break
            if reduce(nexp, dist.ReduceOp.SUM) == 0:
                break
            out = gb.dribbon_exports(nexp) if own else passthrough
            parts = allgather_arrays(out, device)
            incoming = parts[rank - 1] if rank > 0 else np.zeros(0, dtype=np.uint64)
            if own:
                nexp, bad = gb.dribbon_import(incoming)
            else:  # an empty range forwards what it receives
                passthrough, nexp, bad = incoming, len(incoming) // 3, False
        else:  # pragma: no cover
            pass
        if reduce(bad, dist.ReduceOp.MAX):
            continue
        # back substitution, all ranks at once: each range's first 127
        # solution bits are an affine GF(2) function of the 127 bits right of
        # it; one all-gather of those maps lets every rank compose its own
        # right boundary instead of waiting for a right-to-left hand-off
        my_map = gb.dribbon_map() if own else identity_map()
        maps = [m_.reshape(128, 4) for m_ in allgather_arrays(my_map.reshape(-1), device)]
        y = np.zeros(4, dtype=np.uint32)
        for r in reversed(range(rank + 1, world)):
            y = apply_map(maps[r], y)
        words = gb.dribbon_finish(y, c1 - c0) if own else np.zeros(0, dtype=np.uint64)
        return seed, np.concatenate(allgather_arrays(words, device))
    raise RuntimeError(f"retrieval system unsolvable after {max_tries} seeds")


def agree_flag(flag, device=None) -> bool:
    """True on every rank iff any rank's flag is set (all-reduce MAX): the
    ranks' salt decisions must agree (recsplit.py:433-446)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([1 if flag else 0], dtype=torch.int64, device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return bool(t.item())


def build_hashed_device_sharded(hi_ptr, lo_ptr, n_keys, b, n, mode=1, cache_k=8, epsilon=0.05, device=None, salt=0):
    """Bucket-range-sharded build over the current torch.distributed group.

    Every rank returns the whole descriptor (replicated: the stream, the
    bucket table and the ribbon words are all-gathered) and its own
    device-time profile.  Equal 128-bit codes on any rank raise
    HashCollisionError on every rank (the caller's salt loop retries)."""
    import time

    import torch.distributed as dist

    from . import recsplit, retrieval
    from . import shockhash as leaf_mod
    from ._kernels import kernels as K

    recsplit._validate(n, b, mode)
    if n_keys < 1:
        raise recsplit.InvalidParameterError("key set must be non-empty")
    rank, world = dist.get_rank(), dist.get_world_size()
    t0 = time.perf_counter()
    nb = (n_keys + b - 1) // b
    gb = K.GpuBuild(None, None, nb, hi_ptr=hi_ptr, lo_ptr=lo_ptr, n=n_keys)
    if agree_flag(gb.duplicate, device):
        gb.close()
        raise recsplit.HashCollisionError("equal 128-bit codes in the input")
    key_prefix = gb.key_prefix()
    b0, b1 = shard_range(nb, rank, world)
    leaf_g = recsplit.leaf_g_table(n)
    sizes = np.unique(np.diff(key_prefix[b0 : b1 + 1].astype(np.int64)))
    plans = recsplit.packed_plans_for_sizes(sizes, n, leaf_g)
    ck = cache_k if mode == leaf_mod.MODE_ROTATE_CACHED else 0
    # Only this rank's bucket range gets permuted into leaf order, so choice
    # bits travel in the (rank-independent) bucket-sorted key order and rank
    # 0 builds the ribbon rows from its sorted copy of the keys.
    gb.keep_sorted(True)
    st = gb.run(plans, 0 if mode == leaf_mod.MODE_PLAIN else 1, ck, leaf_mod.CACHE_MIN_LEAF, b0, b1,
                leaf_mod.MAX_SEED)
    words, bit_len, bo = gb.stream()
    rel = bo[: b1 - b0 + 1]
    if device is not None and getattr(device, "type", "cpu") == "cuda":  # NCCL: choice bits stay on the devices
        choice_t = exchange_choice_device(gb, key_prefix, nb, device)
        sw, bl, bit_offsets = exchange_streams(words, bit_len, rel, device)
        choice_all = choice_t.data_ptr()
    else:
        choice = gb.choice_sorted(int(key_prefix[b0]), int(key_prefix[b1]))
        sw, bl, bit_offsets, choice_all = exchange_and_merge(words, bit_len, rel, choice, device)
    m = retrieval._columns(n_keys, epsilon)
    if RIBBON_SHARDED:
        rseed, rwords = ribbon_sharded(gb, choice_all, m, retrieval.RETRY_CAP, device)
    else:  # rank 0 solves alone, then the words are shared
        if rank == 0:
            rseed, rwords = gb.ribbon(m, retrieval.RETRY_CAP, choice=choice_all, sorted_keys=True)
            mine = np.concatenate([np.asarray([rseed], dtype=np.uint64), np.asarray(rwords, dtype=np.uint64)])
        else:
            mine = np.zeros(0, dtype=np.uint64)
        got = allgather_arrays(mine, device)[0]
        rseed, rwords = int(got[0]), got[1:].copy()
    ribbon = retrieval.RibbonSystem(epsilon, rseed, m, rwords)
    desc = recsplit.MphfDescriptor(n_keys, b, n, mode, cache_k, salt, leaf_g, key_prefix, bit_offsets, sw, bl, ribbon)
    desc.build_stats = {"build_seconds": time.perf_counter() - t0}
    phase, split_evals = gb.phase_ms()
    gb.close()
    return desc, {"phase_ms": phase, "split_evals": split_evals, "buckets": (b0, b1),
                  "hash_evals": int(st[0]), "filter_passes": int(st[1]), "leaf_count": int(st[6])}


def build_blob_sharded(blob, key_len, b, n, mode=1, cache_k=8, epsilon=0.05, device=None, fingerprint=None):
    """recsplit.build_blob over the process group: every rank fingerprints the
    host key blob (H2D pipelined with blake2b) and builds its bucket range;
    every rank returns (descriptor, profile).

    The salt loop is the single-GPU one (recsplit.py:433-446): equal codes on
    any rank move every rank to the next salt together (all-reduce MAX of
    the duplicate flag); if the input holds a repeated key every rank raises
    DuplicateKeyError, and HashCollisionError after SALT_RETRY_CAP salts.
    ``fingerprint(blob, key_len, N, salt, d_hi, d_lo)`` replaces the blake2b
    stage (tests force a collision with it)."""
    from . import device as dev
    from . import recsplit

    blob = np.ascontiguousarray(np.frombuffer(blob, dtype=np.uint8) if isinstance(blob, (bytes, bytearray)) else blob,
                                dtype=np.uint8)
    n_keys = len(blob) // key_len
    if n_keys == 0:
        raise recsplit.InvalidParameterError("key set must be non-empty")
    recsplit._validate(n, b, mode)
    fp = fingerprint if fingerprint is not None else dev.blake2b_fixed_from_host
    d_hi = dev.DeviceBuffer(8 * n_keys)
    d_lo = dev.DeviceBuffer(8 * n_keys)
    try:
        for salt in range(recsplit.SALT_RETRY_CAP):
            fp(blob, key_len, n_keys, salt, d_hi, d_lo)
            try:
                return build_hashed_device_sharded(d_hi.ptr, d_lo.ptr, n_keys, b, n, mode, cache_k, epsilon, device,
                                                   salt=salt)
            except recsplit.HashCollisionError:
                pass
            keys = [bytes(blob[i * key_len : (i + 1) * key_len]) for i in range(n_keys)]
            dups = recsplit._find_duplicates(keys)
            if dups:
                raise recsplit.DuplicateKeyError(f"{len(dups)} duplicate key(s), first at line {dups[0] + 1}", dups)
        raise recsplit.HashCollisionError(f"master hash collisions persist after {recsplit.SALT_RETRY_CAP} salts")
    finally:
        d_hi.free()
        d_lo.free()


def query_sharded(desc, hi_ptr, lo_ptr, Q, out_ptr):
    """Replicated descriptor, sharded batch: this rank
    answers queries [Q r/W, Q (r+1)/W) of a batch whose device arrays it
    holds; returns that range."""
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    q0, q1 = (Q * rank) // world, (Q * (rank + 1)) // world
    if q1 > q0:
        desc.device().query_device(hi_ptr + 8 * q0, lo_ptr + 8 * q0, q1 - q0, out_ptr + 8 * q0)
    return q0, q1


class SharedLeafQueue:
    """Cross-GPU leaf queue (one device counter shared over CUDA IPC).

    Rank 0 allocates the counter on its GPU and broadcasts its IPC handle;
    every rank maps it and sets it on its library context, so each rank's
    batched plain leaf search (the seed-block stealing kernel) takes leaves
    from the same counter with system-scope atomics over NVLink.  Every rank
    searches the whole leaf array; each leaf is solved by exactly one rank,
    and the ranks finish together whatever the per-leaf seed counts are
    (contiguous leaf ranges finish when their heaviest leaves do).  Use as a
    context manager around ``search``."""

    def __init__(self, device=None):
        import ctypes

        import torch.distributed as dist

        from . import device as dev
        from ._kernels import _lib

        self._L = _lib.load_library()
        self._ctx = dev.ctx()
        self.rank = dist.get_rank()
        self.device = device
        handle = ctypes.create_string_buffer(64)
        ptr = ctypes.c_void_p()
        if self.rank == 0:
            dev.check(self._L.shk_ipc_counter_alloc(self._ctx, handle, ctypes.byref(ptr)), "ipc alloc")
        obj = [bytes(handle.raw) if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, device=device if getattr(device, "type", "cpu") == "cuda" else None)
        if self.rank != 0:
            h = ctypes.create_string_buffer(obj[0], 64)
            dev.check(self._L.shk_ipc_counter_open(self._ctx, h, ctypes.byref(ptr)), "ipc open")
        self.ptr = ptr.value

    def search(self, hi_ptr, lo_ptr, off_ptr, L, seeds_ptr, fbits_ptr, max_seed=1 << 40):
        """All L leaves (device buffers; every rank holds all of them) with the
        shared queue; returns the rank's kernel time in ms.  The output
        buffers hold, after the call, only the leaves this rank solved: seeds
        of the others are < -1, their f bits 0 (see ``combine``)."""
        import torch.distributed as dist

        from . import device as dev
        from ._kernels import kernels as K

        dist.barrier()  # every rank's previous search has finished before the owner resets the counter
        dev.check(self._L.shk_ctx_set_leaf_counter(self._ctx, self.ptr), "set counter")
        try:
            if self.rank == 0:
                dev.check(self._L.shk_ipc_counter_reset(self._ctx, self.ptr), "ipc reset")
            dev.memset_device(seeds_ptr, 0xFE, 8 * L)
            dev.memset_device(fbits_ptr, 0, 8 * L)
            dev.sync()
            dist.barrier()
            with dev.timer() as tm:
                K.leaf_search_device(hi_ptr, lo_ptr, off_ptr, L, 0, seeds_ptr, fbits_ptr, max_seed=max_seed)
            dev.sync()
        finally:
            dev.check(self._L.shk_ctx_set_leaf_counter(self._ctx, None), "set counter")
        return tm.ms

    def combine(self, seeds, fbits):
        """Every rank's full result from the per-rank partial arrays (host
        numpy): MAX over the seeds (unsolved entries are < -1), SUM over the
        f bits (unsolved entries are 0)."""
        import torch
        import torch.distributed as dist

        dev_ = self.device if self.device is not None else torch.device("cpu")
        s = torch.from_numpy(np.ascontiguousarray(seeds, dtype=np.int64)).to(dev_)
        f = torch.from_numpy(np.ascontiguousarray(fbits).view(np.int64)).to(dev_)
        dist.all_reduce(s, op=dist.ReduceOp.MAX)
        dist.all_reduce(f, op=dist.ReduceOp.SUM)
        return s.cpu().numpy(), f.cpu().numpy().view(np.uint64)

    def close(self):
        from . import device as dev

        if self.ptr:
            dev.check(self._L.shk_ipc_counter_close(self._ctx, self.ptr, 1 if self.rank == 0 else 0), "ipc close")
            self.ptr = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        import torch.distributed as dist

        dist.barrier()  # nobody still uses the owner's counter
        self.close()
        return False


# ---------------------------------------------------------------------------
# Input-sharded build: each rank holds 1/W of the keys and never touches the
# others.  Two all-to-alls replace the replicated fingerprinting and bucket
# sort of all N keys on every rank:
#   1. keys -> the rank owning their bucket (shk_route kind 0), which builds
#      its bucket range from exactly its keys; an all-reduce of the per-bucket
#      counts gives the global key_prefix; the Rice streams are all-gathered
#      as in the replicated path;
#   2. (key, choice bit) in leaf order -> the rank owning the row's start
#      column (shk_route kind 1, per ribbon seed), which starts its column
#      range of the sharded ribbon from exactly those rows
#      (shk_build_dribbon_begin_keys); exports, maps and words as before.
# Same descriptor bytes as the single-GPU build (order independence of the
# bucket sort input and of the ribbon rows).

# route through peer memory (PeerRouter, default) or NCCL all-to-all (SHK_P2P=0)
P2P_ROUTE = os.environ.get("SHK_P2P", "1") != "0"


class _CudaArray:
    def __init__(self, p, n, typestr):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(p), False),
                                         "version": 3, "strides": None}


def _torch_view(p, n, typestr="<i8"):
    """A torch CUDA tensor aliasing n elements at device pointer p."""
    import torch

    if n == 0:
        return torch.empty(0, dtype=torch.int64 if typestr == "<i8" else torch.uint8, device="cuda")
    return torch.as_tensor(_CudaArray(p, n, typestr), device="cuda")


def _all_to_all(send, counts, device):
    """All-to-all of a CUDA tensor grouped by destination (counts[r] rows for
    rank r; rows of any trailing shape); returns the received CUDA tensor,
    grouped by source.  NCCL: all_to_all_single; other backends (gloo on one
    GPU): through the host with all-gathers."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    row = int(np.prod(send.shape[1:])) if send.dim() > 1 else 1
    cnt = [int(c) for c in counts]
    all_c = [np.asarray(x, dtype=np.int64) for x in allgather_arrays(np.asarray(cnt, dtype=np.int64), device)]
    recv_cnt = [int(all_c[r][rank]) for r in range(world)]
    if device is not None and getattr(device, "type", "cpu") == "cuda":
        out = torch.empty((sum(recv_cnt),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
        dist.all_to_all_single(out.view(-1), send.contiguous().view(-1), [c * row for c in recv_cnt],
                               [c * row for c in cnt])
        return out
    host = send.contiguous().view(-1).cpu().numpy()
    parts = allgather_arrays(host, device)
    pieces = []
    for r in range(world):
        off = int(all_c[r][:rank].sum()) * row
        pieces.append(parts[r][off : off + recv_cnt[r] * row])
    flat = np.concatenate(pieces) if pieces else host[:0]
    return torch.from_numpy(flat.copy()).to(send.device).view((-1,) + tuple(send.shape[1:]))


def build_hashed_device_sharded_input(hi_ptr, lo_ptr, n_local, n_keys, b, n, mode=1, cache_k=8, epsilon=0.05,
                                      device=None, salt=0):
    """Bucket-range build where rank r holds only its slice of the master
    codes (device arrays hi/lo of n_local keys; n_keys in all).  Returns the
    whole descriptor on every rank and this rank's profile (see the block
    comment above)."""
    import time

    import torch
    import torch.distributed as dist

    from . import device as dev
    from . import recsplit, retrieval
    from . import shockhash as leaf_mod
    from ._kernels import kernels as K

    recsplit._validate(n, b, mode)
    rank, world = dist.get_rank(), dist.get_world_size()
    t0 = time.perf_counter()
    nb = (n_keys + b - 1) // b
    dev.sync()
    pairs = torch.stack([_torch_view(hi_ptr, n_local), _torch_view(lo_ptr, n_local)], dim=1).contiguous()
    routed = torch.empty_like(pairs)
    torch.cuda.current_stream().synchronize()
    bounds = [shard_range(nb, r, world)[0] for r in range(world)] + [nb]
    if P2P_ROUTE:  # one kernel stores every key into its owner's buffer (peer memory)
        mine, _ = _peer_router(device).route(pairs.data_ptr(), None, n_local, 0, nb, 0, bounds)
    else:
        counts = K.route(pairs.data_ptr(), None, n_local, 0, nb, 0, bounds, routed.data_ptr(), None)
        mine = _all_to_all(routed, counts, device)  # the keys of this rank's buckets
    del pairs, routed
    hi_m, lo_m = mine[:, 0].contiguous(), mine[:, 1].contiguous()
    torch.cuda.current_stream().synchronize()
    n_mine = int(mine.shape[0])
    gb = K.GpuBuild(None, None, nb, hi_ptr=hi_m.data_ptr(), lo_ptr=lo_m.data_ptr(), n=max(n_mine, 1)) if n_mine else None
    dup = bool(gb.duplicate) if gb is not None else False
    if agree_flag(dup, device):
        if gb is not None:
            gb.close()
        raise recsplit.HashCollisionError("equal 128-bit codes in the input")
    b0, b1 = shard_range(nb, rank, world)
    local = np.zeros(nb, dtype=np.int64)
    if gb is not None:
        local = np.diff(gb.key_prefix().astype(np.int64))
    cnt_t = torch.from_numpy(local).to(device if device is not None else "cpu")
    dist.all_reduce(cnt_t, op=dist.ReduceOp.SUM)
    key_prefix = np.zeros(nb + 1, dtype=np.uint64)
    key_prefix[1:] = np.cumsum(cnt_t.cpu().numpy()).astype(np.uint64)
    leaf_g = recsplit.leaf_g_table(n)
    ck = cache_k if mode == leaf_mod.MODE_ROTATE_CACHED else 0
    if gb is not None:
        sizes = np.unique(np.diff(key_prefix[b0 : b1 + 1].astype(np.int64)))
        plans = recsplit.packed_plans_for_sizes(sizes, n, leaf_g)
        st = gb.run(plans, 0 if mode == leaf_mod.MODE_PLAIN else 1, ck, leaf_mod.CACHE_MIN_LEAF, b0, b1,
                    leaf_mod.MAX_SEED)
        words, bit_len, bo = gb.stream()
        rel = bo[: b1 - b0 + 1]
    else:
        st = np.zeros(8, dtype=np.int64)
        words, bit_len, rel = np.zeros(0, dtype=np.uint64), 0, np.zeros(b1 - b0 + 1, dtype=np.uint64)
    sw, bl, bit_offsets = exchange_streams(words, bit_len, rel, device)
    m = retrieval._columns(n_keys, epsilon)
    col_bounds = [column_range(m, r, world)[0] for r in range(world)] + [m]
    if gb is not None:
        kp, cp = gb.leaf_arrays()
    held = {}

    def begin(seed, c0, c1, own):
        if P2P_ROUTE:
            rk, rc = _peer_router(device).route(kp if n_mine else None, cp if n_mine else None, n_mine, 1, m, seed,
                                                col_bounds)
        else:
            k_out = torch.empty((n_mine, 2), dtype=torch.int64, device="cuda")
            c_out = torch.empty(n_mine, dtype=torch.uint8, device="cuda")
            counts_r = (K.route(kp, cp, n_mine, 1, m, seed, col_bounds, k_out.data_ptr(), c_out.data_ptr())
                        if n_mine else np.zeros(world, dtype=np.int64))
            rk = _all_to_all(k_out, counts_r, device)
            rc = _all_to_all(c_out, counts_r, device)
        torch.cuda.current_stream().synchronize()
        held["rows"] = (rk, rc)  # alive until the next seed's begin
        if not own:
            return 0, False
        return gb.dribbon_begin_keys(rk.data_ptr(), rc.data_ptr(), int(rk.shape[0]), m, seed, c0, c1)

    if gb is None and column_range(m, rank, world)[1] > column_range(m, rank, world)[0]:
        raise RuntimeError("a rank without keys cannot own ribbon columns in this build")
    rseed, rwords = ribbon_sharded(gb, None, m, retrieval.RETRY_CAP, device, begin=begin)
    ribbon = retrieval.RibbonSystem(epsilon, rseed, m, rwords)
    desc = recsplit.MphfDescriptor(n_keys, b, n, mode, cache_k, salt, leaf_g, key_prefix, bit_offsets, sw, bl, ribbon)
    desc.build_stats = {"build_seconds": time.perf_counter() - t0}
    phase, split_evals = gb.phase_ms() if gb is not None else ([0.0] * 5, 0)
    if gb is not None:
        gb.close()
    return desc, {"phase_ms": phase, "split_evals": split_evals, "buckets": (b0, b1), "keys_owned": n_mine,
                  "hash_evals": int(st[0]), "filter_passes": int(st[1]), "leaf_count": int(st[6])}


def build_blob_sharded_input(blob, key_len, n_keys, b, n, mode=1, cache_k=8, epsilon=0.05, device=None,
                             fingerprint=None):
    """build_blob where rank r holds only ITS slice of the host key blob (keys
    [N r/W, N (r+1)/W) of n_keys, key_len bytes each): the rank copies and
    fingerprints just that slice, then build_hashed_device_sharded_input.
    The salt loop agrees across ranks (all-reduce of the duplicate flag); a
    repeated key raises DuplicateKeyError on every rank."""
    import torch.distributed as dist

    from . import device as dev
    from . import recsplit

    blob = np.ascontiguousarray(np.frombuffer(blob, dtype=np.uint8) if isinstance(blob, (bytes, bytearray)) else blob,
                                dtype=np.uint8)
    n_local = len(blob) // key_len
    recsplit._validate(n, b, mode)
    fp = fingerprint if fingerprint is not None else dev.blake2b_fixed_from_host
    d_hi = dev.DeviceBuffer(8 * max(n_local, 1))
    d_lo = dev.DeviceBuffer(8 * max(n_local, 1))
    try:
        for salt in range(recsplit.SALT_RETRY_CAP):
            if n_local:
                fp(blob, key_len, n_local, salt, d_hi, d_lo)
            try:
                return build_hashed_device_sharded_input(d_hi.ptr, d_lo.ptr, n_local, n_keys, b, n, mode, cache_k,
                                                         epsilon, device, salt=salt)
            except recsplit.HashCollisionError:
                pass
            # a repeated key may span two ranks' slices: look at all keys
            slices = allgather_arrays(blob, device)
            allb = np.concatenate(slices)
            keys = [bytes(allb[i * key_len : (i + 1) * key_len]) for i in range(len(allb) // key_len)]
            dups = recsplit._find_duplicates(keys)
            if dups:
                raise recsplit.DuplicateKeyError(f"{len(dups)} duplicate key(s), first at line {dups[0] + 1}", dups)
        raise recsplit.HashCollisionError(f"master hash collisions persist after {recsplit.SALT_RETRY_CAP} salts")
    finally:
        d_hi.free()
        d_lo.free()


class PeerRouter:
    """Route + all-to-all fused into one kernel over peer memory
    (shk_route_p2p): every rank maps every other rank's receive buffer once
    (CUDA IPC; NVLink on a multi-GPU node) and the routing kernel stores each
    key straight into its owner's buffer at the slot reserved for this
    source -- the transfer overlaps the hashing key by key instead of
    following it as a separate NCCL all-to-all.  Only the W x W counts and,
    on growth, the 64-byte IPC handles travel through torch.distributed.

    route() returns torch views of this rank's receive buffer (valid until the
    next route())."""

    def __init__(self, device=None):
        import torch.distributed as dist

        from . import device as dev
        from ._kernels import _lib

        self._L = _lib.load_library()
        self._ctx = dev.ctx()
        self.device = device
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.cap = 0
        self.ptrs = None

    def _close(self):
        from . import device as dev

        if self.ptrs is None:
            return
        for r, p in enumerate(self.ptrs):
            dev.check(self._L.shk_ipc_counter_close(self._ctx, p, 1 if r == self.rank else 0), "ipc close")
        self.ptrs = None
        self.cap = 0

    def _ensure(self, need):
        """Every rank's buffer holds >= need keys (collective)."""
        import ctypes

        import torch
        import torch.distributed as dist

        from . import device as dev

        t = torch.tensor([int(need)], dtype=torch.int64, device=self.device if self.device is not None else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        need = int(t.item())
        if self.ptrs is not None and need <= self.cap:
            return
        dist.barrier()  # nobody writes into the old buffers any more
        self._close()
        cap = int(need * 1.25) + 4096
        handle = ctypes.create_string_buffer(64)
        mine = ctypes.c_void_p()
        dev.check(self._L.shk_ipc_buffer_alloc(self._ctx, cap * 17, handle, ctypes.byref(mine)), "ipc alloc")
        hs = allgather_arrays(np.frombuffer(handle.raw, dtype=np.uint8).copy(), self.device)
        ptrs = []
        for r in range(self.world):
            if r == self.rank:
                ptrs.append(mine.value)
                continue
            p = ctypes.c_void_p()
            h = ctypes.create_string_buffer(bytes(hs[r]), 64)
            dev.check(self._L.shk_ipc_counter_open(self._ctx, h, ctypes.byref(p)), "ipc open")
            ptrs.append(p.value)
        self.ptrs, self.cap = ptrs, cap

    def route(self, keys_ptr, aux_ptr, n, kind, nbm, seed, bounds):
        import ctypes

        import torch.distributed as dist

        from . import device as dev

        b = np.ascontiguousarray(bounds, dtype=np.int64)
        W, rank = self.world, self.rank
        counts = np.zeros(W, dtype=np.int64)
        dev.check(self._L.shk_route_count(self._ctx, keys_ptr, int(n), int(kind), int(nbm), int(seed),
                                          b.ctypes.data, W, counts.ctypes.data), "route count")
        C = np.stack([np.asarray(x, dtype=np.int64) for x in allgather_arrays(counts, self.device)])  # [src][dst]
        recv = int(C[:, rank].sum())
        base = np.ascontiguousarray([int(C[:rank, d].sum()) for d in range(W)], dtype=np.int64)
        self._ensure(int(C.sum(axis=0).max()))
        dist.barrier()  # every receiver is done with the previous contents
        arr = (ctypes.c_void_p * W)(*self.ptrs)
        dev.check(self._L.shk_route_p2p(self._ctx, keys_ptr, aux_ptr, int(n), int(kind), int(nbm), int(seed),
                                        b.ctypes.data, W, arr, base.ctypes.data, int(self.cap)), "route p2p")
        dist.barrier()  # every sender's stores have landed
        k = _torch_view(self.ptrs[rank], 2 * recv).view(-1, 2) if recv else _torch_view(0, 0).view(-1, 2)
        a = _torch_view(self.ptrs[rank] + 16 * self.cap, recv, "|u1") if recv else _torch_view(0, 0, "|u1")
        return k, a


_PEER = None


def _peer_router(device):
    global _PEER
    import torch.distributed as dist

    if _PEER is None or _PEER.world != dist.get_world_size():
        _PEER = PeerRouter(device)
    return _PEER
