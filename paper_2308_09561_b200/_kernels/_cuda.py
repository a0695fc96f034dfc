"""The CUDA kernel backend: the drop-in for the reference's kernel seam.

Mirrors the function set of ``shockhash._kernels.kernels`` (reference
/root/reference/pkg/src/shockhash/_kernels/_core.pyx, same names, argument
meaning, return values and error behaviour) so upper layers and tests read
like the reference's.  Every hot function runs on the B200 through the C-ABI;
batched variants (``*_batch``) expose the GPU-shaped entry points.

The numpy ``*_batch`` mixers are array utilities of the seam (the reference's
are numpy too, _core.pyx:105-118); the product's bucketing and ribbon rows
hash on the GPU.
"""

import ctypes

import numpy as np

from ..errors import FormatError, InvalidParameterError
from . import _lib
from ._lib import SHK_BUILD_ASYNC, SHK_DEVICE, check, ctx, i64, load_library, ptr, u64

NAME = "cuda"

MASK64 = 0xFFFFFFFFFFFFFFFF
GOLDEN = 0x9E3779B97F4A7C15
_MUL1 = 0xBF58476D1CE4E5B9
_MUL2 = 0x94D049BB133111EB
RIBBON_W = 128

TAG_LEAF = 1
TAG_SPLITBIT = 2
TAG_SPLIT = 3
TAG_BUCKET = 4
TAG_RSTART = 5
TAG_RPAT0 = 6
TAG_RPAT1 = 7


def _L():
    return load_library()


# ---------------------------------------------------------------------------
# Scalar hash family: host entry points of the __host__ __device__ source the
# kernels use (include/shockhash_b200.h).


def mix64(z):
    return int(_L().shk_mix64(int(z) & MASK64))


def seed_mixer(seed, tag):
    return int(_L().shk_seed_mixer(int(seed) & MASK64, int(tag)))


def remix(hi, lo, seed, tag):
    return int(_L().shk_remix(int(hi) & MASK64, int(lo) & MASK64, int(seed) & MASK64, int(tag)))


def hash_range(v, m):
    return int(_L().shk_hash_range(int(v) & MASK64, int(m)))


def leaf_pair(hi, lo, seed, n):
    h0 = ctypes.c_int()
    h1 = ctypes.c_int()
    _L().shk_leaf_pair(int(hi) & MASK64, int(lo) & MASK64, int(seed) & MASK64, int(n), ctypes.byref(h0), ctypes.byref(h1))
    return h0.value, h1.value


def split_bit(hi, lo, seed):
    return int(_L().shk_split_bit(int(hi) & MASK64, int(lo) & MASK64, int(seed) & MASK64))


def leaf_cell(hi, lo, q, mleaf, mode, cache_k, choice):
    return int(_L().shk_leaf_cell(int(hi) & MASK64, int(lo) & MASK64, int(q), int(mleaf), int(mode), int(cache_k), int(choice)))


def mix64_batch(z):
    z = np.asarray(z, dtype=np.uint64)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_MUL1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_MUL2)
    return z ^ (z >> np.uint64(31))


def remix_batch(hi, lo, seed, tag):
    x = np.uint64(seed_mixer(seed, tag))
    return mix64_batch(mix64_batch(np.asarray(hi, dtype=np.uint64) ^ x) ^ np.asarray(lo, dtype=np.uint64))


def hash_range_batch(v, m):
    return ((np.asarray(v, dtype=np.uint64) >> np.uint64(32)) * np.uint64(m)) >> np.uint64(32)


# ---------------------------------------------------------------------------
# Leaf searches


def leaf_search_batch(hi, lo, leaf_off, mode, cache_k=0, cache_min_leaf=0, max_seed=1 << 40, team_warps=0, stats=True):
    """Batched leaf search over CSR leaves on the GPU.

    Returns (seeds i64[L], fbits u64[L], stats i64[L,4] or None).
    mode 0: plain; mode 1: rotation fitting (cache_k applied to leaves with
    more than cache_min_leaf keys).
    """
    hi = u64(hi).ravel()
    lo = u64(lo).ravel()
    off = i64(leaf_off)
    L = len(off) - 1
    seeds = np.empty(max(L, 0), dtype=np.int64)
    fb = np.empty(max(L, 0), dtype=np.uint64)
    st = np.empty((max(L, 0), 4), dtype=np.int64) if stats else None
    if L > 0:
        rc = _L().shk_leaf_search(ctx(), int(mode), int(cache_k), int(cache_min_leaf), ptr(hi), ptr(lo), ptr(off), L,
                                  int(max_seed), int(team_warps), ptr(seeds), ptr(fb), ptr(st), 0)
        check(rc, "leaf search")
    return seeds, fb, st


def leaf_search_device(hi_ptr, lo_ptr, off_ptr, L, mode, seeds_ptr, fbits_ptr=None, stats_ptr=None, cache_k=0,
                       cache_min_leaf=0, max_seed=1 << 40, team_warps=0):
    """Stream-ordered batched leaf search on device pointers (bench path)."""
    check(_L().shk_leaf_search(ctx(), int(mode), int(cache_k), int(cache_min_leaf), hi_ptr, lo_ptr, off_ptr, int(L),
                               int(max_seed), int(team_warps), seeds_ptr, fbits_ptr, stats_ptr, SHK_DEVICE),
          "leaf search")


def _one_leaf(hi, lo, n, mode, cache_k, max_seed):
    hi = u64(hi)
    lo = u64(lo)
    if len(hi) != n or len(lo) != n:
        raise InvalidParameterError(f"expected {n} keys, got {len(hi)}")
    if not 1 <= n <= 64:
        raise InvalidParameterError(f"leaf size must be in 1..64, got {n}")
    if n == 1:
        return (0, 1, 1, 1, 0), 0
    if max_seed < 0:
        return (-1, 0, 0, 0, 0), 0
    off = np.array([0, n], dtype=np.int64)
    seeds, fb, st = leaf_search_batch(hi, lo, off, mode, cache_k, 0, max_seed)
    return (int(seeds[0]), int(st[0, 0]), int(st[0, 1]), int(st[0, 2]), int(st[0, 3])), int(fb[0])


def search_plain(hi, lo, n, max_seed):
    """Minimum plain seed: (seed, evals, passes, checks, a_evals) (_core.pyx:186-229)."""
    return _one_leaf(hi, lo, int(n), 0, 0, int(max_seed))[0]


def search_rotate(hi, lo, n, cache_k, max_seed):
    """Rotation fitting: (base*n + r, evals, passes, checks, a_evals) (_core.pyx:238-334)."""
    return _one_leaf(hi, lo, int(n), 1, int(cache_k), int(max_seed))[0]


def search_plain_fbits(hi, lo, n, max_seed):
    """search_plain plus the orientation bits of the found seed."""
    return _one_leaf(hi, lo, int(n), 0, 0, int(max_seed))


def search_rotate_fbits(hi, lo, n, cache_k, max_seed):
    return _one_leaf(hi, lo, int(n), 1, int(cache_k), int(max_seed))


def orient_batch(edges_u, edges_v, off):
    """Canonical orientation of CSR edge lists on the GPU -> (fbits, ok)."""
    eu = np.ascontiguousarray(np.asarray(edges_u, dtype=np.uint8))
    ev = np.ascontiguousarray(np.asarray(edges_v, dtype=np.uint8))
    off = i64(off)
    L = len(off) - 1
    fb = np.zeros(L, dtype=np.uint64)
    ok = np.zeros(L, dtype=np.int32)
    if L > 0:
        check(_L().shk_orient(ctx(), ptr(eu), ptr(ev), ptr(off), L, ptr(fb), ptr(ok), 0), "orient")
    return fb, ok


# ---------------------------------------------------------------------------
# Splitting


def split_seed_search(hi, lo, sizes, max_seed):
    """Minimum seed realizing the part sizes: (seed, evals) (_core.pyx:385-428)."""
    hi = u64(hi)
    lo = u64(lo)
    sz = i64(list(sizes))
    m = len(hi)
    if int(sz.sum()) != m:
        raise InvalidParameterError("part sizes must sum to the number of keys")
    if max_seed <= 0 or m == 0:
        return (0, 0) if (m == 0 and max_seed > 0) else (-1, 0)
    seed = ctypes.c_int64()
    ev = ctypes.c_int64()
    check(_L().shk_split_search(ctx(), ptr(hi), ptr(lo), m, ptr(sz), len(sz), int(max_seed), ctypes.byref(seed),
                                ctypes.byref(ev)), "split search")
    return int(seed.value), int(ev.value)


def split_parts(hi, lo, seed, sizes):
    """Part index of every key (_core.pyx:378-382)."""
    hi = u64(hi)
    lo = u64(lo)
    sz = i64(list(sizes))
    m = len(hi)
    out = np.zeros(m, dtype=np.int64)
    if m:
        check(_L().shk_split_parts(ctx(), ptr(hi), ptr(lo), m, int(seed) & MASK64, ptr(sz), len(sz), ptr(out)),
              "split parts")
    return out


# ---------------------------------------------------------------------------
# Ribbon


def ribbon_rows(hi, lo, seed, m):
    hi = u64(hi)
    lo = u64(lo)
    N = len(hi)
    starts = np.zeros(N, dtype=np.int64)
    p0 = np.zeros(N, dtype=np.uint64)
    p1 = np.zeros(N, dtype=np.uint64)
    if N:
        check(_L().shk_ribbon_rows(ctx(), ptr(hi), ptr(lo), N, int(m), int(seed) & MASK64, ptr(starts), ptr(p0), ptr(p1), 0),
              "ribbon rows")
    return starts, p0, p1


def ribbon_solve(starts, pat0, pat1, rhs, m):
    """Solution words (u64, LSB-first) or None if inconsistent (_core.pyx:442-524)."""
    starts = i64(starts)
    p0 = u64(pat0)
    p1 = u64(pat1)
    r = np.ascontiguousarray(np.asarray(rhs, dtype=np.uint8))
    m = int(m)
    words = np.zeros((m + 63) // 64, dtype=np.uint64)
    ok = ctypes.c_int(0)
    check(_L().shk_ribbon_solve(ctx(), ptr(starts), ptr(p0), ptr(p1), ptr(r), len(starts), m, ptr(words),
                                ctypes.byref(ok), 0), "ribbon solve")
    return words if ok.value else None


def ribbon_query_many(starts, pat0, pat1, words, m):
    starts = i64(starts)
    p0 = u64(pat0)
    p1 = u64(pat1)
    w = u64(words)
    out = np.zeros(len(starts), dtype=np.uint8)
    if len(starts):
        check(_L().shk_ribbon_query(ctx(), ptr(starts), ptr(p0), ptr(p1), len(starts), ptr(w), len(w), ptr(out), 0),
              "ribbon query")
    return out


def ribbon_build(hi, lo, rhs, m, max_tries=64):
    """The retrieval seed loop on the GPU: (seed, words); raises on failure."""
    hi = u64(hi)
    lo = u64(lo)
    r = np.ascontiguousarray(np.asarray(rhs, dtype=np.uint8))
    m = int(m)
    words = np.zeros((m + 63) // 64, dtype=np.uint64)
    seed = ctypes.c_uint64(0)
    check(_L().shk_ribbon_build(ctx(), ptr(hi), ptr(lo), ptr(r), len(hi), m, int(max_tries), ctypes.byref(seed),
                                ptr(words), 0), "ribbon build")
    return int(seed.value), words


# ---------------------------------------------------------------------------
# Analysis entry points (experiments.py)


def search_bruteforce(hi, lo, n, max_seed):
    """Single-hash bijection retry: (seed or -1, evals) (_core.pyx:337-371)."""
    n = int(n)
    if n < 0 or n > 64:
        raise InvalidParameterError("search_bruteforce supports 0 <= n <= 64")
    hi = u64(np.asarray(hi, dtype=np.uint64)[:n])
    lo = u64(np.asarray(lo, dtype=np.uint64)[:n])
    if len(hi) < n or len(lo) < n:
        raise InvalidParameterError("need n keys")
    seed = ctypes.c_int64()
    ev = ctypes.c_int64()
    check(_L().shk_search_bruteforce(ctx(), ptr(hi), ptr(lo), n, max(0, int(max_seed)), ctypes.byref(seed),
                                     ctypes.byref(ev)), "search bruteforce")
    return int(seed.value), int(ev.value)


def mc_filter_pass_count(n, trials, entropy):
    """Seeds in [0, trials) whose cells cover all n (_core.pyx:832-860)."""
    out = ctypes.c_int64()
    check(_L().shk_mc_filter_pass_count(ctx(), int(n), int(trials), int(entropy) & MASK64, ctypes.byref(out)),
          "mc filter pass count")
    return int(out.value)


def enumerate_outcomes(n):
    """(pseudoforest count, sum of 2^components) over all n^(2n) tuples (_core.pyx:778-829)."""
    n = int(n)
    if n > 8:
        raise ValueError("enumeration limited to n <= 8")
    pf = ctypes.c_uint64()
    s2 = ctypes.c_uint64()
    check(_L().shk_enumerate_outcomes(ctx(), n, ctypes.byref(pf), ctypes.byref(s2)), "enumerate outcomes")
    return int(pf.value), int(s2.value)


# ---------------------------------------------------------------------------
# Bit stream


def rice_decode_stream(words, bit_len, pos, g):
    """Decode one Rice code: (value, new_pos) (_core.pyx:626-635)."""
    v, p = rice_decode_many(words, bit_len, pos, [g])
    return int(v[0]), int(p[0])


def rice_decode_many(words, bit_len, pos, gs):
    w = u64(words)
    g = np.ascontiguousarray(np.asarray(gs, dtype=np.int32))
    vals = np.zeros(len(g), dtype=np.int64)
    poss = np.zeros(len(g), dtype=np.int64)
    if int(pos) >= int(bit_len) and len(g):
        raise FormatError("bit stream overrun")
    check(_L().shk_rice_decode(ctx(), ptr(w), len(w), int(bit_len), int(pos), ptr(g), len(g), ptr(vals), ptr(poss)),
          "rice decode")
    return vals, poss


# ---------------------------------------------------------------------------
# Master hash


def blake2b128_many(keys, salt=0):
    """blake2b-128 (salted) of byte-string keys on the GPU -> (hi, lo)."""
    n = len(keys)
    lens = np.fromiter((len(k) for k in keys), dtype=np.int64, count=n)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    blob = np.frombuffer(b"".join(keys), dtype=np.uint8) if n else np.zeros(1, dtype=np.uint8)
    return blake2b128_blob(blob, off, salt)


def blake2b128_blob(blob, off, salt=0):
    blob = np.ascontiguousarray(blob, dtype=np.uint8)
    off = i64(off)
    n = len(off) - 1
    hi = np.zeros(n, dtype=np.uint64)
    lo = np.zeros(n, dtype=np.uint64)
    if n > 0:
        if len(blob) == 0:
            blob = np.zeros(1, dtype=np.uint8)
        check(_L().shk_blake2b128(ctx(), ptr(blob), int(off[-1]), ptr(off), n, int(salt) & MASK64, ptr(hi), ptr(lo), 0),
              "blake2b")
    return hi, lo


# ---------------------------------------------------------------------------
# Plans + batch query


class PackedPlans:
    """Reference plan arrays (recsplit.flatten_plan) packed for the C-ABI."""

    def __init__(self, plans: dict):
        sizes = sorted(int(m) for m in plans)
        self.plan_m = np.asarray(sizes, dtype=np.int64)
        fields = {k: [] for k in ("kind", "g", "fanout", "sizes_off", "subtree", "m_node")}
        flats = []
        plan_off = [0]
        sizes_base = []
        base = 0
        for m in sizes:
            kind, g, fanout, sizes_off, sizes_flat, subtree, m_node = plans[m]
            for name, arr in zip(("kind", "g", "fanout", "sizes_off", "subtree", "m_node"),
                                 (kind, g, fanout, sizes_off, subtree, m_node)):
                fields[name].append(np.asarray(arr, dtype=np.int64))
            plan_off.append(plan_off[-1] + len(kind))
            sizes_base.append(base)
            sf = np.asarray(sizes_flat, dtype=np.int64)
            flats.append(sf)
            base += len(sf)
        cat = lambda xs: np.ascontiguousarray(np.concatenate(xs) if xs else np.zeros(1, dtype=np.int64))
        for k, v in fields.items():
            setattr(self, k, cat(v))
        self.sizes_flat = cat(flats)
        self.plan_off = np.asarray(plan_off, dtype=np.int64)
        self.sizes_base = np.asarray(sizes_base or [0], dtype=np.int64)
        s = _lib.ShkPlans()
        s.nplans = len(sizes)
        s.plan_m = ptr(self.plan_m) if len(sizes) else None
        s.plan_off = ptr(self.plan_off)
        s.sizes_base = ptr(self.sizes_base)
        s.kind = ptr(self.kind)
        s.g = ptr(self.g)
        s.fanout = ptr(self.fanout)
        s.sizes_off = ptr(self.sizes_off)
        s.subtree = ptr(self.subtree)
        s.m_node = ptr(self.m_node)
        s.sizes_flat = ptr(self.sizes_flat)
        self.struct = s


class DeviceDescriptor:
    """A descriptor uploaded to the GPU with its derived node index."""

    def __init__(self, n_keys, nbuckets, key_prefix, bit_offsets, stream_words, stream_bit_len, plans, mode, cache_k,
                 rib_seed, rib_m, rib_words):
        self._keep = []
        kp = u64(key_prefix)
        bo = u64(bit_offsets)
        sw = u64(stream_words) if len(stream_words) else np.zeros(1, dtype=np.uint64)
        rw = u64(rib_words) if rib_words is not None and len(rib_words) else np.zeros(1, dtype=np.uint64)
        pk = plans if isinstance(plans, PackedPlans) else PackedPlans(plans)
        self._keep += [kp, bo, sw, rw, pk]
        if len(kp) != int(nbuckets) + 1 or len(bo) < int(nbuckets) + 1:
            raise InvalidParameterError("bucket tables do not match nbuckets")
        h = ctypes.c_void_p()
        nw = len(stream_words)
        check(_L().shk_qdesc_create(ctx(), int(n_keys), int(nbuckets), int(mode), int(cache_k), ptr(kp), ptr(bo), ptr(sw),
                                    nw, int(stream_bit_len), ctypes.byref(pk.struct), int(rib_seed) & MASK64, int(rib_m),
                                    ptr(rw), len(rib_words) if rib_words is not None else 0, ctypes.byref(h)),
              "descriptor upload")
        self.handle = h

    def query(self, hi, lo, clamp=True):
        hi = u64(hi).ravel()
        lo = u64(lo).ravel()
        out = np.zeros(len(hi), dtype=np.uint64)
        if len(hi):
            check(_L().shk_query(self.handle, ptr(hi), ptr(lo), len(hi), ptr(out), 1 if clamp else 0, 0), "query")
        return out

    def verify(self, hi, lo):
        """(ok, offender index or -1): outputs of the hashed keys form a
        bijection onto [0, N), checked on the device."""
        hi = u64(hi).ravel()
        lo = u64(lo).ravel()
        ok = ctypes.c_int(0)
        off = ctypes.c_int64(-1)
        check(_L().shk_verify(self.handle, ptr(hi), ptr(lo), len(hi), 0, ctypes.byref(ok), ctypes.byref(off)), "verify")
        return bool(ok.value), int(off.value)

    def query_blob(self, blob, key_len, salt, out=None, clamp=True):
        """Indices of N fixed-length keys packed in a host buffer (ideally
        page-locked): H2D, blake2b, query and D2H pipelined in chunks."""
        blob = np.ascontiguousarray(blob, dtype=np.uint8)
        Q = len(blob) // int(key_len)
        if out is None:
            out = np.empty(Q, dtype=np.uint64)
        if Q:
            check(_L().shk_query_blob(self.handle, ptr(blob), int(key_len), Q, int(salt), ptr(out), 1 if clamp else 0),
                  "query")
        return out

    def query_device(self, hi_ptr, lo_ptr, Q, out_ptr, clamp=True):
        """Stream-ordered query on device pointers (bench / zero-copy)."""
        check(_L().shk_query(self.handle, hi_ptr, lo_ptr, int(Q), out_ptr, 1 if clamp else 0, SHK_DEVICE), "query")

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _lib._lib is not None:
                _lib._lib.shk_qdesc_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def query_stream(hi, lo, nbuckets, key_prefix, bit_offsets, stream_words, stream_bit_len, plans, mode, cache_k,
                 rib_seed, rib_m, rib_words):
    """Batched MPHF evaluation (_core.pyx:642-742), unclamped like the seam."""
    n_keys = int(np.asarray(key_prefix, dtype=np.uint64)[-1])
    d = DeviceDescriptor(n_keys, nbuckets, key_prefix, bit_offsets, stream_words, stream_bit_len, plans, mode, cache_k,
                         rib_seed, rib_m, rib_words)
    return d.query(hi, lo, clamp=False)


# ---------------------------------------------------------------------------
# MPHF construction runtime (native orchestration in the C-ABI)


def route(keys_ptr, aux_ptr, n, kind, nbm, seed, bounds, keys_out_ptr, aux_out_ptr):
    """Partition n device keys (interleaved pairs) by owner rank (kind 0:
    bucket, kind 1: ribbon start column; rank r owns [bounds[r],
    bounds[r+1])) into keys_out (and the per-key bytes aux into aux_out);
    returns the group sizes."""
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    W = len(b) - 1
    counts = np.zeros(W, dtype=np.int64)
    check(_L().shk_route(ctx(), keys_ptr, aux_ptr, int(n), int(kind), int(nbm), int(seed), ptr(b), W, keys_out_ptr,
                         aux_out_ptr, ptr(counts)), "route")
    return counts


class GpuBuild:
    """Handle on a device-side build: bucketed keys, tree, stream, ribbon.

    Phases mirror recsplit._build_hashed (recsplit.py:474-550): bucketize
    (sort by (bucket, hi, lo) + duplicate flag) -> run (split/leaf/Rice over a
    bucket range) -> ribbon (over all keys).
    """

    def __init__(self, hi, lo, nbuckets, hi_ptr=None, lo_ptr=None, n=None, asynchronous=False):
        """asynchronous (device inputs only): return once the key prefix is
        on the host, the sort still running; `duplicate` then waits for it,
        and run() raises HashCollisionError itself on equal codes."""
        self.handle = None
        if hi_ptr is not None:
            N = int(n)
            src_hi, src_lo, flags = hi_ptr, lo_ptr, SHK_DEVICE | (SHK_BUILD_ASYNC if asynchronous else 0)
        else:
            hi = u64(hi)
            lo = u64(lo)
            N = len(hi)
            src_hi, src_lo, flags = ptr(hi), ptr(lo), 0
        self.N = N
        self.nbuckets = int(nbuckets)
        h = ctypes.c_void_p()
        dup = ctypes.c_int(0)
        mb = ctypes.c_int64(0)
        check(_L().shk_build_create(ctx(), src_hi, src_lo, N, self.nbuckets, flags, ctypes.byref(h), ctypes.byref(dup),
                                    ctypes.byref(mb)), "bucketize")
        self.handle = h
        self._dup = None if dup.value < 0 else bool(dup.value)
        self.max_bucket = int(mb.value)

    @property
    def duplicate(self):
        if self._dup is None:
            d = ctypes.c_int(0)
            check(_L().shk_build_duplicate(self.handle, ctypes.byref(d)), "bucketize")
            self._dup = bool(d.value)
        return self._dup

    def key_prefix(self):
        out = np.zeros(self.nbuckets + 1, dtype=np.uint64)
        check(_L().shk_build_key_prefix(self.handle, ptr(out)))
        return out

    def sorted_keys(self):
        hi = np.zeros(self.N, dtype=np.uint64)
        lo = np.zeros(self.N, dtype=np.uint64)
        check(_L().shk_build_sorted_keys(self.handle, ptr(hi), ptr(lo)))
        return hi, lo

    def record_placements(self, on=True):
        check(_L().shk_build_set_record_placements(self.handle, 1 if on else 0))

    def placements(self):
        out = np.zeros(self.N, dtype=np.int64)
        check(_L().shk_build_placements(self.handle, ptr(out)), "placements")
        return out

    def run(self, plans, mode, cache_k, cache_min_leaf, b0, b1, max_seed):
        pk = plans if isinstance(plans, PackedPlans) else PackedPlans(plans)
        st = np.zeros(8, dtype=np.int64)
        check(_L().shk_build_run(self.handle, ctypes.byref(pk.struct), int(mode), int(cache_k), int(cache_min_leaf),
                                 int(b0), int(b1), int(max_seed), ptr(st)), "build")
        return st

    def stream(self):
        bl = ctypes.c_int64()
        nw = ctypes.c_int64()
        check(_L().shk_build_stream_size(self.handle, ctypes.byref(bl), ctypes.byref(nw)))
        words = np.zeros(nw.value, dtype=np.uint64)
        # bit offsets of the run's bucket range (+1)
        bo = np.zeros(self.nbuckets + 1, dtype=np.uint64)
        check(_L().shk_build_stream(self.handle, ptr(words) if nw.value else None, ptr(bo)))
        return words, int(bl.value), bo

    def choice(self):
        out = np.zeros(self.N, dtype=np.uint8)
        check(_L().shk_build_choice(self.handle, ptr(out)))
        return out

    def keep_sorted(self, on=True):
        """Keep the bucket-sorted keys (before run) for choice_sorted/ribbon(sorted_keys=True)."""
        check(_L().shk_build_set_keep_sorted(self.handle, 1 if on else 0))

    def choice_sorted(self, k0, k1, dev_ptr=None):
        """Choice bits of build positions [k0, k1) in bucket-sorted key order
        (host array, or written to the device pointer dev_ptr)."""
        if dev_ptr is not None:
            check(_L().shk_build_choice_sorted(self.handle, int(k0), int(k1), int(dev_ptr), SHK_DEVICE),
                  "choice_sorted")
            return None
        out = np.zeros(max(int(k1) - int(k0), 0), dtype=np.uint8)
        check(_L().shk_build_choice_sorted(self.handle, int(k0), int(k1), ptr(out) if len(out) else None, 0),
              "choice_sorted")
        return out

    # column-sharded ribbon (dist.ribbon_sharded drives the exchange)
    def dribbon_begin(self, choice_sorted, m, seed, c0, c1):
        """choice_sorted: all N choice bits in sorted order, a host array or
        an int device pointer."""
        if isinstance(choice_sorted, int):
            cp, fl = choice_sorted, SHK_DEVICE
        else:
            ch = np.ascontiguousarray(choice_sorted, dtype=np.uint8)
            cp, fl = ptr(ch), 0
        nexp = ctypes.c_int64(0)
        bad = ctypes.c_int(0)
        check(_L().shk_build_dribbon_begin(self.handle, cp, fl, int(m), int(seed), int(c0), int(c1),
                                           ctypes.byref(nexp), ctypes.byref(bad)), "ribbon (sharded)")
        return int(nexp.value), bool(bad.value)

    def dribbon_begin_keys(self, keys_ptr, rhs_ptr, n, m, seed, c0, c1):
        """Column-sharded ribbon from explicit device keys (interleaved pairs)
        and rhs bytes routed to this rank (input-sharded build)."""
        nexp = ctypes.c_int64(0)
        bad = ctypes.c_int(0)
        check(_L().shk_build_dribbon_begin_keys(self.handle, keys_ptr, rhs_ptr, int(n), int(m), int(seed), int(c0),
                                                int(c1), ctypes.byref(nexp), ctypes.byref(bad)), "ribbon (sharded)")
        return int(nexp.value), bool(bad.value)

    def leaf_arrays(self):
        """(keys, choice) device pointers: the keys in leaf order
        (interleaved pairs) and their choice bytes, after run()."""
        k = ctypes.c_void_p()
        c = ctypes.c_void_p()
        check(_L().shk_build_leaf_arrays(self.handle, ctypes.byref(k), ctypes.byref(c)), "leaf arrays")
        return k.value, c.value

    def dribbon_exports(self, n):
        rows = np.zeros(3 * max(int(n), 0), dtype=np.uint64)
        check(_L().shk_build_dribbon_exports(self.handle, ptr(rows) if len(rows) else None, int(n)), "ribbon exports")
        return rows

    def dribbon_import(self, rows):
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        nexp = ctypes.c_int64(0)
        bad = ctypes.c_int(0)
        check(_L().shk_build_dribbon_import(self.handle, ptr(rows) if len(rows) else None, len(rows) // 3,
                                            ctypes.byref(nexp), ctypes.byref(bad)), "ribbon import")
        return int(nexp.value), bool(bad.value)

    def dribbon_backsub(self, y_in, ncols):
        y_in = np.ascontiguousarray(y_in, dtype=np.uint32)
        y_out = np.zeros(4, dtype=np.uint32)
        words = np.zeros((int(ncols) + 63) // 64, dtype=np.uint64)
        check(_L().shk_build_dribbon_backsub(self.handle, ptr(y_in), ptr(y_out), ptr(words)), "ribbon backsub")
        return y_out, words

    def dribbon_map(self):
        """This range's boundary map, uint32[128, 4] (rows j < 127: image of
        e_j, row 127: image of 0)."""
        out = np.zeros((128, 4), dtype=np.uint32)
        check(_L().shk_build_dribbon_map(self.handle, ptr(out)), "ribbon map")
        return out

    def dribbon_finish(self, y_in, ncols):
        y_in = np.ascontiguousarray(y_in, dtype=np.uint32)
        words = np.zeros((int(ncols) + 63) // 64, dtype=np.uint64)
        check(_L().shk_build_dribbon_finish(self.handle, ptr(y_in), ptr(words)), "ribbon finish")
        return words

    def ribbon(self, m, max_tries=64, choice=None, sorted_keys=False):
        words = np.zeros((int(m) + 63) // 64, dtype=np.uint64)
        seed = ctypes.c_uint64(0)
        flags = 4 if sorted_keys else 0  # SHK_RIBBON_SORTED_KEYS
        if isinstance(choice, int):  # device pointer
            ch, flags = choice, flags | SHK_DEVICE
        else:
            ch = None if choice is None else ptr(np.ascontiguousarray(choice, dtype=np.uint8))
        check(_L().shk_build_ribbon(self.handle, ch, flags, int(m), int(max_tries), ctypes.byref(seed),
                                    ptr(words)), "ribbon")
        return int(seed.value), words

    def phase_ms(self):
        """Device ms of [bucketize, splits, leaves, rice, ribbon] + split evals."""
        ms = (ctypes.c_float * 5)()
        ev = ctypes.c_int64(0)
        check(_L().shk_build_phase_ms(self.handle, ms, ctypes.byref(ev)))
        return [float(x) for x in ms], int(ev.value)

    def level_ms(self):
        """Device ms per split level (tree depth) of the last run."""
        ms = (ctypes.c_float * 64)()
        dp = (ctypes.c_int32 * 64)()
        k = _L().shk_build_level_ms(self.handle, ms, dp, 64)
        return {int(dp[i]): round(float(ms[i]), 3) for i in range(k)}

    def close(self):
        if self.handle is not None and _lib._lib is not None:
            _lib._lib.shk_build_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
