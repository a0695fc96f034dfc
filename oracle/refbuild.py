"""Reference CPU arm for bench.py — TEST/BASELINE INFRASTRUCTURE.

Times the reference's CPU implementation of the C4 build on a bounded
sample: the reference's OWN compiled kernels (oracle/_ref/_core*.so, the
Cython module /root/reference/pkg/src/shockhash/_kernels/_core.pyx compiled
by oracle/build_ref.sh) driven by the reference's construction loop,
restated here from recsplit.py:474-594 (per-node split_seed_search +
split_parts + stable argsort, per-leaf search_rotate + edge reconstruction +
pseudoforest.orient, Rice writer, then retrieval_build_arrays).  The
reference runs buckets one after another; here buckets go to a process pool
over all host cores (they are independent), the global ribbon stays
sequential as in the reference.  If _ref is absent the C oracle port
(shk_oracle.c, OpenMP over buckets) is timed instead (kind "port").
"""

import hashlib
import math
import multiprocessing as mp
import os
import struct
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")
MAX_SEED = 1 << 40
C4 = dict(N=10_000_000, n=40, b=2000)

_K = None


def ref_kernels():
    global _K
    if _K is None:
        if REF not in sys.path:
            sys.path.insert(0, REF)
        import _core  # the reference's compiled kernels

        _K = _core
    return _K


def have_ref():
    try:
        ref_kernels()
        return True
    except Exception:
        return False


# ---- restated orchestration (recsplit.py / shockhash.py / pseudoforest.py) --

def plan(m, n):
    if m <= n:
        return ("leaf", m)
    if n <= 24:
        unit = n
    else:
        if m <= 4 * n:
            return ("split", _parts(m, n))
        if m <= 12 * n:
            return ("split", _parts(m, 4 * n))
        unit = 12 * n
    left = unit * ((m + 2 * unit - 1) // (2 * unit))
    return ("split", (min(max(left, 1), m - 1), m - min(max(left, 1), m - 1)))


def _parts(m, part):
    q, r = divmod(m, part)
    return tuple([part] * q + ([r] if r else []))


def split_rice_param(m, sizes):
    logp = math.lgamma(m + 1)
    for s in sizes:
        logp -= math.lgamma(s + 1)
        logp += s * (math.log(s) - math.log(m))
    return max(0, int(-logp / math.log(2.0)))


def leaf_rice_param(m):
    if m <= 1:
        return 0
    t = m * math.log2(math.e / 2.0) + math.log2(math.e) - 0.5 * math.log2(math.pi) - 0.5 * math.log2(m)
    return max(0, int(t))


class BitWriter:
    def __init__(self):
        self.words = []
        self.bit_len = 0

    def append(self, value, nbits):
        pos = self.bit_len
        self.bit_len += nbits
        while (self.bit_len + 63) // 64 > len(self.words):
            self.words.append(0)
        i, sh = pos >> 6, pos & 63
        self.words[i] |= (value << sh) & 0xFFFFFFFFFFFFFFFF
        if sh + nbits > 64:
            self.words[i + 1] |= value >> (64 - sh)

    def rice(self, x, g):
        q = x >> g
        while q >= 63:
            self.append((1 << 63) - 1, 63)
            q -= 63
        self.append((1 << q) - 1, q + 1)
        if g:
            self.append(x & ((1 << g) - 1), g)


def orient(edges, n):
    adj = [[] for _ in range(n)]
    deg = [0] * n
    for k, (u, v) in enumerate(edges):
        adj[u].append(k)
        adj[v].append(k)
        deg[u] += 1
        deg[v] += 1
    choice = [0] * n
    alive = [True] * n
    stack = [u for u in range(n) if deg[u] == 1]
    while stack:
        u = stack.pop()
        if deg[u] != 1:
            continue
        k = next(k for k in adj[u] if alive[k])
        eu, ev = edges[k]
        choice[k] = 0 if eu == u else 1
        alive[k] = False
        deg[eu] -= 1
        deg[ev] -= 1
        other = ev if eu == u else eu
        if deg[other] == 1:
            stack.append(other)
    for k0 in range(n):
        if not alive[k0]:
            continue
        u0, node = edges[k0]
        alive[k0] = False
        while node != u0:
            k = next(k for k in adj[node] if alive[k])
            eu, ev = edges[k]
            choice[k] = 0 if eu == node else 1
            alive[k] = False
            node = ev if eu == node else eu
    return choice


def build_bucket(args):
    """One bucket of recsplit._build_hashed (recsplit.py:499-520, 553-594)."""
    shi, slo, n, ck_rot = args
    K = ref_kernels()
    shi = shi.copy()
    slo = slo.copy()
    w = BitWriter()
    leaf_g = [leaf_rice_param(m) for m in range(n + 1)]
    choice = np.zeros(len(shi), dtype=np.uint8)
    stack = [(0, len(shi))]
    while stack:
        s0, s1 = stack.pop()
        m = s1 - s0
        node = plan(m, n)
        if node[0] == "leaf":
            khi = [int(x) for x in shi[s0:s1]]
            klo = [int(x) for x in slo[s0:s1]]
            q = K.search_rotate(khi, klo, m, ck_rot if m > 32 else 0, MAX_SEED)[0]
            w.rice(q, leaf_g[m])
            base, r = divmod(q, m)
            edges = []
            for a, b in zip(khi, klo):
                if K.split_bit(a, b, base) == 0:
                    edges.append(K.leaf_pair(a, b, base, m))
                else:
                    h0, h1 = K.leaf_pair(a, b, base, m)
                    edges.append(((h0 + r) % m, (h1 + r) % m))
            ori = orient(edges, m)
            choice[s0:s1] = ori
        else:
            sizes = node[1]
            seed, _ = K.split_seed_search(shi[s0:s1], slo[s0:s1], list(sizes), MAX_SEED)
            w.rice(seed, split_rice_param(m, tuple(sizes)))
            parts = K.split_parts(shi[s0:s1], slo[s0:s1], seed, list(sizes))
            order = np.argsort(parts, kind="stable")
            shi[s0:s1] = shi[s0:s1][order]
            slo[s0:s1] = slo[s0:s1][order]
            bounds = [s0]
            for sz in sizes:
                bounds.append(bounds[-1] + sz)
            for i in range(len(sizes) - 1, -1, -1):
                stack.append((bounds[i], bounds[i + 1]))
    return w.bit_len, shi, slo, choice, w.words


def master_hash_many(keys, salt=0):  # keys.py:46-58
    salt_b = struct.pack("<QQ", salt, 0)
    out = np.empty((len(keys), 2), dtype=np.uint64)
    for i, k in enumerate(keys):
        out[i] = struct.unpack("<QQ", hashlib.blake2b(k, digest_size=16, salt=salt_b).digest())
    return out[:, 0].copy(), out[:, 1].copy()


def _hash_chunk(keys):
    return master_hash_many(keys)


def build_sample_ref(keys, b, n, pool):
    """The reference build (bytes -> MPHF parts) with a process pool over
    buckets; returns stream bits + ribbon seed."""
    K = ref_kernels()
    N = len(keys)
    nproc = pool._processes
    chunks = [keys[i::nproc] for i in range(nproc)]  # hashing is per key; order restored below
    parts = pool.map(_hash_chunk, chunks)
    hi = np.empty(N, dtype=np.uint64)
    lo = np.empty(N, dtype=np.uint64)
    for i, (h, l) in enumerate(parts):
        hi[i::nproc] = h
        lo[i::nproc] = l
    nb = (N + b - 1) // b
    bucket = K.hash_range_batch(K.remix_batch(hi, lo, 0, 4), nb).astype(np.int64)
    order = np.lexsort((lo, hi, bucket))
    shi, slo = hi[order], lo[order]
    kp = np.zeros(nb + 1, dtype=np.int64)
    kp[1:] = np.cumsum(np.bincount(bucket, minlength=nb))
    tasks = [(shi[kp[i] : kp[i + 1]], slo[kp[i] : kp[i + 1]], n, 0) for i in range(nb) if kp[i + 1] > kp[i]]
    res = pool.map(build_bucket, tasks, chunksize=1)
    bits = sum(r[0] for r in res)
    shi = np.concatenate([r[1] for r in res])
    slo = np.concatenate([r[2] for r in res])
    choice = np.concatenate([r[3] for r in res])
    m = max(128, int(np.ceil(1.05 * N)))
    for seed in range(64):
        st, p0, p1 = K.ribbon_rows(shi, slo, seed, m)
        if K.ribbon_solve(st, p0, p1, choice, m) is not None:
            return bits, seed
    raise RuntimeError("ribbon unsolvable")


def build_descriptor_ref(keys, b, n, pool, eps=0.05, cache_k=8):
    """The whole reference build (rotate mode, salt 0) -> serialized
    descriptor bytes (format of recsplit.py:295-308).  Same orchestration as
    build_sample_ref; pinned to the stock reference's build() by
    tests/test_oracle.py::test_refbuild_matches_stock_reference."""
    K = ref_kernels()
    N = len(keys)
    hi, lo = master_hash_many(keys)
    nb = (N + b - 1) // b
    bucket = K.hash_range_batch(K.remix_batch(hi, lo, 0, 4), nb).astype(np.int64)
    order = np.lexsort((lo, hi, bucket))
    shi, slo = hi[order], lo[order]
    kp = np.zeros(nb + 1, dtype=np.int64)
    kp[1:] = np.cumsum(np.bincount(bucket, minlength=nb))
    tasks = [(shi[kp[i] : kp[i + 1]], slo[kp[i] : kp[i + 1]], n, 0) for i in range(nb) if kp[i + 1] > kp[i]]
    res = iter(pool.map(build_bucket, tasks, chunksize=1))
    bit_offsets = np.zeros(nb + 1, dtype=np.int64)
    stream = 0  # the concatenated stream as one big integer, LSB first
    total = 0
    parts = []
    for i in range(nb):
        bit_offsets[i] = total
        if kp[i + 1] > kp[i]:
            bl, bhi, blo, ch, words = next(res)
            for k, wd in enumerate(words):
                stream |= int(wd) << (total + 64 * k)
            stream &= (1 << (total + bl)) - 1
            total += bl
            parts.append((bhi, blo, ch))
    bit_offsets[nb] = total
    nw = (total + 63) // 64
    words = np.array([(stream >> (64 * k)) & ((1 << 64) - 1) for k in range(nw)], dtype=np.uint64)
    shi = np.concatenate([p[0] for p in parts])
    slo = np.concatenate([p[1] for p in parts])
    choice = np.concatenate([p[2] for p in parts])
    m = max(128, int(np.ceil((1.0 + eps) * N)))
    for seed in range(64):
        st, p0, p1 = K.ribbon_rows(shi, slo, seed, m)
        rw = K.ribbon_solve(st, p0, p1, choice, m)
        if rw is not None:
            break
    else:
        raise RuntimeError("ribbon unsolvable")
    leaf_g = [leaf_rice_param(x) for x in range(n + 1)]
    width = 32 if N < 2**32 and total < 2**32 else 64
    out = bytearray(b"SHKH")
    out += struct.pack("<HBQIBBBBQ", 1, 1, N, b, n, 1, cache_k, width, 0)
    out += struct.pack("<B", n) + bytes(leaf_g[1:])
    fmt = "<II" if width == 32 else "<QQ"
    for i in range(nb + 1):
        out += struct.pack(fmt, int(kp[i]), int(bit_offsets[i]))
    out += struct.pack("<Q", total) + words.astype("<u8").tobytes()
    out += struct.pack("<IQQ", int(round(eps * 65536)), seed, m) + np.asarray(rw, dtype="<u8").tobytes()
    return bytes(out)


def time_build_sample(seconds_target=15.0, steps=1, warmup=0):
    """keys/s of the reference build on a prefix sample of the C4 key set."""
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_2308_09561_b200 import workloads as W  # input recipe only

    cores = os.cpu_count() or 1
    k = W.raw_keys(4, C4["N"])
    if have_ref():
        kind = "reference"
        ctx = mp.get_context("fork")
        with ctx.Pool(cores) as pool:
            # calibrate: ~0.17 s per 2000-key bucket per core in this image
            per_key = 0.17 / 2000 / cores
            Ns = int(min(C4["N"], max(20 * C4["b"], seconds_target / per_key)))
            Ns -= Ns % C4["b"]
            keys = W.keys_as_bytes(k[:Ns])
            for _ in range(warmup):
                build_sample_ref(keys, C4["b"], C4["n"], pool)
            ts = []
            for _ in range(max(1, steps)):
                t = time.perf_counter()
                build_sample_ref(keys, C4["b"], C4["n"], pool)
                ts.append(time.perf_counter() - t)
        sample = (f"first {Ns:,} of the C4 keys (b=2000, n=40, rotate): master hash + bucket sort + "
                  f"{Ns // C4['b']} buckets (reference _core kernels, restated recsplit loop, {cores} processes) "
                  f"+ sequential ribbon")
    else:
        kind = "port"
        sys.path.insert(0, os.path.dirname(HERE))
        import oracle
        import oracle.host as H

        Ns = int(min(C4["N"], 2_000_000))
        keys = W.keys_as_bytes(k[:Ns])
        ts = []
        for _ in range(max(1, steps)):
            t = time.perf_counter()
            hi, lo = master_hash_many(keys)
            H.build_descriptor(hi, lo, C4["b"], C4["n"])
            ts.append(time.perf_counter() - t)
        sample = f"first {Ns:,} C4 keys, C oracle port (OpenMP over buckets, {cores} threads)"
    sec = float(np.mean(ts))
    return {"value": round(Ns / sec, 1), "unit": "keys/s", "cores": cores, "kind": kind, "sample": sample,
            "ms_per_step": round(sec * 1e3, 1), "sample_keys": Ns}


if __name__ == "__main__":
    print(time_build_sample(float(sys.argv[1]) if len(sys.argv) > 1 else 10.0))


def time_build_c2(steps=2):
    """keys/s of the reference build of all of C2 (N=1e5, b=500, n=24,
    rotate) with the pool over buckets (same orchestration as above)."""
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_2308_09561_b200 import workloads as W  # input recipe only

    if not have_ref():
        return {"error": "oracle/_ref (the reference's compiled kernels) is missing"}
    cores = os.cpu_count() or 1
    keys = W.keys_as_bytes(W.build_keys(2))
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        build_sample_ref(keys, 500, 24, pool)
        ts = []
        for _ in range(steps):
            t = time.perf_counter()
            build_sample_ref(keys, 500, 24, pool)
            ts.append(time.perf_counter() - t)
    sec = float(np.mean(ts))
    return {"value": round(len(keys) / sec, 1), "unit": "keys/s", "cores": cores, "kind": "reference",
            "sample": f"all of C2: master hash + bucket sort + 200 buckets (reference _core kernels, restated "
                      f"recsplit loop, {cores} processes) + sequential ribbon", "ms_per_step": round(sec * 1e3, 1)}
