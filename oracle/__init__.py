"""CPU oracle — TEST INFRASTRUCTURE, not product code.

``shk_oracle.c`` restates the reference's algorithm in plain C (each function
cites the reference file:line it follows); this module binds it with ctypes.
Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline leg may
use it, and only as the checker.  It is pinned against golden vectors
produced by the real reference (tests/golden/, tests/test_oracle.py).

``_ref/`` (built by build_ref.sh from /root/reference) holds the reference's
own compiled kernels for the reference CPU arm of bench.py.
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libshk_oracle.so")

_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64

_SIGS = {
    "o_mix64": (_U64, [_U64]),
    "o_seed_mixer": (_U64, [_U64, _U64]),
    "o_remix": (_U64, [_U64, _U64, _U64, _U64]),
    "o_hash_range": (_U64, [_U64, _U64]),
    "o_leaf_pair": (None, [_U64, _U64, _U64, _I, _P, _P]),
    "o_split_bit": (_I, [_U64, _U64, _U64]),
    "o_leaf_cell": (_I, [_U64, _U64, _I64, _I, _I, _I64, _I]),
    "o_search_plain": (None, [_P, _P, _I, _I64, _P]),
    "o_search_rotate": (None, [_P, _P, _I, _I64, _I64, _P]),
    "o_orient": (_U64, [_P, _P, _I, _P]),
    "o_split_search": (None, [_P, _P, _I64, _P, _I, _I64, _P, _P]),
    "o_split_parts": (None, [_P, _P, _I64, _U64, _P, _I, _P]),
    "o_ribbon_rows": (None, [_P, _P, _I64, _I64, _U64, _P, _P, _P]),
    "o_ribbon_solve": (_I, [_P, _P, _P, _P, _I64, _I64, _P]),
    "o_ribbon_query": (None, [_P, _P, _P, _I64, _P, _I64, _P]),
    "o_rice_decode": (_I, [_P, _I64, _P, _I, _P]),
    "o_build_hashed": (_I64, [_P, _P, _I64, _I64, _I, _I, _I, _P, _P, _I64, _P, _P, _P, _I64, _P, _P, _P, _P]),
    "o_search_plain_batch": (None, [_P, _P, _I64, _I, _P]),
    "o_search_bruteforce": (None, [_P, _P, _I, _I64, _P]),
    "o_mc_filter_pass_count": (_I64, [_I, _I64, _U64]),
    "o_enumerate_outcomes": (None, [_I, _P]),
    "o_query": (_I, [_P, _P, _I64, _I64, _P, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I64, _U64, _I64,
                     _P, _I64, _P]),
}

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        for k, (r, a) in _SIGS.items():
            f = getattr(L, k)
            f.restype = r
            f.argtypes = a
        _lib = L
    return _lib


def _u64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def p(a):
    return None if a is None else a.ctypes.data


MASK64 = (1 << 64) - 1


def mix64(z):
    return int(lib().o_mix64(int(z) & MASK64))


def seed_mixer(s, tag):
    return int(lib().o_seed_mixer(int(s) & MASK64, int(tag)))


def remix(hi, lo, s, tag):
    return int(lib().o_remix(int(hi) & MASK64, int(lo) & MASK64, int(s) & MASK64, int(tag)))


def hash_range(v, m):
    return int(lib().o_hash_range(int(v) & MASK64, int(m)))


def leaf_pair(hi, lo, s, n):
    a, b = ctypes.c_int(), ctypes.c_int()
    lib().o_leaf_pair(int(hi) & MASK64, int(lo) & MASK64, int(s) & MASK64, int(n), ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def split_bit(hi, lo, s):
    return int(lib().o_split_bit(int(hi) & MASK64, int(lo) & MASK64, int(s) & MASK64))


def leaf_cell(hi, lo, q, m, mode, ck, choice):
    return int(lib().o_leaf_cell(int(hi) & MASK64, int(lo) & MASK64, int(q), int(m), int(mode), int(ck), int(choice)))


def search_plain(hi, lo, n, max_seed):
    hi, lo = _u64(hi), _u64(lo)
    out = np.zeros(5, dtype=np.int64)
    lib().o_search_plain(p(hi), p(lo), int(n), int(max_seed), p(out))
    return tuple(int(x) for x in out)


def search_rotate(hi, lo, n, ck, max_seed):
    hi, lo = _u64(hi), _u64(lo)
    out = np.zeros(5, dtype=np.int64)
    lib().o_search_rotate(p(hi), p(lo), int(n), int(ck), int(max_seed), p(out))
    return tuple(int(x) for x in out)


def search_bruteforce(hi, lo, n, max_seed):
    hi, lo = _u64(hi), _u64(lo)
    out = np.zeros(2, dtype=np.int64)
    lib().o_search_bruteforce(p(hi), p(lo), int(n), int(max_seed), p(out))
    return int(out[0]), int(out[1])


def mc_filter_pass_count(n, trials, entropy):
    return int(lib().o_mc_filter_pass_count(int(n), int(trials), int(entropy) & MASK64))


def enumerate_outcomes(n):
    out = np.zeros(2, dtype=np.uint64)
    lib().o_enumerate_outcomes(int(n), p(out))
    return int(out[0]), int(out[1])


def orient(edges, n):
    eu = np.ascontiguousarray([e[0] for e in edges], dtype=np.int32)
    ev = np.ascontiguousarray([e[1] for e in edges], dtype=np.int32)
    ok = ctypes.c_int(0)
    f = int(lib().o_orient(p(eu), p(ev), int(n), ctypes.byref(ok)))
    return f if ok.value else None


def edges_plain(hi, lo, q, n):
    return [leaf_pair(a, b, q, n) for a, b in zip(hi, lo)]


def edges_rotate(hi, lo, q, n, ck):
    base, r = divmod(q, n)
    sa = base - base % ck if ck else base
    out = []
    for a, b in zip(hi, lo):
        if split_bit(a, b, sa) == 0:
            out.append(leaf_pair(a, b, sa, n))
        else:
            x, y = leaf_pair(a, b, base, n)
            out.append(((x + r) % n, (y + r) % n))
    return out


def split_seed_search(hi, lo, sizes, max_seed):
    hi, lo, sz = _u64(hi), _u64(lo), _i64(list(sizes))
    s, e = ctypes.c_int64(), ctypes.c_int64()
    lib().o_split_search(p(hi), p(lo), len(hi), p(sz), len(sz), int(max_seed), ctypes.byref(s), ctypes.byref(e))
    return int(s.value), int(e.value)


def split_parts(hi, lo, seed, sizes):
    hi, lo, sz = _u64(hi), _u64(lo), _i64(list(sizes))
    out = np.zeros(len(hi), dtype=np.int64)
    lib().o_split_parts(p(hi), p(lo), len(hi), int(seed) & MASK64, p(sz), len(sz), p(out))
    return out


def ribbon_rows(hi, lo, seed, m):
    hi, lo = _u64(hi), _u64(lo)
    N = len(hi)
    st = np.zeros(N, dtype=np.int64)
    p0 = np.zeros(N, dtype=np.uint64)
    p1 = np.zeros(N, dtype=np.uint64)
    lib().o_ribbon_rows(p(hi), p(lo), N, int(m), int(seed) & MASK64, p(st), p(p0), p(p1))
    return st, p0, p1


def ribbon_solve(st, p0, p1, rhs, m):
    st, p0, p1 = _i64(st), _u64(p0), _u64(p1)
    r = np.ascontiguousarray(rhs, dtype=np.uint8)
    w = np.zeros((int(m) + 63) // 64, dtype=np.uint64)
    ok = lib().o_ribbon_solve(p(st), p(p0), p(p1), p(r), len(st), int(m), p(w))
    return w if ok else None


def ribbon_query(st, p0, p1, words, m):
    st, p0, p1, w = _i64(st), _u64(p0), _u64(p1), _u64(words)
    out = np.zeros(len(st), dtype=np.uint8)
    lib().o_ribbon_query(p(st), p(p0), p(p1), len(st), p(w), len(w), p(out))
    return out


def rice_decode(words, bit_len, pos, g):
    w = _u64(words)
    ps = ctypes.c_int64(int(pos))
    v = ctypes.c_int64()
    if lib().o_rice_decode(p(w), int(bit_len), ctypes.byref(ps), int(g), ctypes.byref(v)):
        raise ValueError("bit stream overrun")
    return int(v.value), int(ps.value)


def build_hashed(hi, lo, b, n, mode, ck, leaf_g, split_g):
    """Reference build (without the ribbon) -> dict of arrays."""
    hi, lo = _u64(hi), _u64(lo)
    N = len(hi)
    nb = (N + b - 1) // b
    lg = np.ascontiguousarray(leaf_g, dtype=np.int32)
    sg = np.ascontiguousarray(split_g, dtype=np.int32)
    kp = np.zeros(nb + 1, dtype=np.uint64)
    bo = np.zeros(nb + 1, dtype=np.uint64)
    maxw = max(16, N // 8 + 1024)
    words = np.zeros(maxw, dtype=np.uint64)
    choice = np.zeros(N, dtype=np.uint8)
    shi = np.zeros(N, dtype=np.uint64)
    slo = np.zeros(N, dtype=np.uint64)
    st = np.zeros(5, dtype=np.int64)
    bits = lib().o_build_hashed(p(hi), p(lo), N, nb, int(n), int(mode), int(ck), p(lg), p(sg), len(sg) - 1, p(kp),
                                p(bo), p(words), maxw, p(choice), p(shi), p(slo), p(st))
    if bits < 0:
        raise RuntimeError(f"oracle build failed ({bits})")
    return dict(key_prefix=kp, bit_offsets=bo, words=words[: (bits + 63) // 64].copy(), bit_len=int(bits),
                choice=choice, shi=shi, slo=slo, stats=st)


def search_plain_batch(hi2d, lo2d):
    hi, lo = _u64(hi2d), _u64(lo2d)
    L, n = hi.shape
    out = np.zeros(L, dtype=np.int64)
    lib().o_search_plain_batch(p(hi), p(lo), L, n, p(out))
    return out
