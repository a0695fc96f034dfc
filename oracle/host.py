"""Oracle host side — TEST INFRASTRUCTURE.  Restates the reference's plan
shapes, Rice parameters and descriptor byte format
(/root/reference/pkg/src/shockhash/recsplit.py:45-119, :173-199, :295-308;
retrieval.py:29-31, :61-64) so the oracle can assemble complete descriptors
and evaluate queries independently of the product package."""

import math
import struct
from functools import lru_cache

import numpy as np

from . import lib, p, _u64, _i64

LOG2_E_HALF = math.log2(math.e / 2.0)
LOG2_E = math.log2(math.e)
HALF_LOG2_PI = 0.5 * math.log2(math.pi)


def plan(m, n):  # recsplit.py:45-67
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
    left = min(max(left, 1), m - 1)
    return ("split", (left, m - left))


def _parts(m, part):
    q, r = divmod(m, part)
    return tuple([part] * q + ([r] if r else []))


@lru_cache(maxsize=None)
def plan_nodes(m, n):  # recsplit.py:75-92
    node = plan(m, n)
    if node[0] == "leaf":
        return (("leaf", m, (), 1),)
    subs = [plan_nodes(s, n) for s in node[1]]
    return (("split", m, node[1], 1 + sum(s[0][3] for s in subs)),) + tuple(x for s in subs for x in s)


def leaf_rice_param(m):  # recsplit.py:173-184
    if m <= 1:
        return 0
    return max(0, int(m * LOG2_E_HALF + LOG2_E - HALF_LOG2_PI - 0.5 * math.log2(m)))


@lru_cache(maxsize=None)
def split_rice_param(m, sizes):  # recsplit.py:187-199
    logp = math.lgamma(m + 1)
    for s in sizes:
        logp -= math.lgamma(s + 1)
        logp += s * (math.log(s) - math.log(m))
    return max(0, int(-logp / math.log(2.0)))


def flatten_plan(m, n, leaf_g):  # recsplit.py:95-119
    nodes = plan_nodes(m, n)
    c = len(nodes)
    kind, g, fan, soff, sub, mn = (np.zeros(c, dtype=np.int64) for _ in range(6))
    flat = []
    for i, (k, mm, sizes, st) in enumerate(nodes):
        mn[i] = mm
        sub[i] = st
        if k == "leaf":
            kind[i] = 1
            g[i] = leaf_g[mm]
        else:
            g[i] = split_rice_param(mm, sizes)
            fan[i] = len(sizes)
            soff[i] = len(flat)
            flat.extend(sizes)
    return kind, g, fan, soff, np.asarray(flat or [0], dtype=np.int64), sub, mn


def tables(n, max_m):
    leaf_g = [0] + [leaf_rice_param(m) for m in range(1, n + 1)]
    split_g = [0] * (max_m + 1)
    for m in range(n + 1, max_m + 1):
        split_g[m] = split_rice_param(m, plan(m, n)[1])
    return leaf_g, split_g


def columns(N, eps):  # retrieval.py:29-31
    return max(128, int(np.ceil((1.0 + eps) * N)))


def _mix64_np(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def bucket_sizes(hi, lo, nb):
    """recsplit.py:475-483: bucket = hash_range(remix(hi, lo, 0, TAG_BUCKET), nb)."""
    from . import seed_mixer

    x = np.uint64(seed_mixer(0, 4))
    v = _mix64_np(_mix64_np(_u64(hi) ^ x) ^ _u64(lo))
    bk = ((v >> np.uint64(32)) * np.uint64(nb)) >> np.uint64(32)
    return np.bincount(bk.astype(np.int64), minlength=nb)


def build_descriptor(hi, lo, b, n, mode=1, cache_k=8, eps=0.05, salt=0):
    """Whole reference construction on the CPU oracle -> (bytes, parts)."""
    from . import build_hashed, ribbon_rows, ribbon_solve

    N = len(hi)
    nb = (N + b - 1) // b
    mx = int(max(n, bucket_sizes(hi, lo, nb).max()))
    leaf_g, split_g = tables(n, mx)
    res = build_hashed(hi, lo, b, n, 0 if mode == 0 else 1, cache_k if mode == 2 else 0, leaf_g, split_g)
    m = columns(N, eps)
    rseed = None
    for seed in range(64):
        st, p0, p1 = ribbon_rows(res["shi"], res["slo"], seed, m)
        w = ribbon_solve(st, p0, p1, res["choice"], m)
        if w is not None:
            rseed = seed
            break
    if rseed is None:
        raise RuntimeError("ribbon unsolvable")
    width = 32 if N < 2**32 and res["bit_len"] < 2**32 else 64
    out = bytearray(b"SHKH")
    out += struct.pack("<HBQIBBBBQ", 1, 1, N, b, n, mode, cache_k, width, salt)
    out += struct.pack("<B", n) + bytes(leaf_g[1:])
    fmt = "<II" if width == 32 else "<QQ"
    for i in range(nb + 1):
        out += struct.pack(fmt, int(res["key_prefix"][i]), int(res["bit_offsets"][i]))
    out += struct.pack("<Q", res["bit_len"]) + res["words"].astype("<u8").tobytes()
    out += struct.pack("<IQQ", int(round(eps * 65536)), rseed, m) + w.astype("<u8").tobytes()
    res.update(ribbon_seed=rseed, ribbon_m=m, ribbon_words=w, leaf_g=leaf_g, nb=nb)
    return bytes(out), res


def query(res, n, mode, cache_k, hi, lo):
    """Reference-style query_stream on the oracle build result."""
    kp = _u64(res["key_prefix"])
    sizes = sorted(set(int(x) for x in np.diff(kp.astype(np.int64)) if x > 0))
    plans = {m: flatten_plan(m, n, res["leaf_g"]) for m in sizes}
    pid = {m: i for i, m in enumerate(sizes)}
    poff, sbase = [0], []
    cols = {k: [] for k in ("kind", "g", "soff", "sub", "mn")}
    flats = []
    base = 0
    for m in sizes:
        kind, g, fan, soff, flat, sub, mn = plans[m]
        for k2, arr in zip(("kind", "g", "soff", "sub", "mn"), (kind, g, soff, sub, mn)):
            cols[k2].append(arr)
        poff.append(poff[-1] + len(kind))
        sbase.append(base)
        flats.append(flat)
        base += len(flat)
    cat = lambda xs: _i64(np.concatenate(xs)) if xs else np.zeros(1, dtype=np.int64)
    bp = _i64([pid.get(int(x), -1) for x in np.diff(kp.astype(np.int64))])
    hi, lo = _u64(hi), _u64(lo)
    out = np.zeros(len(hi), dtype=np.uint64)
    rw = _u64(res["ribbon_words"])
    sw = _u64(res["words"]) if len(res["words"]) else np.zeros(1, dtype=np.uint64)
    arrs = [_i64(poff), _i64(sbase or [0]), cat(cols["kind"]), cat(cols["g"]), cat(cols["soff"]), cat(cols["sub"]),
            cat(cols["mn"]), cat(flats)]
    ck = cache_k if mode == 2 else 0
    rc = lib().o_query(p(hi), p(lo), len(hi), res["nb"], p(kp), p(_u64(res["bit_offsets"])), p(sw), res["bit_len"],
                       p(bp), *[p(a) for a in arrs], int(mode), int(ck), int(res["ribbon_seed"]), int(res["ribbon_m"]),
                       p(rw), len(rw), p(out))
    if rc:
        raise ValueError("bit stream overrun")
    return np.minimum(out, np.uint64(max(len(res["shi"]) - 1, 0)))
