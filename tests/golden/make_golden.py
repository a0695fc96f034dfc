"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Runs only in the build container, where /root/reference exists.  The
reference package is built out of tree (never copied into this repo):

    cp -r /root/reference/pkg /tmp/refbuild
    (cd /tmp/refbuild && python setup.py build_ext --inplace)
    mkdir -p /tmp/refpkg && cp -r /tmp/refbuild/src/shockhash /tmp/refpkg/shockhash_ref

and imported as ``shockhash_ref`` with its compiled (Cython) backend active.
Usage:  PYTHONPATH=/tmp/refpkg python tests/golden/make_golden.py <part>...
Parts: kat leaves split ribbon rice c1 c2 c3 c5 c4  (c4 takes ~20 min).
Every fixture is small; large outputs are pinned by sha256.
"""

import hashlib
import json
import os
import struct
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import shockhash_ref as ref  # noqa: E402
from shockhash_ref._kernels import get_backend  # noqa: E402
from shockhash_ref import recsplit as ref_recsplit  # noqa: E402
from shockhash_ref import shockhash as ref_sh  # noqa: E402
from shockhash_ref.keys import synthetic_hashed  # noqa: E402

from paper_2308_09561_b200 import workloads as W  # noqa: E402

K = get_backend("compiled")
assert ref.BACKEND_NAME == "compiled"


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, indent=1, sort_keys=True)
    print("wrote", name, file=sys.stderr)


def u64s(a):
    return [int(x) for x in np.asarray(a, dtype=np.uint64)]


def orient_bits(edges, n):
    from shockhash_ref import pseudoforest

    ori = pseudoforest.orient(edges, n)
    return sum(int(b) << i for i, b in enumerate(ori))


def leaf_record(hi, lo, n, mode, ck=0):
    """Seed, 5-tuple stats and f bits exactly as the reference computes them."""
    hi = [int(x) for x in hi]
    lo = [int(x) for x in lo]
    if mode == 0:
        t = K.search_plain(hi, lo, n, ref_sh.MAX_SEED)
    else:
        t = K.search_rotate(hi, lo, n, ck, ref_sh.MAX_SEED)
    q = int(t[0])
    hk = [ref.HashedKey(a, b) for a, b in zip(hi, lo)]
    edges = ref_sh._edges_plain(hk, q, n) if mode == 0 else ref_sh._edges_rotate(hk, q, n, ck)
    return dict(seed=q, stats=[int(x) for x in t], fbits=orient_bits(edges, n))


def part_kat():
    out = {}
    rng = np.random.default_rng(1)
    rows = []
    for _ in range(200):
        hi, lo, s = (int(x) for x in rng.integers(0, 2**63, 3))
        n = int(rng.integers(1, 65))
        tag = int(rng.integers(1, 8))
        rows.append(dict(hi=hi, lo=lo, s=s, n=n, tag=tag, mix64=K.mix64(hi), seed_mixer=K.seed_mixer(s, tag),
                         remix=K.remix(hi, lo, s, tag), hash_range=K.hash_range(hi, n),
                         leaf_pair=list(K.leaf_pair(hi, lo, s, n)), split_bit=int(K.split_bit(hi, lo, s))))
    out["scalars"] = rows
    cells = []
    for _ in range(300):
        hi, lo = (int(x) for x in rng.integers(0, 2**63, 2))
        n = int(rng.integers(1, 65))
        q = int(rng.integers(0, 10000))
        mode = int(rng.integers(0, 3))
        ck = 8 if mode == 2 else 0
        choice = int(rng.integers(0, 2))
        cells.append(dict(hi=hi, lo=lo, q=q, n=n, mode=mode, ck=ck, choice=choice,
                          cell=int(K.leaf_cell(hi, lo, q, n, mode, ck, choice))))
    out["leaf_cell"] = cells
    # blake2b-128 master hash (keys.py:39-43) for several lengths and salts
    bl = []
    r2 = np.random.default_rng(7)
    for ln in [0, 1, 3, 7, 8, 9, 15, 16, 17, 31, 32, 63, 64, 65, 127, 128, 129, 200, 256, 300]:
        for salt in (0, 1, 7, 2**63 + 5):
            key = bytes(r2.integers(0, 256, ln, dtype=np.uint8))
            h = ref.master_hash(key, salt)
            bl.append(dict(key=key.hex(), salt=salt, hi=int(h.hi), lo=int(h.lo)))
    out["blake2b"] = bl
    out["mix64_kat"] = [[int((k * 0x9E3779B97F4A7C15) & (2**64 - 1)), K.mix64((k * 0x9E3779B97F4A7C15) & (2**64 - 1))] for k in (1, 2, 3)]
    dump("kat.json", out)


def part_leaves():
    """Leaf searches (plain, rotate ck=0/8) on reference-style synthetic leaves."""
    recs = []
    for n in [1, 2, 3, 5, 8, 10, 12, 16, 20, 24, 31, 32, 33, 40]:
        reps = 12 if n <= 24 else 4
        for rep in range(reps):
            gen = 313 + 100 * n + rep
            hi, lo = synthetic_hashed(n, gen)
            r = dict(n=n, gen=gen, hi=u64s(hi), lo=u64s(lo))
            r["plain"] = leaf_record(hi, lo, n, 0)
            r["rotate"] = leaf_record(hi, lo, n, 1, 0)
            ck = 8 if n > ref_sh.CACHE_MIN_LEAF else 0
            r["rotate_cached"] = leaf_record(hi, lo, n, 2, ck)
            r["rotate_cached"]["ck"] = ck
            recs.append(r)
    dump("leaves.json", recs)


def part_split():
    rng = np.random.default_rng(3)
    recs = []
    for rep in range(60):
        n = int(rng.integers(8, 64))
        m = int(rng.integers(n + 1, 15 * n))
        node = ref_recsplit.plan(m, n)
        if node[0] != "split":
            continue
        sizes = list(node[1])
        hi, lo = synthetic_hashed(m, 999 + rep)
        seed, evals = K.split_seed_search(hi, lo, sizes, 1 << 30)
        parts = K.split_parts(hi, lo, seed, sizes)
        recs.append(dict(m=m, n=n, gen=999 + rep, sizes=sizes, seed=int(seed), evals=int(evals),
                         parts_sha=sha(np.asarray(parts, dtype="<i8").tobytes()),
                         g=int(ref_recsplit.split_rice_param(m, tuple(sizes)))))
    # plan shapes and Rice parameters for every bucket size that C2/C4 can produce
    plans = {}
    for n in (8, 16, 20, 24, 30, 40, 56, 64):
        for m in list(range(0, 200)) + list(range(400, 2600, 37)):
            plans[f"{m},{n}"] = [list(x) for x in ref_recsplit.flatten_plan(m, n, np.arange(65))] if m > 0 else None
    leaf_g = [int(ref_recsplit.leaf_rice_param(m)) for m in range(0, 65)]
    dump("split.json", dict(cases=recs, leaf_g=leaf_g, plans_sha=sha(json.dumps(plans, sort_keys=True, default=int).encode())))


def part_ribbon():
    recs = []
    for N in [0, 1, 50, 3000, 20000]:
        rng = np.random.default_rng(N)
        hi, lo = synthetic_hashed(N, 5150 + N)
        rhs = rng.integers(0, 2, N).astype(np.uint8)
        m = max(128, int(np.ceil(1.05 * N)))
        for seed in (0, 3):
            st, p0, p1 = K.ribbon_rows(hi, lo, seed, m)
            w = K.ribbon_solve(st, p0, p1, rhs, m)
            recs.append(dict(N=N, seed=seed, m=m, gen=5150 + N,
                             rows_sha=sha(np.asarray(st, "<i8").tobytes() + np.asarray(p0, "<u8").tobytes() + np.asarray(p1, "<u8").tobytes()),
                             solvable=w is not None,
                             words=u64s(w) if (w is not None and N <= 3000) else None,
                             words_sha=sha(np.asarray(w, "<u8").tobytes()) if w is not None else None))
    # the retrieval_build_arrays seed loop on an overloaded system (forces retries / failure)
    dump("ribbon.json", recs)


def part_rice():
    from shockhash_ref.recsplit import BitWriter

    rng = np.random.default_rng(4)
    items = [(int(rng.integers(0, 5000)), int(rng.integers(0, 12))) for _ in range(300)]
    items += [(200, 0), (1000, 1), (64, 0), (63, 0), (127, 0)]
    w = BitWriter()
    for v, g in items:
        w.rice(v, g)
    dump("rice.json", dict(items=items, bit_len=w.bit_len, words=u64s(w.to_array())))


def part_leafcfg(cfg, sample):
    hi, lo = W.leaf_inputs(cfg, sample)
    n = W.LEAF_CONFIGS[cfg]["n"]
    t0 = time.time()
    seeds, fb, stats = [], [], []
    for i in range(len(hi)):
        r = leaf_record(hi[i], lo[i], n, 0)
        seeds.append(r["seed"])
        fb.append(r["fbits"])
        stats.append(r["stats"][1:4])
    dt = time.time() - t0
    seeds_a = np.asarray(seeds, dtype="<i8")
    fb_a = np.asarray(fb, dtype="<u8")
    dump(f"c{cfg}.json", dict(cfg=cfg, leaves=len(hi), n=n, seeds=seeds, fbits=[int(x) for x in fb],
                              stats=stats, sum_seed=int(seeds_a.sum()),
                              sha16=sha(seeds_a.tobytes() + fb_a.tobytes())[:16], ref_seconds=dt,
                              hi0=u64s(hi[0]), lo0=u64s(lo[0])))


def part_build(cfg):
    spec = W.BUILD_CONFIGS[cfg]
    t0 = time.time()
    k = W.build_keys(cfg)
    keys = W.keys_as_bytes(k)
    t1 = time.time()
    desc = ref.build(keys, spec["b"], spec["n"])
    t2 = time.time()
    blob = desc.serialize()
    hi, lo = ref.keys.master_hash_many(keys, desc.salt)
    idx = W.query_indices(cfg)
    t3 = time.time()
    out = desc.query_hashed_many(hi[idx], lo[idx])
    t4 = time.time()
    own = desc.query_hashed_many(hi, lo)
    ok = bool((np.bincount(own.astype(np.int64), minlength=spec["N"]) == 1).all())
    st = desc.stats()
    rec = dict(cfg=cfg, N=spec["N"], b=spec["b"], n=spec["n"], salt=int(desc.salt), desc_bytes=len(blob),
               desc_sha=sha(blob), bits_per_key=st["bits_per_key"], ribbon_seed=int(desc.ribbon.seed),
               ribbon_m=int(desc.ribbon.m), stream_bit_len=int(desc.stream_bit_len),
               query_sha=sha(np.asarray(out, "<u8").tobytes()), queries=len(idx),
               query_head=u64s(out[:64]), own_sha=sha(np.asarray(own, "<u8").tobytes()), bijective=ok,
               build_stats={k2: v for k2, v in st.items() if isinstance(v, (int, float))},
               ref_build_seconds=t2 - t1, ref_query_seconds=t4 - t3)
    if len(blob) < 100_000:
        with open(os.path.join(HERE, f"c{cfg}_desc.bin"), "wb") as f:
            f.write(blob)
    dump(f"c{cfg}.json", rec)


def part_small_builds():
    """Reference descriptors for small builds in all modes (drop-in API parity)."""
    recs = []
    for (N, b, n, mode, gen) in [(1, 100, 16, 1, 1), (3, 16, 8, 1, 3), (17, 16, 8, 0, 17), (3000, 300, 20, 0, 1),
                                 (3000, 300, 20, 1, 2), (3000, 300, 20, 2, 3), (5000, 500, 24, 1, 21),
                                 (4000, 400, 40, 2, 5), (6000, 2000, 30, 1, 6), (2500, 1000, 56, 0, 7),
                                 (20000, 1000, 24, 1, 11)]:
        keys = ref.synthetic_keys(N, gen)
        desc = ref.build(keys, b, n, mode)
        blob = desc.serialize()
        q = desc.query_many(keys)
        recs.append(dict(N=N, b=b, n=n, mode=mode, gen=gen, desc_sha=sha(blob), desc_len=len(blob),
                         query_sha=sha(np.asarray(q, "<u8").tobytes()),
                         desc_hex=blob.hex() if len(blob) < 4000 else None))
    hi, lo = synthetic_hashed(4000, 0xABC)
    desc = ref_recsplit.build_hashed(hi, lo, 400, 24, 1)
    recs.append(dict(hashed=True, N=4000, b=400, n=24, mode=1, gen=0xABC, desc_sha=sha(desc.serialize()),
                     query_sha=sha(np.asarray(desc.query_hashed_many(hi, lo), "<u8").tobytes())))
    dump("builds.json", recs)


def part_experiments():
    """The analysis entry points of the kernel seam: search_bruteforce,
    enumerate_outcomes, mc_filter_pass_count (_core.pyx:337-371, 778-860)."""
    brute = []
    for n in [1, 2, 3, 5, 8, 10, 12, 14, 16]:
        for rep in range(4 if n <= 12 else 2):
            gen = 313 + 100 * n + rep
            hi, lo = synthetic_hashed(n, gen)
            s, ev = K.search_bruteforce(hi, lo, n, 1 << 30)
            brute.append(dict(n=n, gen=gen, max_seed=1 << 30, seed=int(s), evals=int(ev)))
    for n, ms in [(10, 50), (16, 1000), (12, 0)]:
        hi, lo = synthetic_hashed(n, 77)
        s, ev = K.search_bruteforce(hi, lo, n, ms)
        brute.append(dict(n=n, gen=77, max_seed=ms, seed=int(s), evals=int(ev)))
    enum = []
    for n in range(1, 7):
        pf, s2 = K.enumerate_outcomes(n)
        enum.append(dict(n=n, pf_count=int(pf), sum_2c=int(s2)))
    mc = []
    for n, trials, ent in [(1, 1000, 0), (2, 1000, 1), (12, 2000, 42), (16, 300000, 7), (24, 200000, 3),
                           (32, 300000, 5), (40, 100000, 2**64 - 3), (56, 50000, 11), (64, 50000, 13)]:
        mc.append(dict(n=n, trials=trials, entropy=ent, passes=int(K.mc_filter_pass_count(n, trials, ent))))
    from shockhash_ref import experiments as ex

    trials = []
    for ns, mode, reps, seed in [([4, 8], "plain", 300, 2), ([10], "rotate", 300, 2), ([12, 16], "plain", 200, 7),
                                 ([24], "rotate", 100, 1), ([36], "rotate-cached", 20, 3), ([6], "bruteforce", 50, 1)]:
        for r in ex.trial_statistics(ns, mode, reps, seed):
            trials.append(dict(n=r.n, mode=r.mode, reps=r.reps, seed=seed, mean_seed=r.mean_seed,
                               mean_log2_seed=r.mean_log2_seed, overhead_bits=r.overhead_bits))
    comp = [dict(n=n, trials=t, seed=s, value=ex.mc_component_factor(n, t, s)) for n, t, s in [(8, 2000, 5), (16, 500, 1)]]
    filt = [dict(n=n, trials=t, seed=s, value=ex.mc_filter_pass(n, t, s)) for n, t, s in [(16, 40000, 3), (32, 40000, 3)]]
    dump("experiments.json", dict(bruteforce=brute, enumerate=enum, mc_filter=mc, trial_statistics=trials,
                                  component=comp, filter_pass=filt))


if __name__ == "__main__":
    parts = sys.argv[1:] or ["kat", "leaves", "split", "ribbon", "rice", "c1", "c3", "c5", "c2", "builds"]
    for p in parts:
        t = time.time()
        if p == "kat":
            part_kat()
        elif p == "leaves":
            part_leaves()
        elif p == "split":
            part_split()
        elif p == "ribbon":
            part_ribbon()
        elif p == "rice":
            part_rice()
        elif p == "c1":
            part_leafcfg(1, None)
        elif p == "c3":
            part_leafcfg(3, 2000)
        elif p == "c5":
            part_leafcfg(5, int(os.environ.get("C5_SAMPLE", "24")))
        elif p == "c2":
            part_build(2)
        elif p == "c4":
            part_build(4)
        elif p == "experiments":
            part_experiments()
        elif p == "builds":
            part_small_builds()
        print(p, "done in", round(time.time() - t, 1), "s", file=sys.stderr)
