"""Full-population leaf goldens for C3 and C5 from the REAL reference.

Every leaf of the config is solved by the reference's compiled
``search_plain`` (``/root/reference/pkg/src/shockhash/_kernels/_core.pyx:186-229``)
and oriented by its ``pseudoforest.orient``
(``/root/reference/pkg/src/shockhash/pseudoforest.py:149-201``), fanned out
over all host cores with a process pool.  Runs only in the build container
(see make_golden.py for how ``shockhash_ref`` is built out of tree):

    PYTHONPATH=/tmp/refpkg python tests/golden/make_leaf_full.py c3 c5

Output ``tests/golden/c{cfg}_full.bin``: three little-endian blocks of L
entries each, back to back --
    seeds  <i8[L]   (the reference's minimum seed; -1 never occurs here)
    fbits  <u8[L]   (bit i = f(key i), orient() in leaf key order)
    passes <u8[L]   (the reference's filter-pass counter, tuple field 2)
and ``c{cfg}_full.json`` with L, n, sha256 of the file and of the seed||fbits
blocks, sum of seeds, and the reference core-seconds it took.
"""

import hashlib
import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_2308_09561_b200 import workloads as W  # noqa: E402

_HI = _LO = _N = None


def _init(cfg):
    global _HI, _LO, _N
    _HI, _LO = W.leaf_inputs(cfg)
    _N = W.LEAF_CONFIGS[cfg]["n"]


def _solve(i):
    import shockhash_ref as ref
    from shockhash_ref import pseudoforest
    from shockhash_ref import shockhash as ref_sh
    from shockhash_ref._kernels import get_backend

    K = get_backend("compiled")
    hi = [int(x) for x in _HI[i]]
    lo = [int(x) for x in _LO[i]]
    t0 = time.process_time()
    t = K.search_plain(hi, lo, _N, ref_sh.MAX_SEED)
    dt = time.process_time() - t0
    s = int(t[0])
    hk = [ref.HashedKey(a, b) for a, b in zip(hi, lo)]
    ori = pseudoforest.orient(ref_sh._edges_plain(hk, s, _N), _N)
    fb = sum(int(b) << k for k, b in enumerate(ori))
    return i, s, fb, int(t[2]), dt


def run(cfg, procs):
    L = W.LEAF_CONFIGS[cfg]["leaves"]
    n = W.LEAF_CONFIGS[cfg]["n"]
    seeds = np.full(L, -2, dtype="<i8")
    fbits = np.zeros(L, dtype="<u8")
    passes = np.zeros(L, dtype="<u8")
    cpu = 0.0
    t0 = time.time()
    done = 0
    with Pool(procs, initializer=_init, initargs=(cfg,)) as pool:
        for i, s, fb, ps, dt in pool.imap_unordered(_solve, range(L), chunksize=16 if cfg == 3 else 1):
            seeds[i], fbits[i], passes[i] = s, fb, ps
            cpu += dt
            done += 1
            if done % max(1, L // 50) == 0:
                print(f"c{cfg}: {done}/{L} leaves, {time.time() - t0:.0f} s", file=sys.stderr, flush=True)
    assert (seeds >= 0).all()
    blob = seeds.tobytes() + fbits.tobytes() + passes.tobytes()
    path = os.path.join(HERE, f"c{cfg}_full.bin")
    with open(path, "wb") as f:
        f.write(blob)
    meta = dict(cfg=cfg, leaves=L, n=n, layout="seeds<i8[L] | fbits<u8[L] | passes<u8[L]",
                file_sha256=hashlib.sha256(blob).hexdigest(),
                sha16=hashlib.sha256(seeds.tobytes() + fbits.tobytes()).hexdigest()[:16],
                sum_seed=int(seeds.sum()), seeds_tested=int((seeds + 1).sum()),
                mean_seeds_per_leaf=float((seeds + 1).mean()), max_seed=int(seeds.max()),
                ref_search_core_seconds=round(cpu, 1), wall_seconds=round(time.time() - t0, 1), procs=procs,
                generator="tests/golden/make_leaf_full.py (reference compiled search_plain + pseudoforest.orient)")
    with open(os.path.join(HERE, f"c{cfg}_full.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", path, meta, file=sys.stderr)


if __name__ == "__main__":
    procs = int(os.environ.get("PROCS", os.cpu_count()))
    for p in sys.argv[1:]:
        run(int(p.lstrip("c")), procs)
