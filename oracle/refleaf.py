"""Reference CPU baseline of the leaf-only configs C1/C3/C5 for bench.py —
TEST/BASELINE INFRASTRUCTURE.

Times the reference's OWN compiled ``search_plain`` (oracle/_ref/_core*.so,
the Cython module /root/reference/pkg/src/shockhash/_kernels/_core.pyx:186-229
compiled by oracle/build_ref.sh) per leaf, as BASELINE.md §3 items 3-4 ask:
on one core, and with a process pool over all host cores (leaves are
independent).  Only the seed search is timed (the Python ``orient`` of the
reference is not part of the number).  Reports leaf seeds tested/s =
sum(seed + 1) / seconds on a bounded sample of the config's leaves.
"""

import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
MAX_SEED = 1 << 40

# (leaves on one core, leaves on the pool): ~1 s / ~1-2 s / ~5 s + ~15 s on 16 cores
SAMPLES = {1: (2000, 2000), 3: (1000, 20000), 5: (4, 200)}

_HI = _LO = _N = None


def _init(hi, lo, n):
    global _HI, _LO, _N
    _HI, _LO, _N = hi, lo, n


def _solve(i):
    import refbuild

    K = refbuild.ref_kernels()
    t = time.perf_counter()
    s = K.search_plain(_HI[i], _LO[i], _N, MAX_SEED)[0]
    return int(s) + 1, time.perf_counter() - t


def time_leaf_config(cfg, one_core=None, pool=None):
    """{'one_core': ..., 'pool': ...} seeds tested/s of the reference search."""
    if HERE not in sys.path:
        sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    import refbuild
    from paper_2308_09561_b200 import workloads as W  # input recipe only

    if not refbuild.have_ref():
        return {"error": "oracle/_ref (the reference's compiled kernels) is missing"}
    K = refbuild.ref_kernels()
    n = W.LEAF_CONFIGS[cfg]["n"]
    l1, lp = SAMPLES[cfg]
    l1 = one_core or l1
    lp = pool or lp
    hi, lo = W.leaf_inputs(cfg, max(l1, lp))
    out = {}
    t = time.perf_counter()
    seeds1 = sum(int(K.search_plain(hi[i], lo[i], n, MAX_SEED)[0]) + 1 for i in range(l1))
    dt = time.perf_counter() - t
    out["one_core"] = {"value": round(seeds1 / dt, 1), "unit": "leaf seeds tested/s", "cores": 1,
                       "sample": f"leaves 0..{l1 - 1} of C{cfg}", "seconds": round(dt, 3), "seeds_tested": seeds1}
    cores = os.cpu_count() or 1
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=_init, initargs=(hi[:lp], lo[:lp], n)) as p:
        p.map(_solve, range(min(cores, lp)))  # warm the workers
        t = time.perf_counter()
        res = p.map(_solve, range(lp), chunksize=1 if cfg == 5 else 64)
        dt = time.perf_counter() - t
    seedsp = sum(r[0] for r in res)
    out["pool"] = {"value": round(seedsp / dt, 1), "unit": "leaf seeds tested/s", "cores": cores,
                   "sample": f"leaves 0..{lp - 1} of C{cfg}, multiprocessing.Pool({cores}) one leaf per task",
                   "seconds": round(dt, 3), "seeds_tested": seedsp}
    out["kind"] = "reference"
    return out


if __name__ == "__main__":
    for c in sys.argv[1:] or ["1", "3"]:
        print(c, time_leaf_config(int(c)))
