"""Probe: the ribbon solve alone on N synthetic rows (kernel timing)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2308_09561_b200._kernels import kernels as K
from paper_2308_09561_b200.keys import synthetic_hashed
from paper_2308_09561_b200 import device as dev

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
hi, lo = synthetic_hashed(N, 1)
rhs = (hi & np.uint64(1)).astype(np.uint8)
m = max(128, int(np.ceil(1.05 * N)))
for it in range(3):
    t = time.perf_counter()
    seed, w = K.ribbon_build(hi, lo, rhs, m)
    print("ribbon_build", N, "seed", seed, "ms", round((time.perf_counter() - t) * 1e3, 2), flush=True)
