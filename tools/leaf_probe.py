"""Leaf-search-only run for profiling (no build, no queries):
  python tools/leaf_probe.py CFG [LEAVES] [REPS]
Runs the batched plain leaf search of config C1/C3/C5 (BASELINE.json) REPS
times on cuda:0 and prints ms per launch and leaf seeds tested/s, so that
`ncu -k regex:leaf_kernel` sees only the leaf kernel of that config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

from paper_2308_09561_b200 import device as dev
from paper_2308_09561_b200 import workloads as W
from paper_2308_09561_b200._kernels import kernels as K

if os.environ.get("SHK_LEAF_FIXED") == "1":  # A/B: fixed team per leaf, no seed-block stealing
    dev.set_option(dev.OPT_LEAF_FIXED_TEAMS, 1)
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
spec = W.LEAF_CONFIGS[cfg]
L = int(sys.argv[2]) if len(sys.argv) > 2 else spec["leaves"]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
n = spec["n"]
hi, lo = W.leaf_inputs(cfg, L)
hi, lo = hi.ravel(), lo.ravel()
d_hi, d_lo = dev.DeviceBuffer.from_host(hi), dev.DeviceBuffer.from_host(lo)
d_off = dev.DeviceBuffer.from_host(np.arange(0, (L + 1) * n, n, dtype=np.int64))
d_seed, d_fb = dev.DeviceBuffer(8 * L), dev.DeviceBuffer(8 * L)
for r in range(reps):
    with dev.timer() as tm:
        K.leaf_search_device(d_hi.ptr, d_lo.ptr, d_off.ptr, L, 0, d_seed.ptr, d_fb.ptr)
    seeds = d_seed.download(np.int64, L)
    st = float((seeds + 1).sum())
    print(f"C{cfg} {L} leaves n={n}: {tm.ms:.3f} ms, {st / (tm.ms * 1e-3):.4g} seeds/s, mean seeds {st / L:.1f}")
