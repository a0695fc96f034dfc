"""Fingerprint kernel alone: python tools/probe_blake.py [N] [REPS] -> ms per launch, keys/s
(8-byte keys resident on the device; CUDA events on the context stream)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

from paper_2308_09561_b200 import device as dev

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
keys = np.random.default_rng(4).integers(0, 2**64, N, dtype=np.uint64)
d_blob = dev.DeviceBuffer.from_host(keys.view(np.uint8))
d_hi, d_lo = dev.DeviceBuffer(8 * N), dev.DeviceBuffer(8 * N)
best = 1e9
for r in range(reps + 2):
    with dev.timer() as tm:
        dev.blake2b_fixed_device(d_blob, 8, N, 0, d_hi, d_lo)
    if r >= 2:
        best = min(best, tm.ms)
hi = d_hi.download(np.uint64, N)
print(f"blake2b_fixed 8-byte keys N={N}: {best:.3f} ms, {N / best / 1e6:.2f} G keys/s, hi[0..1]={hi[0]:#x},{hi[1]:#x}")
