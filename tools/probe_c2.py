"""Phase breakdown of the C2 build (N=1e5, n=24, b=500, rotate) from resident
codes: device phases (CUDA events) against the host wall time per build."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

from paper_2308_09561_b200 import device as dev
from paper_2308_09561_b200 import recsplit
from paper_2308_09561_b200 import workloads as W

N, n, b = 100_000, 24, 500
k = W.build_keys(2)
blob = np.frombuffer(np.ascontiguousarray(k, dtype="<u8").tobytes(), dtype=np.uint8)
d_blob = dev.DeviceBuffer.from_host(blob)
d_hi, d_lo = dev.DeviceBuffer(8 * N), dev.DeviceBuffer(8 * N)
dev.blake2b_fixed_device(d_blob, 8, N, 0, d_hi, d_lo)
dev.sync()
for _ in range(5):
    recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, b, n, 1)
for _ in range(5):
    dev.sync()
    t = time.perf_counter()
    d = recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, b, n, 1)
    dev.sync()
    wall = (time.perf_counter() - t) * 1e3
    ph = {k_: round(v, 3) for k_, v in d.device_profile["phase_ms"].items()}
    print(f"wall {wall:.3f} ms, phases {ph}, sum {sum(ph.values()):.3f}")
