"""C4 build phases under the per-level schedule (one split launch per tree
level, then the leaf launch), so split and leaf search are timed apart:
  python tools/probe_phase.py [schedule]   (0 = persistent tree kernel)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

from paper_2308_09561_b200 import device as dev
from paper_2308_09561_b200 import recsplit
from paper_2308_09561_b200 import workloads as W

sched = int(sys.argv[1]) if len(sys.argv) > 1 else 1
N, b, n = 10_000_000, 2000, 40
keys = W.build_keys(4)[:N]
blob = np.frombuffer(np.ascontiguousarray(keys, dtype="<u8").tobytes(), dtype=np.uint8)
d_blob = dev.DeviceBuffer.from_host(blob)
d_hi, d_lo = dev.DeviceBuffer(8 * N), dev.DeviceBuffer(8 * N)
dev.blake2b_fixed_device(d_blob, 8, N, 0, d_hi, d_lo)
dev.sync()
dev.set_option(dev.OPT_SCHEDULE, sched)
for it in range(3):
    d = recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, b, n, 1)
    ph = {k_: round(v, 3) for k_, v in d.device_profile["phase_ms"].items()}
    print(f"schedule {sched} build {it}: phases {ph}", flush=True)
