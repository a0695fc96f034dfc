"""Probe: host-side time breakdown of one C4 build (device-resident codes)."""
import sys, os, time, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2308_09561_b200 import device as dev, recsplit, workloads as W
k = W.build_keys(4)
blob = np.frombuffer(np.ascontiguousarray(k, dtype="<u8").tobytes(), dtype=np.uint8)
N = len(k)
d_blob = dev.DeviceBuffer.from_host(blob); d_hi = dev.DeviceBuffer(8 * N); d_lo = dev.DeviceBuffer(8 * N)
dev.blake2b_fixed_device(d_blob, 8, N, 0, d_hi, d_lo); dev.sync()
for _ in range(2):
    recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, 2000, 40)
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
d = recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, 2000, 40)
pr.disable()
print("build wall ms", (time.perf_counter() - t) * 1e3, d.device_profile["phase_ms"])
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
