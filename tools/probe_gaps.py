"""Host stage timestamps (SHK_HOST_TRACE) of one C4 build next to its device
timeline (torch.profiler): where the device waits for the host.
  SHK_HOST_TRACE=1 python tools/probe_gaps.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2308_09561_b200 import device as dev
from paper_2308_09561_b200 import recsplit
from paper_2308_09561_b200 import workloads as W

N = 10_000_000
keys = W.build_keys(4)[:N]
blob = np.frombuffer(np.ascontiguousarray(keys, dtype="<u8").tobytes(), dtype=np.uint8)
d_blob = dev.DeviceBuffer.from_host(blob)
d_hi, d_lo = dev.DeviceBuffer(8 * N), dev.DeviceBuffer(8 * N)
dev.blake2b_fixed_device(d_blob, 8, N, 0, d_hi, d_lo)
dev.sync()
torch.cuda.init()
for _ in range(3):
    recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, 2000, 40, 1)
dev.sync()
print("---- traced build", file=sys.stderr, flush=True)
if os.environ.get("NO_PROF"):  # host stages without the profiler's API callbacks
    d = recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, 2000, 40, 1)
    print({k: round(v, 3) for k, v in d.device_profile["phase_ms"].items()}, file=sys.stderr)
    sys.exit(0)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, 2000, 40, 1)
    dev.sync()
path = "/tmp/gaps_trace.json"
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
dev_ev = sorted((e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e),
                key=lambda e: e["ts"])
t0 = dev_ev[0]["ts"]
for e in dev_ev:
    print(f"{e['ts'] - t0:10.1f} {e['dur']:9.1f} {e['name'][:60]}")
