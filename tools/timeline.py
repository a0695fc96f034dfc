"""Device timeline of one C4 build (torch.profiler / CUPTI sees every kernel
and memcpy in the process, ours included): prints the idle gaps between
consecutive device activities, largest first.

  python tools/timeline.py [N]
"""
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

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
keys = W.build_keys(4)[:N]
blob = np.frombuffer(np.ascontiguousarray(keys, dtype="<u8").tobytes(), dtype=np.uint8)
d_blob = dev.DeviceBuffer.from_host(blob)
d_hi, d_lo = dev.DeviceBuffer(8 * N), dev.DeviceBuffer(8 * N)
dev.blake2b_fixed_device(d_blob, 8, N, 0, d_hi, d_lo)
dev.sync()
torch.cuda.init()
for _ in range(2):
    recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, 2000, 40, 1)
dev.sync()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, 2000, 40, 1)
    dev.sync()
path = "/tmp/timeline_trace.json"
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
dev_ev = sorted((e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e),
                key=lambda e: e["ts"])
t0, t1 = dev_ev[0]["ts"], dev_ev[-1]["ts"] + dev_ev[-1]["dur"]
busy = sum(e["dur"] for e in dev_ev)
print(f"device span {1e-3 * (t1 - t0):.3f} ms, busy {1e-3 * busy:.3f} ms, {len(dev_ev)} activities")
gaps = []
end = dev_ev[0]["ts"] + dev_ev[0]["dur"]
prev = dev_ev[0]["name"]
for e in dev_ev[1:]:
    g = e["ts"] - end
    if g > 0:
        gaps.append((g, prev, e["name"]))
    if e["ts"] + e["dur"] > end:
        end = e["ts"] + e["dur"]
        prev = e["name"]
if os.environ.get("SHK_TIMELINE_ALL"):
    for e in dev_ev:
        print(f"{1e-3 * (e['ts'] - t0):10.3f} {e['dur']:9.1f} {e['name'][:70]}")
gaps.sort(reverse=True)
print(f"idle total {1e-3 * sum(g for g, _, _ in gaps):.3f} ms")
for g, a, b in gaps[:25]:
    print(f"{g:9.1f} us  after {a[:60]:60s} before {b[:60]}")
