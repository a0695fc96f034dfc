"""Per-rank share of a sharded leaf-only config, measured on ONE GPU.

  python tools/leaf_shard_proxy.py CFG W

Rank r of W searches the contiguous leaf range [L r/W, L (r+1)/W) (what
bench.py --gpus W runs on W GPUs).  Each range is searched alone here, one
after another, so no rank's kernel waits on another's; the slowest range's
time against (time of all leaves) / W is the scaling efficiency the W-GPU
run can reach with no exchange.  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

from paper_2308_09561_b200 import device as dev
from paper_2308_09561_b200 import workloads as W
from paper_2308_09561_b200._kernels import kernels as K

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
spec = W.LEAF_CONFIGS[cfg]
L, n = spec["leaves"], spec["n"]
hi, lo = W.leaf_inputs(cfg)


def run(l0, l1):
    m = l1 - l0
    d_hi = dev.DeviceBuffer.from_host(np.ascontiguousarray(hi[l0:l1]).ravel())
    d_lo = dev.DeviceBuffer.from_host(np.ascontiguousarray(lo[l0:l1]).ravel())
    d_off = dev.DeviceBuffer.from_host(np.arange(0, (m + 1) * n, n, dtype=np.int64))
    d_seed, d_fb = dev.DeviceBuffer(8 * m), dev.DeviceBuffer(8 * m)
    with dev.timer() as tm:
        K.leaf_search_device(d_hi.ptr, d_lo.ptr, d_off.ptr, m, 0, d_seed.ptr, d_fb.ptr)
    seeds = d_seed.download(np.int64, m)
    for b in (d_hi, d_lo, d_off, d_seed, d_fb):
        b.free()
    return tm.ms, float((seeds + 1).sum())


if cfg != 5:
    run(0, L)  # warm-up
full_ms, full_seeds = run(0, L)
shares = [run((L * r) // world, (L * (r + 1)) // world) for r in range(world)]
worst = max(s[0] for s in shares)
print(json.dumps({"config": f"C{cfg}", "world": world, "all_leaves_ms": round(full_ms, 2),
                  "rank_ms": [round(s[0], 2) for s in shares],
                  "rank_seed_share": [round(s[1] / full_seeds, 4) for s in shares],
                  "ideal_ms": round(full_ms / world, 2), "slowest_rank_ms": round(worst, 2),
                  "efficiency": round(full_ms / world / worst, 4)}))
