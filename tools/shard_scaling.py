"""Per-rank work of the bucket-range-sharded C4 build, measured on one GPU:
rank 0's share (the first 1/W of the buckets) for W = 1, 2, 4, 8, timed alone
(no other rank on the device, so nothing waits).  Prints the tree-kernel time
of the share against (full time / W): the strong-scaling efficiency of the
search phase before any exchange.

  python tools/shard_scaling.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

from paper_2308_09561_b200 import device as dev
from paper_2308_09561_b200 import recsplit
from paper_2308_09561_b200 import shockhash as leaf_mod
from paper_2308_09561_b200 import workloads as W
from paper_2308_09561_b200._kernels import kernels as K

N, b, n = 10_000_000, 2000, 40
keys = W.build_keys(4)[:N]
blob = np.frombuffer(np.ascontiguousarray(keys, dtype="<u8").tobytes(), dtype=np.uint8)
d_blob = dev.DeviceBuffer.from_host(blob)
d_hi, d_lo = dev.DeviceBuffer(8 * N), dev.DeviceBuffer(8 * N)
dev.blake2b_fixed_device(d_blob, 8, N, 0, d_hi, d_lo)
dev.sync()
nb = (N + b - 1) // b
lg = recsplit.leaf_g_table(n)


def tree_ms(b0, b1, reps=3, warm=1):
    # the first build of a new bucket range can pay pool allocations inside
    # the timed phase window (seen as one 30-190 ms outlier): untimed warm-up
    out = []
    for i in range(warm + reps):
        gb = K.GpuBuild(None, None, nb, hi_ptr=d_hi.ptr, lo_ptr=d_lo.ptr, n=N)
        kp = gb.key_prefix()
        plans = recsplit.packed_plans_for_sizes(np.unique(np.diff(kp.astype(np.int64))), n, lg)
        gb.run(plans, 1, 0, leaf_mod.CACHE_MIN_LEAF, b0, b1, leaf_mod.MAX_SEED)
        if i >= warm:
            out.append(gb.phase_ms()[0][1])
        gb.close()
    return float(np.median(out))


full = tree_ms(0, nb)
print(f"W=1 tree {full:.2f} ms")
for w in [int(x) for x in os.environ.get("SHK_SHARDS", "2,4,8").split(",")]:
    times = []
    for r in range(w):
        b0, b1 = (nb * r) // w, (nb * (r + 1)) // w
        times.append(tree_ms(b0, b1, reps=1))
    worst = max(times)
    print("  per rank:", " ".join(f"{t:.2f}" for t in times))
    print(f"W={w} slowest rank share {worst:.2f} ms, ideal {full / w:.2f} ms, efficiency {full / w / worst:.3f}")
