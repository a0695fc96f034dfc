"""Dump the C4 build's Rice stream and choice bits (leaf order) of the library
in SHK_LIB_PATH to gpurun_out/ph_<tag>.npz; `compare A B` diffs two dumps.
Used to A/B the tree kernel's tail hand-off for exactness."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

if sys.argv[1] == "compare":
    a = np.load(f"gpurun_out/ph_{sys.argv[2]}.npz")
    b = np.load(f"gpurun_out/ph_{sys.argv[3]}.npz")
    for k in a.files:
        x, y = a[k], b[k]
        if x.shape != y.shape:
            print(k, "shape", x.shape, y.shape)
            continue
        d = np.nonzero(x != y)[0]
        print(k, "differs at", len(d), "positions", d[:20])
    sys.exit(0)

from paper_2308_09561_b200 import device as dev
from paper_2308_09561_b200 import recsplit
from paper_2308_09561_b200 import shockhash as leaf_mod
from paper_2308_09561_b200 import workloads as W
from paper_2308_09561_b200._kernels import kernels as K

tag = sys.argv[1]
N, b, n = 10_000_000, 2000, 40
keys = W.build_keys(4)[:N]
blob = np.frombuffer(np.ascontiguousarray(keys, dtype="<u8").tobytes(), dtype=np.uint8)
d_blob = dev.DeviceBuffer.from_host(blob)
d_hi, d_lo = dev.DeviceBuffer(8 * N), dev.DeviceBuffer(8 * N)
dev.blake2b_fixed_device(d_blob, 8, N, 0, d_hi, d_lo)
dev.sync()
nb = (N + b - 1) // b
lg = recsplit.leaf_g_table(n)
gb = K.GpuBuild(None, None, nb, hi_ptr=d_hi.ptr, lo_ptr=d_lo.ptr, n=N)
kp = gb.key_prefix()
plans = recsplit.packed_plans_for_sizes(np.unique(np.diff(kp.astype(np.int64))), n, lg)
st = gb.run(plans, 1, 0, leaf_mod.CACHE_MIN_LEAF, 0, nb, leaf_mod.MAX_SEED)
words, bl, bo = gb.stream()
ch = gb.choice()
np.savez(f"gpurun_out/ph_{tag}.npz", words=words, bo=bo, choice=ch, stats=st)
print(tag, "stream bits", bl, "stats", st)
