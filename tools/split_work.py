"""Issued vs algorithmic split work of the C4 build (analysis build only):
  tools/build_variant.sh sw -DSHK_SPLIT_WORK
  SHK_LIB_PATH=.../libshockhash_b200_sw.so python tools/split_work.py
Counts the lane-key evaluations the fast split searches of the tree kernel
issue (32 lanes x keys processed per 32-seed block) against the reference's
split `evals` (the exact instrumented build), i.e. the work the lock-step
32-seed blocks and the every-8-keys overflow check add."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

from paper_2308_09561_b200 import device as dev
from paper_2308_09561_b200 import recsplit
from paper_2308_09561_b200 import workloads as W
from paper_2308_09561_b200._kernels import _lib

N, b, n = 10_000_000, 2000, 40
keys = W.build_keys(4)[:N]
blob = np.frombuffer(np.ascontiguousarray(keys, dtype="<u8").tobytes(), dtype=np.uint8)
d_blob = dev.DeviceBuffer.from_host(blob)
d_hi, d_lo = dev.DeviceBuffer(8 * N), dev.DeviceBuffer(8 * N)
dev.blake2b_fixed_device(d_blob, 8, N, 0, d_hi, d_lo)
dev.sync()
lib = _lib.load_library()
lib.shk_debug_split_work.restype = ctypes.c_int
lib.shk_debug_split_work.argtypes = [ctypes.c_void_p, ctypes.c_int]
ctr = np.zeros(2, dtype=np.uint64)

dev.set_option(dev.OPT_EXACT_SPLIT_EVALS, 1)
d = recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, b, n, 1)
dev.set_option(dev.OPT_EXACT_SPLIT_EVALS, 0)
ref_evals = d.device_profile["split_evals"]
lib.shk_debug_split_work(ctr.ctypes.data, 1)
d = recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, b, n, 1)
lib.shk_debug_split_work(ctr.ctypes.data, 1)
issued, blocks = int(ctr[0]), int(ctr[1])
print(f"reference split evals {ref_evals:.4e}")
print(f"issued lane-key evals {issued:.4e} in {blocks} seed blocks (32 seeds each)")
print(f"issued / reference = {issued / ref_evals:.3f}")
print("phase_ms", d.device_profile["phase_ms"])
