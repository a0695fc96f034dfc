"""Node-level timeline of the persistent tree kernel (analysis build only):
  tools/build_variant.sh trace -DSHK_TREE_TRACE
  SHK_LIB_PATH=.../libshockhash_b200_trace.so python tools/tree_trace.py [W]
Builds C4 (or rank 0's 1/W bucket share), reads every node's start/end
globaltimer and prints the busy-warp profile of the launch and the longest
nodes."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

from paper_2308_09561_b200 import device as dev
from paper_2308_09561_b200 import recsplit
from paper_2308_09561_b200 import shockhash as leaf_mod
from paper_2308_09561_b200 import workloads as W
from paper_2308_09561_b200._kernels import _lib
from paper_2308_09561_b200._kernels import kernels as K

Wn = int(sys.argv[1]) if len(sys.argv) > 1 else 1
N, b, n = 10_000_000, 2000, 40
keys = W.build_keys(4)[:N]
blob = np.frombuffer(np.ascontiguousarray(keys, dtype="<u8").tobytes(), dtype=np.uint8)
d_blob = dev.DeviceBuffer.from_host(blob)
d_hi, d_lo = dev.DeviceBuffer(8 * N), dev.DeviceBuffer(8 * N)
dev.blake2b_fixed_device(d_blob, 8, N, 0, d_hi, d_lo)
dev.sync()
nb = (N + b - 1) // b
lg = recsplit.leaf_g_table(n)
for rep in range(2):
    gb = K.GpuBuild(None, None, nb, hi_ptr=d_hi.ptr, lo_ptr=d_lo.ptr, n=N)
    kp = gb.key_prefix()
    plans = recsplit.packed_plans_for_sizes(np.unique(np.diff(kp.astype(np.int64))), n, lg)
    gb.run(plans, 1, 0, leaf_mod.CACHE_MIN_LEAF, 0, nb // Wn, leaf_mod.MAX_SEED)
    ms = gb.phase_ms()[0][1]
    gb.close()
lib = _lib.load_library()
lib.shk_debug_tree_trace.restype = ctypes.c_int
lib.shk_debug_tree_trace.argtypes = [ctypes.c_void_p, ctypes.c_int64]
tr = np.zeros((1 << 20, 2), dtype=np.uint64)
lib.shk_debug_tree_trace(tr.ctypes.data, 1 << 20)
lib.shk_debug_tree_trace_m.restype = ctypes.c_int
lib.shk_debug_tree_trace_m.argtypes = [ctypes.c_void_p, ctypes.c_int64]
tm = np.zeros(1 << 20, dtype=np.uint32)
lib.shk_debug_tree_trace_m(tm.ctypes.data, 1 << 20)
# nodes of this run: start >= the run's earliest (older entries are from the first rep or stale)
valid = tr[:, 1] > 0
t_end_max = tr[valid, 1].max()
t_first = tr[valid & (tr[:, 0] > t_end_max - np.uint64(int(ms * 1e6 * 1.5))), 0].min()
sel = valid & (tr[:, 0] >= t_first)
info = tm[sel] & np.uint32(0xFFFFFF)
wid = (tm[sel] >> np.uint32(24)).astype(np.int64)
st = (tr[sel, 0] - t_first).astype(np.float64) / 1e6
en = (tr[sel, 1] - t_first).astype(np.float64) / 1e6
dur = en - st
span = en.max()
print(f"W={Wn}: tree phase {ms:.2f} ms, traced span {span:.2f} ms, nodes {sel.sum()}")
print(f"node durations: mean {dur.mean()*1e3:.1f} us, p99 {np.percentile(dur,99)*1e3:.1f} us, max {dur.max():.2f} ms")
grid = np.linspace(0, span, 401)
busy = np.array([np.count_nonzero((st <= t) & (en > t)) for t in grid])
peak = busy.max()
for frac in (0.9, 0.5, 0.25, 0.1):
    idx = np.nonzero(busy >= frac * peak)[0]
    last = grid[idx[-1]] if len(idx) else 0
    print(f"busy >= {int(frac*100)}% of peak ({peak} warps) until {last:.2f} ms ({100*last/span:.1f}% of span)")
work = dur.sum()
print(f"warp-ms of work {work:.0f}; at peak occupancy the span would be {work / peak:.2f} ms")
order = np.argsort(-dur)[:12]
for i in order:
    print(f"  node m={info[i] >> 8} fanout={info[i] & 255} warpid={wid[i]}: start {st[i]:7.2f} end {en[i]:7.2f} ms, {dur[i]:.2f} ms")
# per node type: count, mean / max duration, share of warp-time
kinds = {}
for key in np.unique(info & 255):
    for big in (False, True):
        msk = ((info & 255) == key) & (((info >> 8) > 200) == big)
        if msk.any():
            kinds[(int(key), big)] = msk
for (f, big), msk in sorted(kinds.items()):
    d = dur[msk]
    print(f"  {'leaf' if f == 0 else f'split F={f}'} {'m>200' if big else 'm<=200'}: {msk.sum()} nodes, "
          f"mean {d.mean()*1e3:.0f} us, max {d.max():.2f} ms, {100*d.sum()/work:.1f}% of warp-time")
# per hardware warp slot (%warpid; the scheduler favours high slots): work done
# (node count, busy time) and the mean duration of the 4 x 40 split nodes
print("warpid: nodes, mean node us, mean 4x40-split us")
f40 = ((info & 255) == 4) & ((info >> 8) <= 200)
for w_ in range(int(wid.max()) + 1):
    m_ = wid == w_
    if m_.any():
        d40 = dur[m_ & f40]
        print(f"  {w_:3d}: {m_.sum():7d} {dur[m_].mean()*1e3:9.0f} {d40.mean()*1e3 if len(d40) else 0:9.0f}")
# the tail: the nodes still running in the last 3 ms of the launch
tail_t = span - 3.0
late = np.nonzero(en > tail_t)[0]
print(f"nodes running after {tail_t:.2f} ms: {len(late)} "
      f"(leaves {np.count_nonzero((info[late] & 255) == 0)}, splits {np.count_nonzero((info[late] & 255) != 0)})")
for i in late[np.argsort(-en[late])][:24]:
    print(f"  m={info[i] >> 8} fanout={info[i] & 255} warpid={wid[i]}: start {st[i]:7.2f} end {en[i]:7.2f} ms, {dur[i]:.2f} ms")
