"""The integer-issue microbenchmark alone (csrc/shk_peak.cu), for ncu:
  python tools/int_peak.py
prints Tops/s per instruction mix; under ncu --metrics the pipe counters
(sm__pipe_alu_cycles_active, sm__pipe_fmaheavy_cycles_active,
smsp__issue_active) confirm which pipes each mix saturates."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2308_09561_b200 import device as dev

for kind, name in {**dev.INT_PEAK_KINDS, **dev.INT_PEAK_KINDS_EXTRA}.items():
    ms, ops = dev.int_peak(kind, 16384)
    print(f"{name}: {ops / (ms * 1e-3) / 1e12:.2f} Tops/s ({ms:.3f} ms)")
