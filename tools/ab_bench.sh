#!/bin/bash
# A/B the C4 build across library variants (tools/build_variant.sh):
#   tools/ab_bench.sh v0 v1 ...   -> gpurun_out/ab_<v>.json, one summary line each
mkdir -p gpurun_out
for v in "$@"; do
  SHK_LIB_PATH=$PWD/paper_2308_09561_b200/_lib/variants/libshockhash_b200_$v.so \
    python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --queries 0 --leaf-configs "" --no-check \
    > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
    print(v, d["ms_per_step"], d["phase_ms"], d["e2e"]["ms_per_step"])
except Exception as e:
    print(v, "FAILED", e)
PY
done
