#!/bin/bash
# A/B of the C4 build across environment settings on one box:
#   tools/ab_env.sh "SHK_RIBBON_EMIT=1" "SHK_RIBBON_EMIT=0" ...  -> one summary line per setting
mkdir -p gpurun_out
i=0
for e in "$@"; do
  i=$((i+1))
  env $e python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --queries 0 --leaf-configs "" --no-check \
    > gpurun_out/abenv_$i.json 2> gpurun_out/abenv_$i.err
  python - "$e" "$i" <<'PY'
import json, sys
e, i = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/abenv_{i}.json").read().strip().splitlines()[-1])
    print(e, d["ms_per_step"], {k: round(v, 3) for k, v in d["phase_ms"].items()}, d["e2e"]["ms_per_step"])
except Exception as ex:
    print(e, "FAILED", ex)
PY
done
