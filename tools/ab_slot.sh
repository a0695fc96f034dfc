#!/bin/bash
# A/B of the slot-aware tree schedule (shk_tree.cu) on the C4 step and the
# per-rank shard scaling:  tools/ab_slot.sh "ENV=.. ENV2=.." ...
for e in "$@"; do
  echo "== $e"
  env $e python bench.py --steps 5 --warmup 3 --no-cpu-baseline --queries 0 --leaf-configs "" 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms']['split_search'], d['parity']['desc_matches_reference'], d['e2e']['ms_per_step'])"
  env $e SHK_SHARDS=${SHARDS:-2,4,8} python tools/shard_scaling.py 2>/dev/null | grep -v "per rank"
done
