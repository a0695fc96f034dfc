#!/bin/bash
# A/B of library variants on the C4 step and on the per-rank shard scaling:
#   tools/ab_shard.sh v0 v1 ...
for v in "$@"; do
  L=$PWD/paper_2308_09561_b200/_lib/variants/libshockhash_b200_$v.so
  echo "== $v"
  SHK_LIB_PATH=$L python bench.py --steps 5 --warmup 3 --no-cpu-baseline --queries 0 --leaf-configs "" 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms']['split_search'], d['parity']['desc_matches_reference'])"
  SHK_LIB_PATH=$L SHK_SHARDS=${SHARDS:-4,8,16} python tools/shard_scaling.py 2>/dev/null | grep -v "per rank"
done
