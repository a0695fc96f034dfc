#!/bin/bash
# query-only A/B: the C4 bench's query phase (1e8 queries) per library variant
for v in "$@"; do
  SHK_LIB_PATH=$PWD/paper_2308_09561_b200/_lib/variants/libshockhash_b200_$v.so python bench.py --steps 3 --warmup 3 --no-cpu-baseline --leaf-configs "" --no-check --query-reps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); q=d['query']; print('$v', q['ms'], q['value'], d['ms_per_step'])"
done
