#!/bin/bash
# A/B of leaf-search runtime knobs (environment) on C3 and the full C5:
#   tools/ab_leaf_env.sh "SHK_LEAF_TAIL_K=0" "SHK_LEAF_TAIL_K=1" ...
for e in "$@"; do
  echo "== $e"
  env $e python tools/leaf_probe.py 3 100000 4 2>&1 | tail -3
  [ -n "$C5" ] && env $e python tools/leaf_probe.py 5 20000 1 2>&1 | tail -1
done
