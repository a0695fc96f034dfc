#!/bin/bash
# A/B the leaf-search-only configs across library variants (tools/build_variant.sh):
#   tools/ab_leaf.sh v0 v1 ...   -> C3 (3 launches) and a 2,000-leaf C5 sample per variant
for v in "$@"; do
  L=$PWD/paper_2308_09561_b200/_lib/variants/libshockhash_b200_$v.so
  echo "== $v"
  SHK_LIB_PATH=$L python tools/leaf_probe.py 3 100000 3 2>&1 | tail -2
  SHK_LIB_PATH=$L python tools/leaf_probe.py 5 2000 1 2>&1 | tail -1
done
