#!/bin/bash
# A/B of the tree kernel's tail hand-off on one box (run from the repo root):
#   tools/build_variant.sh base   (on a checkout without the hand-off, copied into _lib/variants)
#   tools/ab_handoff.sh [variant ...]
# Each variant is timed as built, then the current library with the hand-off
# off (SHK_TREE_HANDOFF_TW=0) and with resume teams of 4 and 8 warps.
L=$PWD/paper_2308_09561_b200/_lib/variants
export STEPS=${STEPS:-10}
args=()
for v in "$@"; do args+=("SHK_LIB_PATH=$L/libshockhash_b200_$v.so"); done
for rep in 1 2; do
  tools/ab_env.sh "${args[@]}" "SHK_TREE_HANDOFF_TW=0" "SHK_TREE_HANDOFF_TW=4" "SHK_TREE_HANDOFF_TW=8"
done
