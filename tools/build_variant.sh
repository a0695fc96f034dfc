#!/bin/bash
# Build an experimental variant of the library with extra nvcc defines:
#   tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"
# -> paper_2308_09561_b200/_lib/variants/libshockhash_b200_NAME.so (load with SHK_LIB_PATH).
set -e
NAME=$1; shift
DEFS="$*"
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2308_09561_b200/csrc
OUT=$ROOT/paper_2308_09561_b200/_lib/variants
B=$(mktemp -d)
mkdir -p "$OUT"
for f in "$SRC"/*.cu; do
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -O3 \
    -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr $DEFS -c "$f" -o "$B/$(basename "$f" .cu).o" &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$OUT/libshockhash_b200_$NAME.so" "$B"/*.o
rm -rf "$B"
echo "$OUT/libshockhash_b200_$NAME.so"
