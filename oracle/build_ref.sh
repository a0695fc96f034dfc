#!/usr/bin/env bash
# Compile the REFERENCE's own CPU kernels (its Cython module _core.pyx, read
# in place from /root/reference) into oracle/_ref/ — the reference CPU arm of
# bench.py.  Nothing from /root/reference is copied into the repo: Cython
# writes its generated C into a temp dir, gcc links the extension into
# oracle/_ref/ (git-ignored; it travels to the GPU box with the snapshot).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=/root/reference/pkg/src/shockhash/_kernels/_core.pyx
OUT="$HERE/_ref"
if [ ! -f "$SRC" ]; then echo "reference sources not present; skipping" >&2; exit 0; fi
mkdir -p "$OUT"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
python -m cython -3 -o "$TMP/_core.c" "$SRC"
PYINC="$(python -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
NPINC="$(python -c 'import numpy; print(numpy.get_include())')"
EXT="$(python -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
gcc -O3 -fPIC -shared -fwrapv -I"$PYINC" -I"$NPINC" "$TMP/_core.c" -o "$OUT/_core$EXT"
echo "built $OUT/_core$EXT"
