#!/usr/bin/env bash
# Build the UNMODIFIED reference package (blockcumulants, Python + its one
# Cython kernel _core.pyx) from /root/reference/pkg into oracle/_ref/.
#
# Test/bench infrastructure only: oracle/_ref is the parity checker and the
# `bench.py --impl reference` CPU arm; no product code imports it.
#
# /root/reference is read-only, so the build happens in a scratch copy under
# /tmp (the reference's own setup.py, `build_ext --inplace`, -O3 per
# pkg/setup.py:4-14); only the built package lands in oracle/_ref/, which is
# git-ignored (never committed) but travels to the GPU box with the snapshot.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${REFERENCE_ROOT:-/root/reference}/pkg"
OUT="$HERE/_ref"
if [ ! -d "$SRC" ]; then
  echo "build_ref: $SRC absent (GPU box?) - keeping prebuilt $OUT" >&2
  exit 0
fi
WORK="$(mktemp -d /tmp/bcref.XXXXXX)"
trap 'rm -rf "$WORK"' EXIT
cp -r "$SRC" "$WORK/pkg"
chmod -R u+w "$WORK/pkg"
( cd "$WORK/pkg" && python3 setup.py build_ext --inplace >"$WORK/build.log" 2>&1 ) || {
  cat "$WORK/build.log" >&2; exit 1; }
rm -rf "$OUT"
mkdir -p "$OUT"
cp -r "$WORK/pkg/src/blockcumulants" "$OUT/blockcumulants"
rm -rf "$OUT/blockcumulants/__pycache__" "$OUT/blockcumulants"/*.c "$OUT/blockcumulants"/*.pyx
ls "$OUT/blockcumulants"/_core*.so >/dev/null
echo "build_ref: built $(ls "$OUT/blockcumulants"/_core*.so)"
