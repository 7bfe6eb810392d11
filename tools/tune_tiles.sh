#!/usr/bin/env bash
# Time each v1 tile shape per (config, order) in its own process (BCG_TILE).
for cfgord in "cfg2 3" "cfg2 4" "cfg3 4" "cfg3 5" "cfg4 4" "cfg4 5" "cfg4 6"; do
  set -- $cfgord
  for tile in 64x64 16x128 128x16 32x64 64x32 32x32; do
    BCG_TILE=$tile python tools/tune_moment.py --configs $1 --order $2 --reps 2 2>&1 | sed "s/^/$tile /"
  done
done
