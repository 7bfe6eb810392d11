# A/B of the streamed order-6 recursion variants (BCG_RS_TILE) at the cfg5 layout:
# bitwise check against v2 (tools/dbg_rs2.py) then the L2-flushed timing.
mkdir -p gpurun_out
for v in "$@"; do
  echo "== BCG_RS_TILE=$v"
  BCG_RS_TILE=$v timeout 120 python tools/dbg_rs2.py 60 3000
  BCG_RS_TILE=$v timeout 120 python tools/bench_recursion.py --configs cfg5 --reps 10
done
