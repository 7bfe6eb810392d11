for c in cfg2 cfg3 cfg4; do
 for v in "BCG_RF_VARIANT=2 BCG_RF_TILE=-1" "BCG_RF_VARIANT=2 BCG_RF_TILE=0" "BCG_RF_VARIANT=2 BCG_RF_TILE=1" "BCG_RF_VARIANT=3" "BCG_RF_VARIANT=4"; do
  echo -n "$v: "; env $v timeout 300 python tools/bench_recursion.py --configs $c --reps 10 2>&1 | tail -1
 done
done
for v in "BCG_RF_TILE=0" "BCG_RF_TILE=1"; do echo -n "$v: "; env $v timeout 300 python tools/bench_recursion.py --configs cfg5 --reps 5 2>&1 | tail -1; done
