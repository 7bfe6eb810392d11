# A/B of the recursion kernel variants (knobs: BCG_RF_VARIANT=2|3|6, BCG_RF_TILE, BCG_RF_STEPS; see recursion_fact.cu).
# VARIANTS: space-separated settings, each a comma-separated list of VAR=value.
for c in ${CONFIGS:-cfg2 cfg3 cfg4}; do
 for v in ${VARIANTS:-BCG_RF_VARIANT=2,BCG_RF_TILE=-1 BCG_RF_VARIANT=2,BCG_RF_TILE=0 BCG_RF_VARIANT=2,BCG_RF_TILE=1 BCG_RF_VARIANT=3 BCG_RF_VARIANT=6}; do
  echo -n "$v: "; env $(echo $v | tr , ' ') timeout 300 python tools/bench_recursion.py --configs $c --reps ${REPS:-10} 2>&1 | tail -1
 done
done
