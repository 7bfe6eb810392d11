# v7d (0) / v8 (16) / v9 (default) on ONE box, three interleaved repetitions (L2 flushed, median of 10 launches each)
for rep in 1 2 3; do
  for v in 0 16 -1; do
    echo "== rep $rep BCG_RS_TILE=$v"
    BCG_RS_TILE=$v timeout 120 python tools/bench_recursion.py --configs cfg5 --reps 10
  done
done
