set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for o in "cfg3 5" "cfg3 3" "cfg4 5" "cfg4 3" "cfg2 3"; do set -- $o
  timeout 300 python tools/tune_moment.py --configs $1 --order $2 --reps 5 2>&1 | tail -1
  BCG_NO_HYBRID=1 timeout 300 python tools/tune_moment.py --configs $1 --order $2 --reps 5 2>&1 | tail -1
done
