timeout 600 python tools/ab_priv.py
for cfg in cfg4 cfg2 cfg3; do
  for env in "BCG_X=0" "BCG_MOMENT_PRIV=1"; do
    echo "== $cfg $env"
    env $env timeout 400 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['avg_launch_ms'])"
  done
done
