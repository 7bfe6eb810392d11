# One GPU session: the full GPU test suite, bench lines for the single-GPU BASELINE configs, the reference arm,
# the launch list of the default bench command, the recursion at every config layout, the cfg5 per-rank shard.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; tail -2 gpurun_out/bench_cfg4.err
timeout 600 python bench.py --config cfg2 --steps 10 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 900 python bench.py --config cfg3 --steps 5 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference_cfg4.json 2> gpurun_out/bench_reference_cfg4.err
timeout 600 python tools/bench_recursion.py --configs cfg2 cfg3 cfg4 cfg5 --reps 10 --copy-ref > gpurun_out/rec.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_cfg4.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
timeout 900 python tools/run_cfg.py --config cfg5 --t 500000 --reps 1 > gpurun_out/cfg5_shard.log 2>&1
cat gpurun_out/bench_cfg*.json gpurun_out/bench_reference_cfg4.json gpurun_out/rec.log; tail -5 gpurun_out/cfg5_shard.log
