# FP64 DMMA peak with SM clocks sampled under load (profiles/r02_fp64_peak.log)
set -e
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 200 > gpurun_out/peak_clocks.csv &
SMI=$!
./tools/fp64_peak > gpurun_out/peak.log
./tools/fp64_peak 8 >> gpurun_out/peak.log
kill $SMI
cat gpurun_out/peak.log
echo "clocks during the run (sm MHz, max MHz, W, reasons): median of samples above 1 GHz:"
python - <<'PY'
import statistics
rows=[l.split(',') for l in open('gpurun_out/peak_clocks.csv') if l.strip()]
sm=[float(r[0].split()[0]) for r in rows]
load=[v for v in sm if v>1000]
print("samples", len(rows), "under load", len(load), "median", statistics.median(load) if load else None,
      "max", max(float(r[1].split()[0]) for r in rows), "reasons", sorted(set(r[3].strip() for r in rows)))
PY
