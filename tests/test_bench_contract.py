"""bench.py's JSON contract, checked on the CPU-only reference arm (the GPU
arm is exercised by the driver on the B200): one JSON line with the metric,
unit, config, cpu_baseline and e2e keys the contract names."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_contract_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["unit"] == "TFLOP/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("cfg1")
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_non_zero_ranks_exit_silently():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env={**os.environ, "RANK": "1", "WORLD_SIZE": "2", "CUDA_VISIBLE_DEVICES": ""})
    assert out.returncode == 0 and not out.stdout.strip()


def test_reference_arm_extrapolates_by_a_linear_fit():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    d = json.loads(out.stdout.strip().splitlines()[-1])
    fit = d["cpu_baseline"]["fit"]
    assert fit["t1"] < fit["t2"] and fit["b_s_per_row"] > 0 and fit["a_s"] >= 0
    assert abs(fit["full_t_s_extrapolated"] - (fit["a_s"] + fit["b_s_per_row"] * fit["full_t"])) < 1e-9
    assert abs(d["ms_per_step"] - 1e3 * fit["full_t_s_extrapolated"]) < 1e-6
    assert d["cpu_baseline"]["threads"]["host_cores"] >= 1 and "cgroup" in d["cpu_baseline"]["threads"]
    assert len(d["cpu_baseline"]["engines_s_at_t2"]) >= 1


def test_gpus_flag_launches_one_rank_per_gpu():
    # --gpus 2 outside torchrun re-launches bench.py under torch.distributed.run
    # with two ranks; the dry run rendezvous over gloo and counts them (no GPU)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                          "--config", "cfg4"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["ranks_seen"] == 2
    # strong scaling by default: the two shards cover the canonical t rows once
    assert d["rows_total"] == 1_000_000 and d["config"]["t"] == 1_000_000
    assert "strong" in d["config"]["parallelism"]
