"""Benchmark: cumulants_upto (center -> packed moments of orders 2..m -> recursion)
on BASELINE.json's configs, B200 sm_100a path vs the reference's CPU path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

A "step" is one full cumulants_upto pass over the config's synthetic matrix.
``value`` times it with the matrix already resident in HBM; ``e2e`` times the
public call on a pinned HOST matrix (H2D of X and D2H of C_1..C_m inside the
timed region).  The metric is algorithmic FP64 TFLOP/s, sum_k 2 t S_k over
k = 2..m (SURVEY.md §8 d), plus ms per step.  N > 1 (torchrun): each rank holds
its own t-row shard (weak scaling), partial moments are all-reduced over NCCL
(distributed.py).  Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402

METRIC = "moment+cumulant time & FP64 TFLOP/s at (n,m,t); % of DMMA / HBM roofline"
# FP64 DMMA peak measured on this pool's B200 (tools/fp64_peak.cu,
# profiles/r01_fp64_peak.log: mma.sync m8n8k4 f64 = 37.1 TFLOP/s at 1965 MHz).
# MEASURED_PEAKS.json carries no FP64 figure.
FP64_PEAK_TFLOPS = 37.1
FP64_PEAK_SOURCE = "measured DMMA.8x8x4 microbenchmark (tools/fp64_peak.cu, profiles/r01_fp64_peak.log)"
DEFAULT_WORKLOAD = "cfg2"  # configs[1]: the single-GPU headline case


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_WORKLOAD, choices=sorted(workloads.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-rows", type=int, default=0, help="rows of the CPU baseline sample (0 = auto)")
    ap.add_argument("--t", type=int, default=0,
                    help="rows per GPU instead of the config's t (exploration only: the line then says so; "
                         "e.g. cfg5 at its BASELINE t=4e6 takes ~13 min per step on one B200)")
    return ap.parse_args()


def config_dict(cfg, t_total, world):
    note = "" if t_total == cfg.t * world else f"; t overridden, BASELINE t={cfg.t} per GPU"
    return {
        "workload": f"{cfg.name}: cumulants_upto C1..C{cfg.m}, t={t_total} x n={cfg.n}, b={cfg.b} ({cfg.desc}){note}",
        "t": t_total, "n": cfg.n, "b": cfg.b, "m_max": cfg.m,
        "parallelism": f"t-shard x{world}" if world > 1 else "single GPU",
        "l2": "inputs larger than L2 (X = %.0f MB per GPU vs 126 MB L2)" % (cfg.t * cfg.n * 8 / 1e6),
    }


# --------------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        return False

    def summary(self):
        rows = []
        for line in (self.out or "").splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[2:6]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower().startswith("active")})
        loaded = [r[0] for r in rows if r[0] > 0.5 * r[1]] or [r[0] for r in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- CPU (reference)


def _load_reference():
    """The unmodified reference built by oracle/build_ref.sh (kind
    "reference"), else the oracle port (kind "port")."""
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref_dir, "blockcumulants")):
        sys.path.insert(0, ref_dir)
        import blockcumulants as bc

        if bc.HAVE_COMPILED:
            return "reference", bc
    return "port", None


def _cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _reference_run(kind, bc, x, cfg, engine):
    if kind == "reference":
        bc.cumulants_upto(x, cfg.m, b=cfg.b, engine=engine)
    else:
        from oracle import oracle as orc

        orc.cumulants_upto(x, cfg.m, cfg.b)


def cpu_sample_rows(cfg, requested: int) -> int:
    if requested:
        return requested
    # ~2-5 s per pass of the reference's best engine (SURVEY.md §6 rates)
    return {"cfg1": 20_000, "cfg2": 20_000, "cfg3": 4_000, "cfg4": 1_000, "cfg5": 400}[cfg.name]


def cpu_baseline(cfg, rows: int):
    """Reference cumulants_upto on a bounded t-row sample of the same recipe,
    best of its compiled (1 thread) and gram (BLAS threads) engines."""
    kind, bc = _load_reference()
    x = workloads.generate(cfg.name, rows)
    flops = workloads.moment_flops(rows, cfg.n, cfg.b, cfg.m)
    best = None
    engines = ("compiled", "gram") if kind == "reference" else ("port",)
    if cfg.name == "cfg5":
        engines = tuple(e for e in engines if e != "gram")  # refused by its 2e8 guard
    for eng in engines:
        t0 = time.perf_counter()
        _reference_run(kind, bc, x, cfg, eng)
        dt = time.perf_counter() - t0
        if best is None or dt < best[1]:
            best = (eng, dt)
    eng, dt = best
    cores = 1 if eng in ("compiled", "port") else _cpu_cores()
    return {
        "value": flops / dt / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": kind,
        "sample": f"cumulants_upto(X[:{rows}], {cfg.m}, b={cfg.b}, engine={eng!r}) of the {cfg.name} recipe, "
                  f"{dt:.2f} s (best of {', '.join(engines)}; host has {_cpu_cores()} cores)",
        "ms_per_sample": dt * 1e3,
    }


def run_reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    kind, bc = _load_reference()
    rows = cpu_sample_rows(cfg, args.cpu_sample_rows)
    x = workloads.generate(cfg.name, rows)
    flops = workloads.moment_flops(rows, cfg.n, cfg.b, cfg.m)
    engines = ("compiled", "gram") if kind == "reference" else ("port",)
    if cfg.name == "cfg5":
        engines = ("compiled",) if kind == "reference" else engines
    # calibrate: the faster engine is the reference's best CPU path on this host
    times = {}
    for eng in engines:
        t0 = time.perf_counter()
        _reference_run(kind, bc, x, cfg, eng)
        times[eng] = time.perf_counter() - t0
    eng = min(times, key=times.get)
    for _ in range(max(0, args.warmup - 1)):
        _reference_run(kind, bc, x, cfg, eng)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _reference_run(kind, bc, x, cfg, eng)
    dt = (time.perf_counter() - t0) / args.steps
    value = flops / dt / 1e12
    cores = 1 if eng in ("compiled", "port") else _cpu_cores()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic ({cfg.name} recipe, workloads.py), bounded sample of {rows} rows per step",
        "config": config_dict(cfg, rows, 1),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": kind,
                         "sample": f"cumulants_upto(X[:{rows}], {cfg.m}, b={cfg.b}, engine={eng!r}); "
                                   f"calibration {', '.join(f'{k}={v:.2f}s' for k, v in times.items())}"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU (ours)


def main():
    args = parse()
    cfg = workloads.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return

    import torch
    import torch.distributed as dist

    import paper_1701_05420_b200 as bcg
    from paper_1701_05420_b200 import _native
    from paper_1701_05420_b200.cumulants import cumulants_device
    from paper_1701_05420_b200.distributed import cumulants_upto_sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    t_local = args.t or cfg.t
    t_total = t_local * world
    x_host = workloads.generate(cfg.name, t_local, shard=rank)
    X = torch.from_numpy(x_host).cuda()
    x_pinned = torch.from_numpy(x_host).pin_memory()
    flops_total = workloads.moment_flops(t_total, cfg.n, cfg.b, cfg.m)
    S_top = workloads.stored_elements(cfg.n, cfg.m, cfg.b)
    top_flops_local = 2.0 * t_local * S_top

    def barrier():
        if world > 1:
            dist.barrier()

    def step_device(timer=None):
        if world > 1:
            return cumulants_upto_sharded(X, cfg.m, cfg.b, timer=timer)
        return cumulants_device(X, cfg.m, cfg.b, c1_host=False, timer=timer)

    def step_e2e():
        if world > 1:
            mean, ts = cumulants_upto_sharded(x_pinned, cfg.m, cfg.b)
            return [mean.cpu()] + [t.cpu() for t in ts]
        cs = bcg.cumulants_upto(x_pinned, cfg.m, b=cfg.b)
        return [cs[1]] + [cs[k].packed_host() for k in range(2, cfg.m + 1)]

    def timed(fn, steps, timer=None):
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn(timer) if timer is not None else fn()
        e1.record()
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            v = torch.tensor([ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(v, op=dist.ReduceOp.MAX)
            ms = float(v.item())
        return ms

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()

    launches0 = _native.launch_count()
    with ClockSampler(local) as clk:
        ms = timed(step_device, args.steps)
    launches = _native.launch_count() - launches0
    # roofline of the dominant kernel: the top-order GEMM timed with events on
    # its stream in the serial schedule (orders one after the other, as in the
    # ncu launch list), so no other GEMM shares the GPU during its launch
    timer: dict = {}
    timed(step_device, max(2, min(5, args.steps)), timer)
    kern_ms = [a.elapsed_time(b) for a, b in timer.get("moment_top", [])]
    kern_avg = sum(kern_ms) / len(kern_ms) if kern_ms else float("nan")
    achieved = top_flops_local / (kern_avg / 1e3) / 1e12

    e2e = None
    if not args.no_e2e:
        for _ in range(max(1, args.warmup // 2)):
            step_e2e()
        e2e_steps = max(3, args.steps // 2)
        ms_e2e = timed(step_e2e, e2e_steps)
        d2h = 8 * (cfg.n + sum(workloads.stored_elements(cfg.n, k, cfg.b) for k in range(2, cfg.m + 1)))
        e2e = {"value": flops_total / (ms_e2e / 1e3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": int(x_host.nbytes), "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
               "api": "paper_1701_05420_b200.cumulants_upto(pinned host tensor) + packed_host() per order"}

    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg.name}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, cpu_sample_rows(cfg, args.cpu_sample_rows))

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": flops_total / (ms / 1e3) / 1e12,
            "unit": "TFLOP/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": f"synthetic ({cfg.name} recipe, workloads.py; seeded PCG64), resident in HBM",
            "config": config_dict(cfg, t_total, world),
            "roofline": {
                "bound": "tensor", "kernel": f"k_moment_dmma (order {cfg.m}, incl. split-K reduce)",
                "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                "algorithmic_flops_per_launch": top_flops_local, "avg_launch_ms": kern_avg,
                "peak_source": FP64_PEAK_SOURCE,
            },
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
