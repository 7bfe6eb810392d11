"""One timed cumulants_upto pass on a config recipe at a chosen t (device-
resident), with plan-build and memory figures -- used for cfg5-scale checks.

    python tools/run_cfg.py --config cfg5 --t 20000
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1701_05420_b200 import _native  # noqa: E402
from paper_1701_05420_b200.cumulants import cumulants_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--t", type=int, default=20000)
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    cfg = workloads.CONFIGS[a.config]
    m = a.m or cfg.m
    x = torch.from_numpy(workloads.generate(cfg.name, a.t)).cuda()
    t0 = time.perf_counter()
    for k in range(2, m + 1):
        _native.plan(cfg.n, k, cfg.b)
    print(f"plans built in {time.perf_counter() - t0:.2f} s")
    for rep in range(a.reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c1, ts = cumulants_device(x, m, cfg.b, c1_host=False)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        fl = workloads.moment_flops(a.t, cfg.n, cfg.b, m)
        ex = sum(2.0 * a.t * _native.plan(cfg.n, k, cfg.b).output()[1] for k in range(2, m + 1))
        print(f"{cfg.name} t={a.t} m={m}: {ms:.1f} ms, {fl / ms / 1e9:.2f} TFLOP/s reference-equivalent, "
              f"{ex / ms / 1e9:.2f} TFLOP/s executed ({100 * ex / ms / 1e9 / 37.1:.1f}% of the 37.1 TFLOP/s "
              f"DMMA peak, all orders), max mem {torch.cuda.max_memory_allocated() / 1e9:.1f} GB", flush=True)
    top = ts[-1].data
    print("C_m finite:", bool(torch.isfinite(top).all()), "elements", top.numel(),
          "checksum", float(top.abs().sum()))


if __name__ == "__main__":
    main()
