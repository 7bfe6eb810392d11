"""Small driver for ncu captures: `steps` cumulants_upto passes (device-resident)
on a config recipe at a reduced t, or only the top-order moment (--moment-only).

    python tools/prof_step.py --config cfg2 --t 200000 --steps 2 [--moment-only]
"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1701_05420_b200.cumulants import cumulants_device  # noqa: E402
from paper_1701_05420_b200.moments import _moment_device, center  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--t", type=int, default=0)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--order", type=int, default=0)
    ap.add_argument("--moment-only", action="store_true")
    a = ap.parse_args()
    cfg = workloads.CONFIGS[a.config]
    x = torch.from_numpy(workloads.generate(cfg.name, a.t or cfg.t)).cuda()
    order = a.order or cfg.m
    if a.moment_only:
        xc = center(x)
        for _ in range(a.steps):
            _moment_device(xc, order, cfg.b)
    else:
        for _ in range(a.steps):
            cumulants_device(x, cfg.m, cfg.b, c1_host=False)
    torch.cuda.synchronize()
    # plain timing (not meaningful under ncu)
    t0 = time.perf_counter()
    if a.moment_only:
        _moment_device(xc, order, cfg.b)
    else:
        cumulants_device(x, cfg.m, cfg.b, c1_host=False)
    torch.cuda.synchronize()
    print(f"one pass {1e3 * (time.perf_counter() - t0):.1f} ms")


if __name__ == "__main__":
    main()
