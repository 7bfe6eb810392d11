"""Time the order-m moment GEMM of the bench configs under several plan
settings (environment knobs read when a plan is built: BCG_TILE=TMxTN,
BCG_NO_HYBRID=1), checking every setting bitwise against the
first on the same data.

    python tools/tune_moment.py --configs cfg2 cfg3 --settings "" BCG_TILE=16x128 [--t 0] [--order 0]
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1701_05420_b200.moments import _moment_device, center  # noqa: E402

KNOBS = ("BCG_TILE", "BCG_NO_HYBRID")


def apply(setting):
    for k in KNOBS:
        os.environ.pop(k, None)
    for kv in setting.split(","):
        if kv:
            k, v = kv.split("=")
            os.environ[k] = v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--settings", nargs="+", default=[""])
    ap.add_argument("--configs", nargs="+", default=["cfg2", "cfg3", "cfg4"])
    ap.add_argument("--t", type=int, default=0)
    ap.add_argument("--order", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    for name in a.configs:
        cfg = workloads.CONFIGS[name]
        t = a.t or cfg.t
        m = a.order or cfg.m
        xc = center(torch.from_numpy(workloads.generate(name, t)).cuda())
        flops = 2.0 * t * workloads.stored_elements(cfg.n, m, cfg.b)
        ref = None
        for st in a.settings:
            apply(st)
            out = _moment_device(xc, m, cfg.b).data  # warm-up + plan
            if ref is None:
                ref = out.clone()
            diff = int((out != ref).sum())
            err = float(((out - ref).abs() / ref.abs().clamp_min(1e-300)).max())
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                _moment_device(xc, m, cfg.b)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = min(ts)
            print(f"{name} m={m} t={t} [{st or 'default'}]: {ms:9.2f} ms  {flops / ms / 1e9:6.2f} TFLOP/s "
                  f"({100 * flops / ms / 1e9 / 37.1:5.1f}% of 37.1)  vs first: {diff} differ, max rel {err:.1e}",
                  flush=True)
        apply("")


if __name__ == "__main__":
    main()
