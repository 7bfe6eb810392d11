"""Stage-by-stage CUDA-event breakdown of one cumulants_upto pass, with and
without the nvidia-smi clock sampler, to locate non-kernel time."""

import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1701_05420_b200 import moments as M  # noqa: E402
from paper_1701_05420_b200 import cumulants as C  # noqa: E402


def staged(X, m, b, ev):
    def mark(name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        ev.append((name, e, time.perf_counter()))

    mark("start")
    st = M._colstats(X, mean=True, bad=True)
    mark("colstats")
    M._raise_if_nonfinite(X, st["bad"])
    mark("bad.item")
    Xc = M._center_device(X, st["mean"])
    mark("center")
    C._check_centered(Xc)
    mark("check_centered")
    ts = []
    for k in range(2, m + 1):
        Mk = M._moment_device(Xc, k, b)
        mark(f"moment{k}")
        if k >= 4:
            C._recursion_inplace(Mk, ts)
            mark(f"recursion{k}")
        ts.append(Mk)
    torch.cuda.synchronize()
    mark("end")


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    cfg = workloads.CONFIGS[name]
    X = torch.from_numpy(workloads.generate(name)).cuda()
    for _ in range(2):
        staged(X, cfg.m, cfg.b, [])
    for label in ("plain", "plain", "sampler"):
        proc = None
        if label == "sampler":
            proc = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm", "--format=csv", "-lms", "100"],
                                    stdout=subprocess.DEVNULL)
            time.sleep(0.3)
        ev = []
        staged(X, cfg.m, cfg.b, ev)
        if proc:
            proc.terminate()
        print(f"--- {label}: total gpu {ev[0][1].elapsed_time(ev[-1][1]):.2f} ms, wall {1e3 * (ev[-1][2] - ev[0][2]):.2f} ms")
        for (n0, e0, w0), (n1, e1, w1) in zip(ev[:-1], ev[1:]):
            print(f"  {n1:16s} gpu {e0.elapsed_time(e1):9.3f} ms   wall {1e3 * (w1 - w0):9.3f} ms")


if __name__ == "__main__":
    main()
