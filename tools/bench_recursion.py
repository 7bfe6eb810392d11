"""Time the cumulant recursion (K3) on the BASELINE configs' block layouts.

The recursion is t-independent: lower cumulants come from a small-t sample of
the recipe; M_m is a synthetic packed buffer of the right size.  Reports
algorithmic bytes (16 S_m + 8 sum_{j<=m-2} S_j, SURVEY §8 d) / time against
the measured HBM copy bandwidth (MEASURED_PEAKS.json hbm_gbs).  L2 is
flushed (512 MB write) before every timed launch."""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1701_05420_b200.cumulants import cumulants_device, _recursion_inplace  # noqa: E402
from paper_1701_05420_b200.symtensor import BlockSymTensor  # noqa: E402


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["cfg2", "cfg3", "cfg4"])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--copy-ref", action="store_true", help="also time a same-size device copy (the HBM ceiling at this size)")
    a = ap.parse_args()
    peak, src = hbm_peak()
    for name in a.configs:
        cfg = workloads.CONFIGS[name]
        m = cfg.m
        x = torch.from_numpy(workloads.generate(name, 4096)).cuda()
        _, lower = cumulants_device(x, m - 1, cfg.b, c1_host=False)
        lower = lower[: m - 3]  # C_2 .. C_{m-2}
        central = {t.m: t.data.clone() for t in lower if t.m >= 4}  # stand-in central moments
        S = workloads.stored_elements(cfg.n, m, cfg.b)
        base = torch.randn(S, dtype=torch.float64, device="cuda")
        alg = 16 * S + 8 * sum(workloads.stored_elements(cfg.n, j, cfg.b) for j in range(2, m - 1))
        label = "partition" if os.environ.get("BCG_RECURSION_PARTITION") else "factored"
        for env in (None,):
            if env:
                os.environ["BCG_RECURSION_PARTITION"] = env
            mk = BlockSymTensor(cfg.n, m, cfg.b, data=base.clone())
            _recursion_inplace(mk, lower, central)  # warm-up (+ plan)
            # back-to-back launches through the C ABI with prebuilt arguments
            # (in place: values change between launches, the work does not)
            import ctypes
            from paper_1701_05420_b200 import _native
            from paper_1701_05420_b200.layout import layout
            plan = _native.plan(cfg.n, m, cfg.b)
            lo = (ctypes.c_void_p * 15)()
            cm = (ctypes.c_void_p * 15)()
            for t in lower:
                lo[t.m - 2] = t.data.data_ptr()
            for k, v in central.items():
                cm[k - 2] = v.data_ptr()
            mk = base.clone()
            K = layout(cfg.n, m, cfg.b).K
            fn = _native.lib().bcg_cumulant_recursion_ex
            s = _native.stream_handle()
            fn(plan.handle, mk.data_ptr(), lo, cm, 0, K, s)
            flush = torch.empty(512 * 2**20 // 8, dtype=torch.float64, device="cuda")  # > L2 (126 MB)
            ts = []
            for _ in range(a.reps):
                flush.fill_(1.0)  # evict L2; keeps the GPU busy while the launch below is queued
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn(plan.handle, mk.data_ptr(), lo, cm, 0, K, s)
                e1.record()
                ts.append((e0, e1))
            torch.cuda.synchronize()
            ms = sorted(x.elapsed_time(y) for x, y in ts)[len(ts) // 2]
            gbs = alg / (ms / 1e3) / 1e9
            # copy ceiling: a device copy of the same S_m doubles (16 S_m bytes),
            # timed the same way (L2 flushed, one launch between two events)
            if a.copy_ref:
                src_buf = base
                dst_buf = torch.empty_like(base)
                cts = []
                for _ in range(a.reps):
                    flush.fill_(1.0)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    dst_buf.copy_(src_buf)
                    e1.record()
                    cts.append((e0, e1))
                torch.cuda.synchronize()
                cms = sorted(x.elapsed_time(y) for x, y in cts)[len(cts) // 2]
                copy_note = (f"; same-size copy {cms * 1e3:.1f} us = {100 * 16 * S / (cms / 1e3) / 1e9 / peak:.1f}%"
                             f" -> recursion at {100 * cms / ms:.0f}% of copy speed")
                del dst_buf
            else:
                copy_note = ""
            print(f"{name} m={m} S_m={S} recursion[{label}] {ms * 1e3:9.1f} us  {gbs:8.1f} GB/s "
                  f"= {100 * gbs / peak:5.1f}% of {peak:.0f} GB/s ({src}){copy_note}", flush=True)
        os.environ.pop("BCG_RECURSION_PARTITION", None)


if __name__ == "__main__":
    main()
