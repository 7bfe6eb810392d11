"""Turn an ncu launch list with DRAM metrics of `tools/prof_step.py --moment-only
--steps 1` (two identical top-order moment passes) into
profiles/ncu_traffic_<cfg>.json, the `roofline.traffic` bench.py reports:

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        --clock-control none -k regex:'k_moment_dmma|k_reduce_slices|k_sym_fill' --csv \\
        --log-file gpurun_out/traffic_<cfg>.csv python tools/prof_step.py --config <cfg> --moment-only --steps 1
    python tools/traffic_json.py <cfg> gpurun_out/traffic_<cfg>.csv
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    cfg, path = sys.argv[1], sys.argv[2]
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = {}
    order = []
    iid = hdr.index("ID")
    for r in rows[1:]:
        key = r[iid]
        if key not in per:
            per[key] = {"kernel": r[ik]}
            order.append(key)
        per[key][r[im]] = float(r[iv].replace(",", ""))
    launches = [per[k] for k in order]
    tot = lambda name, sel=lambda k: True: sum(l.get(name, 0.0) for l in launches if sel(l["kernel"]))  # noqa: E731
    passes = 2
    rd, wr = tot("dram__bytes_read.sum") / passes, tot("dram__bytes_write.sum") / passes
    gemm = lambda k: "k_moment_dmma" in k  # noqa: E731
    out = {
        "plan": "canonical",
        "kernel": "top-order k_moment_dmma launches + k_reduce_slices + k_sym_fill of one moment pass "
                  "(what bench.py's avg_launch_ms brackets)",
        "source": f"ncu dram__bytes_read/write.sum over tools/prof_step.py --config {cfg} --moment-only --steps 1, "
                  f"2 passes averaged ({os.path.basename(path)})",
        "launches_per_pass": len(launches) // passes,
        "dram_bytes_read": int(rd), "dram_bytes_write": int(wr), "dram_bytes_per_launch": int(rd + wr),
        "gemm_dram_bytes_read": int(tot("dram__bytes_read.sum", gemm) / passes),
        "gemm_dram_bytes_write": int(tot("dram__bytes_write.sum", gemm) / passes),
        "gpu_ms_per_pass": tot("gpu__time_duration.sum") / passes / 1e6,
    }
    with open(os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
