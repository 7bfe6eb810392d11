"""Summarise an ncu report (`--set full`) into the few lines we track.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/<round>_<name>.txt
"""

import csv
import io
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 (DMUL/DFMA) pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__sass_inst_executed_op_shared_ld.sum", "shared loads (inst)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        print(f"kernel: {d.get('Kernel Name', '?')[:100]}")
        for k, label in KEYS:
            if k in d:
                print(f"  {label:34s} {d[k]} {u.get(k, '')}")
        stalls = {h.split("stalled_")[1]: float(v) for h, v in d.items()
                  if re.match(r"smsp__pcsamp_warps_issue_stalled_[a-z_]+$", h) and not h.endswith("not_issued")
                  and v not in ("", None)}
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
        print("  stall samples: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1])
