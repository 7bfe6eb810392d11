"""In-tree build of the native library (nvcc, sm_100a) -> libbcgpu.so.

The .so is git-ignored but travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbcgpu.so")
SOURCES = ["plan.cu", "moment.cu", "elementwise.cu", "recursion.cu", "recursion_fact.cu", "recursion_stream.cu", "dense.cu", "capi.cu"]
# moment.cu is compiled once per part: part 0 = host code + dispatch, parts
# 1..6 = the kernel instantiations of one CTA tile shape each (parallel nvcc)
# (recursion_fact.cu likewise: part 0 = dispatch, 1..6 = (m, b) instantiations)
PARTS = {"moment.cu": ("BCG_MOMENT_PART", 9), "recursion_fact.cu": ("BCG_RF_PART", 7)}
UNITS = [(s, []) for s in SOURCES if s not in PARTS] + [
    (s, [f"-D{d}={k}"]) for s, (d, n) in PARTS.items() for k in range(n)]
HEADERS = ["plan.h", "kernels.h", "kr.cuh", "rf_terms.cuh"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "bcgpu.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


DEBUG_LIB = os.path.join(HERE, "libbcgpu_checks.so")


def build(force: bool = False, verbose: bool = False, checks: bool = False) -> str:
    """Compile the sources in parallel (one nvcc per .cu) and link libbcgpu.so.
    ``checks`` builds libbcgpu_checks.so with device bounds checks
    (-DBCG_CHECKS); select it at run time with BCG_LIB=checks."""
    out = DEBUG_LIB if checks else os.environ.get("BCG_BUILD_OUT", LIB)
    if not force and not checks and not _stale():
        return out
    from concurrent.futures import ThreadPoolExecutor

    nvcc = os.environ.get("NVCC", "nvcc")
    extra = (["-DBCG_CHECKS"] if checks else []) + os.environ.get("BCG_NVCC_EXTRA", "").split()
    tag = "chk" if checks else "rel"

    hdr_mtime = max(os.path.getmtime(d) for d in
                    [os.path.join(CSRC, f) for f in HEADERS] +
                    [os.path.join(os.path.dirname(HERE), "include", "bcgpu.h")])
    flags_key = " ".join(extra)

    def compile_one(unit):
        src, defs = unit
        obj = os.path.join(CSRC, f".{src}{''.join(defs)}.{tag}.o")
        stamp = obj + ".flags"
        # incremental: reuse an object newer than its source and every header,
        # built with the same extra flags
        if (os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read() == flags_key
                and os.path.getmtime(obj) > max(hdr_mtime, os.path.getmtime(os.path.join(CSRC, src)))):
            return obj
        cmd = [nvcc, *NVCC_FLAGS[:-1], *extra, *defs, "-c", "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd, cwd=CSRC)
        with open(stamp, "w") as f:
            f.write(flags_key)
        return obj

    # the slowest units (the kernel instantiations) first
    units = sorted(UNITS, key=lambda u: u[0] != "recursion_fact.cu" or u[1][0].endswith("=0"))
    with ThreadPoolExecutor(min(len(units), os.cpu_count() or 8)) as ex:
        objs = list(ex.map(compile_one, units))
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out + ".tmp", *objs],
                          cwd=CSRC)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    import sys

    print(build(force=True, verbose="-v" in sys.argv, checks="--checks" in sys.argv))  # force: relink, objects reused
