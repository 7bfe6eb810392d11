"""In-tree build of the native library (nvcc, sm_100a) -> libbcgpu.so.

The .so is git-ignored but travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbcgpu.so")
SOURCES = ["plan.cu", "moment.cu", "elementwise.cu", "recursion.cu", "recursion_fact.cu", "capi.cu"]
HEADERS = ["plan.h", "kernels.h", "kr.cuh"]
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

    def compile_one(src):
        obj = os.path.join(CSRC, f".{src}.{tag}.o")
        cmd = [nvcc, *NVCC_FLAGS[:-1], *extra, "-c", "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd, cwd=CSRC)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out + ".tmp", *objs],
                          cwd=CSRC)
    os.replace(out + ".tmp", out)
    for o in objs:
        os.remove(o)
    return out


if __name__ == "__main__":
    import sys

    print(build(force=True, verbose="-v" in sys.argv, checks="--checks" in sys.argv))
