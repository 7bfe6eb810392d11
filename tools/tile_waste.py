"""Where the moment plans' tile waste sits (host-only): valid pairs vs tiled
area, and how much of the waste is whole empty 8 x 8 DMMA sub-tiles / 32 x 32
warp tiles (what a sub-tile skip could save).

    python tools/tile_waste.py
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1701_05420_b200 import _native  # noqa: E402

lib = _native.lib()
for name, (n, b, m) in {"cfg2": (64, 8, 4), "cfg3": (48, 4, 5), "cfg4": (36, 3, 6), "cfg4 o5": (36, 3, 5), "cfg5": (96, 6, 6)}.items():
    p = ctypes.c_void_p()
    _native.check(lib.bcg_plan_create_host(n, m, b, ctypes.byref(p)))
    out = (ctypes.c_int64 * 5)()
    lib.bcg_plan_waste(p, out)
    S, prod = ctypes.c_int64(), ctypes.c_int64()
    lib.bcg_plan_output(p, ctypes.byref(S), ctypes.byref(prod))
    t = out[0]
    print(f"{name} order {m}: tiled {t:,} produced {prod.value:,} ({prod.value / t:.3f}) valid pairs {out[1]:,} ({out[1] / t:.3f}) "
          f"empty 8x8 {out[2] / t:.3f}  empty 32x32 {out[3] / t:.3f}  overhang {out[4] / t:.3f}")
    lib.bcg_plan_destroy(p)
