"""Tile efficiency of the moment plans (produced / tiled elements) for the
BASELINE configs' orders -- host-only plans, no GPU.

    python tools/tile_efficiency.py [BCG_NO_EDGE_TILES=1 to compare]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1701_05420_b200 import _native  # noqa: E402

lib = _native.lib()
for name, (n, b, mmax) in {"cfg2": (64, 8, 4), "cfg3": (48, 4, 5), "cfg4": (36, 3, 6), "cfg5": (96, 6, 6)}.items():
    for m in range(max(2, mmax - 2), mmax + 1):
        p = ctypes.c_void_p()
        _native.check(lib.bcg_plan_create_host(n, m, b, ctypes.byref(p)))
        S, prod, tiled, ne = (ctypes.c_int64() for _ in range(4))
        lib.bcg_plan_output(p, ctypes.byref(S), ctypes.byref(prod))
        lib.bcg_plan_tiled(p, ctypes.byref(tiled), ctypes.byref(ne))
        print(f"{name} order {m}: produced {prod.value:>13,} tiled {tiled.value:>13,} "
              f"efficiency {prod.value / tiled.value:.3f}  edge tiles {ne.value}")
        lib.bcg_plan_destroy(p)
