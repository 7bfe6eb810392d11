"""The C-ABI library on a CPU-only host: it loads, exports every symbol the
header declares, and its host-built tables equal the reference's layout and
map every stored element exactly once (no GPU compute here)."""

import hashlib
import json
import os
import re

import numpy as np
import pytest

from paper_1701_05420_b200 import _native
from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "bcgpu.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(bcg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    bound = {name for name, _, _ in _native.SIGNATURES}
    assert set(syms) == bound, set(syms) ^ bound
    assert lib.bcg_version() == 100


def test_library_is_sm100a(tmp_path):
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("n,m,b", [(5, 3, 2), (7, 4, 3), (3, 3, 5), (2, 6, 1), (6, 6, 2), (24, 4, 4),
                                   (5, 2, 2), (9, 5, 4), (10, 1, 3)])
def test_native_layout_matches_reference(n, m, b, golden):
    g = golden("layout.npz")
    tag = f"{n}_{m}_{b}"
    plan = _native.Plan(n, m, b, host_only=True)
    keys, col0, edges, offs = plan.layout(m)
    np.testing.assert_array_equal(keys, g[f"keys_{tag}"])
    np.testing.assert_array_equal(col0, g[f"col0_{tag}"])
    np.testing.assert_array_equal(edges, g[f"edges_{tag}"])
    np.testing.assert_array_equal(offs, g[f"offs_{tag}"])


def test_native_layout_config_digests(golden):
    digests = json.loads(str(golden("layout.npz")["digests"]))
    plans = {}
    for tag, want in digests.items():
        n, m, b = map(int, tag.split("_"))
        top = max(int(t.split("_")[1]) for t in digests if t.startswith(f"{n}_") and t.endswith(f"_{b}"))
        plan = plans.setdefault((n, b), _native.Plan(n, top, b, host_only=True))
        keys, col0, edges, offs = plan.layout(m)
        h = hashlib.sha256()
        for a in (keys, col0, edges, offs):
            h.update(np.ascontiguousarray(a).tobytes())
        assert h.hexdigest() == want, tag


@pytest.mark.parametrize("n,m,b", [(4, 3, 2), (5, 4, 2), (5, 4, 3), (3, 5, 2), (6, 2, 4), (2, 6, 1),
                                   (3, 3, 5), (6, 6, 2), (7, 4, 3), (24, 4, 4), (64, 4, 8), (48, 5, 4),
                                   (36, 6, 3), (13, 7, 3), (11, 8, 5), (1, 3, 1), (100, 2, 7)])
@pytest.mark.parametrize("full", [False, True])
def test_gemm_mapping_selfcheck(n, m, b, full):
    plan = _native.Plan(n, m, b, host_only=True, full=full)
    _native.check(_native.lib().bcg_plan_selfcheck(plan.handle))
    S, produced = plan.output()
    assert S == orc.block_layout(n, m, b)[3][-1]
    assert produced == S if full else produced <= S


def _canonical_count(n, m, b):
    """Elements a symmetric plan's GEMM(s) produce: per key, the in-block
    offsets whose digits are non-decreasing within each run of equal block
    indices of the FULL key (runs that straddle the row | column split
    included) -- one per multiset of m variables, C(n+m-1, m) when b | n."""
    from itertools import combinations_with_replacement, groupby
    from math import comb

    nb = -(-n // b)
    edge = lambda j: min(j * b, n) - (j - 1) * b  # noqa: E731

    def part(t):
        r = 1
        for j, g in groupby(t):
            L = len(list(g))
            r *= comb(edge(j) + L - 1, L)
        return r

    return sum(part(k) for k in combinations_with_replacement(range(1, nb + 1), m))


@pytest.mark.parametrize("n,m,b", [(36, 6, 3), (64, 4, 8), (24, 4, 4), (7, 4, 3), (48, 5, 4), (13, 6, 4),
                                   (10, 5, 3), (20, 6, 6)])
def test_symmetric_plan_produced_count(n, m, b):
    # the GEMMs produce exactly the canonical elements (the multisets of m
    # variables); k_sym_fill copies the rest (cfg4: 49.8% of S_6, cfg2: 56.7%
    # of S_4)
    from math import comb

    plan = _native.Plan(n, m, b, host_only=True)
    S, produced = plan.output()
    assert produced == _canonical_count(n, m, b)
    if n % b == 0:
        assert produced == comb(n + m - 1, m)
    if (n, m, b) == (36, 6, 3):
        assert abs(produced / S - 0.498) < 1e-3
    _native.check(_native.lib().bcg_plan_selfcheck(plan.handle))


def test_hybrid_odd_order_plan():
    # odd orders split the keys by their middle entry into an (h | h+1) and an
    # (h+1 | h) GEMM when that tiles the staircase with less area; both parts
    # together must still produce every element once (selfcheck)
    plan = _native.Plan(48, 5, 4, host_only=True)
    T, parts = plan.gemms()
    assert T >= 2 and [(h, r) for h, r, *_ in parts] == [(2, 3), (3, 2)]
    assert plan.kernel()[3] == sum(p[4] for p in parts)
    _native.check(_native.lib().bcg_plan_selfcheck(plan.handle))
    # even orders keep the single balanced GEMM
    T, parts = _native.Plan(64, 4, 8, host_only=True).gemms()
    assert T == 0 and [(h, r) for h, r, *_ in parts] == [(2, 2)]


def test_plan_errors():
    from paper_1701_05420_b200 import ValidationError

    with pytest.raises(ValidationError, match="2 <= m <= 16"):
        _native.Plan(4, 17, 2, host_only=True)
    with pytest.raises(ValidationError):
        _native.Plan(0, 3, 2, host_only=True)


def test_native_partitions_match_python():
    # sub-key ranks: C++ multiset_rank vs Python key index, via the layout
    plan = _native.Plan(9, 6, 2, host_only=True)
    for k in range(2, 7):
        keys, _, _, _ = plan.layout(k)
        lay = orc.block_layout(9, k, 2)
        assert [tuple(r) for r in keys.tolist()] == lay[0]


def test_no_cpu_fallback_without_a_device():
    """The compute entry points fail loudly when no CUDA device is visible
    (there is no CPU fallback): run in a subprocess with CUDA hidden."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, numpy as np; sys.path.insert(0, %r)\n"
            "import paper_1701_05420_b200 as bcg\n"
            "try:\n"
            "    bcg.cumulants_upto(np.ones((10, 2)), 3, b=1)\n"
            "except bcg.NativeUnavailableError as e:\n"
            "    print('raised:', e)\n"
            "else:\n"
            "    print('no error')\n" % root)
    out = subprocess.run([sys.executable, "-c", code], env={**os.environ, "CUDA_VISIBLE_DEVICES": ""},
                         capture_output=True, text=True, timeout=300)
    assert "raised:" in out.stdout, out.stdout + out.stderr


def test_edge_tiles_cover_the_staircase_overhang():
    # band-edge tiles (tm x tn/2) where at most half a tile of columns remains:
    # cfg4's order-6 plan covers its 4.50M canonical elements with >= 0.90 of
    # the tiled area (0.88 without them), and every element exactly once
    import ctypes

    lib = _native.lib()
    plan = _native.Plan(36, 6, 3, host_only=True)
    tiled, edges = ctypes.c_int64(), ctypes.c_int64()
    _native.check(lib.bcg_plan_tiled(plan.handle, ctypes.byref(tiled), ctypes.byref(edges)))
    _, produced = plan.output()
    assert edges.value > 0 and produced / tiled.value >= 0.90
    _native.check(lib.bcg_plan_selfcheck(plan.handle))


def test_plan_waste_breakdown():
    """bcg_plan_waste (tools/tile_waste.py): the valid (row, column) pairs
    inside the tiles are exactly the produced elements, and most of the cover's
    waste at cfg4's order 6 is whole empty 8 x 8 DMMA sub-tiles."""
    import ctypes

    lib = _native.lib()
    plan = _native.Plan(36, 6, 3, host_only=True)
    out = (ctypes.c_int64 * 5)()
    _native.check(lib.bcg_plan_waste(plan.handle, out))
    tiled, edges = ctypes.c_int64(), ctypes.c_int64()
    _native.check(lib.bcg_plan_tiled(plan.handle, ctypes.byref(tiled), ctypes.byref(edges)))
    _, produced = plan.output()
    assert out[0] == tiled.value and out[1] == produced
    assert out[3] <= out[2] <= out[0] - out[1]          # empty warp tiles within empty sub-tiles within the waste
    assert 0.05 < out[2] / out[0] < 0.10 and out[4] <= out[0] - out[1]
