"""The shared-memory wavefront rule behind the streamed recursion's lane order
(tools/rs_wavefront_model.py) against what ncu measured on the B200
(profiles/r02_rs_wavefront_rule.txt, profiles/r02_rs_v7d_v8_v9_ncu.txt): the
numbers asserted here are the measured ones."""

import os
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import rs_wavefront_model as model  # noqa: E402


def _per_instruction(cfg):
    (lpf, wpe, nthr, tile), rows = model.evaluate(cfg["reg"], cfg["coords"], detail=True)
    hist = Counter()
    total = 0.0
    for _, _, _, loads, w in rows:
        hist[round(w, 2)] += loads
        total += loads * w
    return lpf, nthr, tile, hist, total


def test_v7d_matches_the_ncu_histogram():
    lpf, nthr, tile, hist, total = _per_instruction(model.V7D)
    assert (nthr, tile) == (96, 27)
    assert abs(lpf - 364 / 675) < 1e-12          # 364 factor loads for 675 FMAs per thread and unit
    # ncu, v7d: 157 loads x 1, 36 x 4/3, 171 x 2 wavefronts = 547 per warp and unit
    assert dict(hist) == {1.0: 157, 1.33: 36, 2.0: 171}
    assert abs(total - 547.0) < 1e-9
    assert model.ring_wavefronts(model.V7D["reg"], model.V7D["coords"]) == 2.0   # ncu: 27 ring loads x 2


def test_v8_lane_order_matches_ncu():
    _, _, _, hist, total = _per_instruction(model.V8)
    # ncu, v8: 317 loads x 1 + 47 x 2 = 411
    assert dict(hist) == {1.0: 317, 2.0: 47}
    assert abs(total - 411.0) < 1e-9
    assert model.ring_wavefronts(model.V8["reg"], model.V8["coords"]) == 4.0    # ncu: 27 ring loads x 4


def test_quad_rule_on_known_patterns():
    # 4 distinct doubles indexed by lane bits 0 and 1: two wavefronts (C2[i4, i5] in v7d)
    addrs = [8 * ((l & 1) + 6 * ((l >> 1) & 1)) for l in range(32)]
    assert model.lds_wavefronts(addrs) == 2
    # the same 4 doubles indexed by lane bits 0 and 2: one
    addrs = [8 * ((l & 1) + 6 * ((l >> 2) & 1)) for l in range(32)]
    assert model.lds_wavefronts(addrs) == 1
    # 32 distinct consecutive doubles: two (256 bytes)
    assert model.lds_wavefronts([8 * l for l in range(32)]) == 2
