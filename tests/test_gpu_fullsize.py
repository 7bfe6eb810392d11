"""Parity at BASELINE.json's full sizes (cfg2 t=1e6 n=64 b=8 C2..C4, cfg3
t=2e6 n=48 b=4 C2..C5, cfg4 t=1e6 n=36 b=3 C2..C6), where the CPU reference
cannot run, through size-independent properties:

* power-of-two scaling is exact in binary floating point, so
  C_k(2 X) == 2^k C_k(X) BITWISE for every element of every order (centering,
  Khatri-Rao products, DMMA sums, split-K adds, the recursion all commute
  with it);
* translation invariance C_k(X + c) = C_k(X), k >= 2 (to rounding);
* sampled blocks of the top-order moment M_m of the centered data against an
  independent host computation (numpy Khatri-Rao columns + BLAS GEMM over all
  t samples), the reference's gram engine formulation (bc/_engines.py:141-208).
"""

import numpy as np
import pytest

import paper_1701_05420_b200 as bcg
import workloads
from paper_1701_05420_b200.layout import layout

pytestmark = pytest.mark.gpu

_CFGS = ["cfg2", "cfg3", "cfg4"]
_cache: dict = {}


def _data(name):
    if name not in _cache:
        _cache.clear()  # one full-size matrix at a time (cfg3 is 768 MB)
        cfg = workloads.CONFIGS[name]
        x = workloads.generate(name)
        cs = bcg.cumulants_upto(x, cfg.m, b=cfg.b)
        _cache[name] = (cfg, x, cs)
    return _cache[name]


@pytest.mark.parametrize("name", _CFGS)
def test_fullsize_power_of_two_scaling_is_bitwise(name):
    cfg, x, cs = _data(name)
    cs2 = bcg.cumulants_upto(2.0 * x, cfg.m, b=cfg.b)
    np.testing.assert_array_equal(cs2[1], 2.0 * cs[1])
    for k in range(2, cfg.m + 1):
        np.testing.assert_array_equal(cs2[k].packed_host(), (2.0 ** k) * cs[k].packed_host(), err_msg=f"C{k}")


@pytest.mark.parametrize("name", _CFGS)
def test_fullsize_translation_invariance(name):
    cfg, x, cs = _data(name)
    shift = np.linspace(-3.0, 3.0, cfg.n)
    cs_s = bcg.cumulants_upto(x + shift, cfg.m, b=cfg.b)
    np.testing.assert_allclose(cs_s[1], cs[1] + shift, rtol=1e-12, atol=1e-12)
    for k in range(2, cfg.m + 1):
        want = cs[k].packed_host()
        scale = float(np.max(np.abs(want)))
        np.testing.assert_allclose(cs_s[k].packed_host(), want, rtol=1e-9, atol=1e-11 * scale, err_msg=f"C{k}")


def _host_block(xc, key, b, h):
    """M[key] of centered data: Khatri-Rao columns of the first h modes and of
    the rest, one GEMM over all samples, / t (row-major block order)."""
    def kr(modes):
        w = np.ones((xc.shape[0], 1))
        for j in modes:
            cols = xc[:, (j - 1) * b: j * b]
            w = (w[:, :, None] * cols[:, None, :]).reshape(xc.shape[0], -1)
        return w

    return (kr(key[:h]).T @ kr(key[h:])).ravel() / xc.shape[0]


@pytest.mark.parametrize("name", _CFGS)
def test_fullsize_top_moment_blocks_match_host_gemm(name):
    cfg, x, _ = _data(name)
    xc = x - x.mean(axis=0)
    m, b = cfg.m, cfg.b
    mt = bcg.moment(xc, m, b=b)  # validates and centers-checks on the device, like the reference
    flat = mt.packed_host()
    lay = layout(cfg.n, m, b)
    rng = np.random.default_rng(11)
    picks = sorted({0, lay.K - 1, *rng.integers(0, lay.K, 3).tolist()})
    for k in picks:
        key = lay.keys[k]
        got = flat[lay.offs[k]:lay.offs[k + 1]]
        want = _host_block(xc, key, b, m // 2)
        scale = float(np.max(np.abs(want)))
        np.testing.assert_allclose(got, want, rtol=1e-11, atol=1e-13 * scale, err_msg=f"{name} block {key}")


@pytest.mark.parametrize("name", _CFGS)
def test_fullsize_rerun_is_bitwise(name):
    """Deterministic reductions everywhere (fixed split-K slices, ordered
    partial sums, no float atomics, concurrent order schedule): a rerun at
    full size reproduces every element of every order bit for bit."""
    cfg, x, cs = _data(name)
    again = bcg.cumulants_upto(x, cfg.m, b=cfg.b)
    np.testing.assert_array_equal(again[1], cs[1])
    for k in range(2, cfg.m + 1):
        np.testing.assert_array_equal(again[k].packed_host(), cs[k].packed_host(), err_msg=f"C{k}")
