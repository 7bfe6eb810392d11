"""Statistical and blocking properties of the GPU path, after the reference's
acceptance criteria and cumulant tests (pkg/tests/test_acceptance.py:109-125,
C4 Gaussian vanishing; pkg/tests/test_cumulants.py:200-207, Exp(1) C3 ~ 2),
plus block-size invariance: the same tensor comes out for every b.

The spread bound restates the reference's `element_std_bound`
(bc/stats.py:18-40): 5 * sqrt(mean(y^2) / t), y the product over the doubled
index, i.e. y^2 = prod_k x_{i_k}^4 on centered data.
"""

import itertools

import numpy as np
import pytest

import paper_1701_05420_b200 as bcg

pytestmark = pytest.mark.gpu


def _gaussian(n, t, seed):
    """Correlated Gaussian data as the reference's generator draws it
    (bc/dataio.py:108-147: random SPD covariance a a^T / n + I, Cholesky)."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n))
    cov = a @ a.T / n + np.eye(n)
    return rng.standard_normal((t, n)) @ np.linalg.cholesky(cov).T


def _bound(xc, index):
    y = np.ones(xc.shape[0])
    for i in index + index:
        y = y * xc[:, i - 1]
    return 5.0 * float(np.sqrt(np.mean(y * y) / xc.shape[0]))


def test_gaussian_cumulants_vanish():
    """Acceptance C4: C3 and C4 of Gaussian data lie within the 5x spread bound
    in at least 19 of 20 seeded runs at t = 1e6 (n = 3, b = 2)."""
    n, t, runs = 3, 1_000_000, 20
    failures = 0
    for seed in range(runs):
        x = _gaussian(n, t, seed)
        xc = x - x.mean(axis=0)
        cs = bcg.cumulants_upto(x, 4, b=2)
        ok = all(abs(cs[m].get(idx)) < _bound(xc, idx)
                 for m in (3, 4) for idx in itertools.combinations_with_replacement(range(1, n + 1), m))
        failures += 0 if ok else 1
    assert failures <= 1, f"{failures}/{runs} runs outside the 5x bound"


def test_gaussian_higher_cumulants_vanish():
    """The same through order 6 (the orders the reference's CPU path makes
    expensive): C3..C6 within the bound, 4 seeds, n = 3, b = 3."""
    n, t = 3, 1_000_000
    for seed in range(4):
        x = _gaussian(n, t, 100 + seed)
        xc = x - x.mean(axis=0)
        cs = bcg.cumulants_upto(x, 6, b=3)
        for m in range(3, 7):
            for idx in itertools.combinations_with_replacement(range(1, n + 1), m):
                assert abs(cs[m].get(idx)) < _bound(xc, idx), (seed, m, idx)


def test_exponential_third_cumulant():
    """Exp(1): kappa_3 = 2 within 5 sqrt(M6 / t) (test_cumulants.py:200-207)."""
    t = 400_000
    x = np.random.default_rng(5).exponential(1.0, (t, 2))
    xc = x - x.mean(axis=0)
    cs = bcg.cumulants_upto(x, 3, b=2)
    for i in (1, 2):
        tol = 5.0 * float(np.sqrt(np.mean(xc[:, i - 1] ** 6) / t))
        assert abs(cs[3].get((i, i, i)) - 2.0) < tol


def test_block_size_invariance(rng):
    """Every block size b gives the same moment and cumulant tensors (dense
    views agree to rounding), incl. b that do not divide n and b > n."""
    x = rng.exponential(1.0, (3000, 7)) + rng.standard_normal((3000, 7))
    ref = {m: t.to_dense() for m, t in enumerate(bcg.cumulants_upto(x, 5, b=1).tensors, start=2)}
    for b in (2, 3, 4, 6, 9):
        cs = bcg.cumulants_upto(x, 5, b=b)
        for m in range(2, 6):
            d = cs[m].to_dense()
            scale = float(np.max(np.abs(ref[m])))
            np.testing.assert_allclose(d, ref[m], rtol=1e-10, atol=1e-12 * scale, err_msg=f"b={b} m={m}")
