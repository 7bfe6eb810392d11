"""GPU dense-entry oracle (paper_1701_05420_b200/verify.py, csrc/dense.cu):
SURVEY §8 f row 4 -- verification beyond the reference's dense oracle, which
materialises n^m elements and stops at n^m <= 1e8 (bc/oracle.py:22-34).

* the dense oracle itself against the CPU oracle (oracle/oracle.py, pinned to
  the reference's golden vectors) on small data, all orders 2..6, and the
  reference's two-point known answer C_4 = -2 (pkg/tests/test_oracle.py:77-80);
* cumulants_upto at BASELINE.json's FULL sizes (cfg2 t=1e6, cfg3 t=2e6, cfg4
  t=1e6, every order) and the cfg5 layout (n=96, b=6) to order 6, against the
  oracle on sampled elements -- random tuples, tuples with a repeated index
  and all-equal tuples (diagonal blocks, symmetric fills).

Criterion: |got - want| <= 1e-9 * scale, scale = the sum of the absolute
values of the moment-cumulant formula's terms (the magnitude the cancellation
starts from), i.e. the north_star's 1e-9 relative error measured against the
quantities actually subtracted; the worst ratio is logged to
$BCG_HIGHORDER_LOG when set.
"""

import json
import math
import os

import numpy as np
import pytest

from paper_1701_05420_b200 import verify

torch = pytest.importorskip("torch")

TOL = 1e-9


def _scale(mom, m):
    s = np.zeros(mom.shape[0])
    for parts in verify.partitions_min2_masks(m):
        k = len(parts)
        term = float(math.factorial(k - 1)) * np.ones(mom.shape[0])
        for blk in parts:
            term = term * np.abs(mom[:, blk])
        s = s + term
    return s


def _log(record):
    path = os.environ.get("BCG_HIGHORDER_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(record) + "\n")


def test_partition_counts_and_gaussian_formula():
    # F(m): set partitions into blocks of size >= 2 (the reference's
    # partitions.py counts F(6) = 41, pkg/tests/test_partitions.py:115-172)
    assert [len(verify.partitions_min2_masks(m)) for m in range(2, 9)] == [1, 1, 4, 11, 41, 162, 715]
    # exact N(0,1) moments of one variable: every cumulant of order >= 3 vanishes
    gauss = {0: 1.0, 1: 0.0, 2: 1.0, 3: 0.0, 4: 3.0, 5: 0.0, 6: 15.0, 7: 0.0, 8: 105.0}
    for m in range(2, 9):
        mom = np.array([[gauss[bin(s).count("1")] for s in range(1 << m)]])
        assert verify.element_cumulants(mom, m)[0] == (1.0 if m == 2 else 0.0)


gpu = pytest.mark.gpu


def _cuda():
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("needs a CUDA device")


@gpu
def test_dense_oracle_matches_the_cpu_oracle():
    _cuda()
    from oracle import oracle as orc

    rng = np.random.default_rng(11)
    x = rng.exponential(1.0, size=(3000, 7)) ** 2 + rng.standard_normal((3000, 7))
    b = 3
    _, want = orc.cumulants_upto(x, 6, b)
    for k in range(2, 7):
        idx = verify.sample_tuples(7, k, 48, rng)
        mom = verify.subset_moments(x, idx)
        got = verify.element_cumulants(mom, k)
        ref = verify.packed_values(want[k], 7, b, idx)
        assert np.all(np.abs(got - ref) <= TOL * _scale(mom, k)), k


@gpu
def test_dense_oracle_two_point_known_answer():
    _cuda()
    # two-point +-1 data: C_4 = -2 (pkg/tests/test_oracle.py:77-80)
    x = np.tile(np.array([[1.0], [-1.0]]), (500, 3))
    mom = verify.subset_moments(x, np.array([[0, 0, 0, 0], [0, 1, 2, 1]]))
    np.testing.assert_allclose(verify.element_cumulants(mom, 4), [-2.0, -2.0], rtol=0, atol=1e-14)


def _check(name, x, cs, b, orders, count, seed):
    res = verify.check_cumulant_set(x, cs, b, count=count, seed=seed, orders=orders)
    rng = np.random.default_rng(seed)
    for k, (got, want) in res.items():
        idx = verify.sample_tuples(x.shape[1], k, count, rng)
        scale = _scale(verify.subset_moments(x, idx), k)
        ratio = float(np.max(np.abs(got - want) / (TOL * scale)))
        _log({"test": "dense_oracle", "case": name, "order": k, "elements": len(got),
              "worst_err_over_1e-9_scale": ratio})
        assert ratio <= 1.0, (name, k, ratio)


@gpu
@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_full_size_cumulants_match_the_dense_oracle(name):
    _cuda()
    import paper_1701_05420_b200 as bcg
    import workloads

    cfg = workloads.CONFIGS[name]
    x = torch.from_numpy(workloads.generate(name)).cuda()
    cs = bcg.cumulants_upto(x, cfg.m, b=cfg.b)
    _check(name, x, cs, cfg.b, range(2, cfg.m + 1), count=48, seed=5)


@gpu
def test_cfg5_layout_to_order_6_matches_the_dense_oracle():
    _cuda()
    import paper_1701_05420_b200 as bcg
    import workloads

    x = torch.from_numpy(workloads.generate("cfg5", 65536)).cuda()  # n = 96, b = 6, Student-t copula
    cs = bcg.cumulants_upto(x, 6, b=6)
    _check("cfg5@t=65536", x, cs, 6, range(2, 7), count=48, seed=6)
