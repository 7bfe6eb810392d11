"""paper_1701_05420_b200.core_dropin against the reference's own compiled
module (blockcumulants._core, built from /root/reference into oracle/_ref by
oracle/build_ref.sh; the CPU oracle's restatement where it is absent): same
arguments, accumulate semantics, key ranges and errors (bc/_core.pyx:126-175)."""

import os
import sys

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _reference_core():
    path = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(path, "blockcumulants")):
        return None
    sys.path.insert(0, path)
    try:
        from blockcumulants import _core  # the unmodified reference's Cython kernel
        return _core
    except ImportError:
        return None
    finally:
        sys.path.remove(path)


@pytest.mark.parametrize("n,m,b,t", [(7, 4, 3, 513), (9, 3, 2, 1000), (5, 6, 2, 300), (12, 5, 4, 257)])
def test_moment_blocks_matches_reference_core(n, m, b, t, rng):
    from paper_1701_05420_b200 import core_dropin

    ref = _reference_core()
    x = rng.standard_normal((t, n))
    xt = np.ascontiguousarray(x.T)
    keys, col0, edges, offs = orc.block_layout(n, m, b)
    K = len(keys)
    got = np.zeros(int(offs[-1]))
    for k0, k1 in ((0, K // 3), (K // 3, K)):  # disjoint key ranges, like moment_parallel_blocks
        core_dropin.moment_blocks(xt, col0, edges, got, offs, k0, k1)
    want = np.zeros_like(got)
    if ref is not None:
        ref.moment_blocks(xt, col0, edges, want, offs, 0, K)
    else:
        want = orc.moment_raw_sums(x, m, b)
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)
    # accumulate semantics: a second full call adds the sums again
    core_dropin.moment_blocks(xt, col0, edges, got, offs, 0, K)
    np.testing.assert_allclose(got, 2 * want, rtol=1e-12, atol=1e-12)
    # a key range touches only its slice of out
    part = np.full_like(got, 7.0)
    core_dropin.moment_blocks(xt, col0, edges, part, offs, 1, 2)
    lo, hi = int(offs[1]), int(offs[2])
    assert np.all(part[:lo] == 7.0) and np.all(part[hi:] == 7.0)
    np.testing.assert_allclose(part[lo:hi], 7.0 + want[lo:hi], rtol=1e-12, atol=1e-12)


def test_moment_blocks_errors_match_reference(rng):
    from paper_1701_05420_b200 import core_dropin

    x = rng.standard_normal((50, 4))
    xt = np.ascontiguousarray(x.T)
    keys, col0, edges, offs = orc.block_layout(4, 3, 2)
    out = np.zeros(int(offs[-1]))
    with pytest.raises(ValueError, match="Buffer dtype mismatch"):
        core_dropin.moment_blocks(xt, col0.astype(np.int32), edges, out, offs, 0, len(keys))
    with pytest.raises(ValueError, match="C-contiguous"):
        core_dropin.moment_blocks(x.T, col0, edges, out, offs, 0, len(keys))
    wide = np.zeros((len(keys), 17), dtype=np.int64)
    with pytest.raises(ValueError, match="2 <= m <= 16"):
        core_dropin.moment_blocks(xt, wide, wide, out, offs, 0, len(keys))
    ref = _reference_core()
    if ref is not None:
        with pytest.raises(ValueError, match="2 <= m <= 16"):
            ref.moment_blocks(xt, wide, wide, out, offs, 0, len(keys))


def test_naive_moment4_matches_reference_core(rng):
    from paper_1701_05420_b200 import core_dropin

    x = rng.standard_normal((400, 5))
    xt = np.ascontiguousarray(x.T)
    got = np.ones((5, 5, 5, 5))
    core_dropin.naive_moment4(xt, got)
    ref = _reference_core()
    want = np.ones((5, 5, 5, 5))
    if ref is not None:
        ref.naive_moment4(xt, want)
    else:
        want += np.einsum("ta,tb,tc,td->abcd", x, x, x, x)
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-11)


def _reference_package():
    path = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(path, "blockcumulants")):
        return None
    sys.path.insert(0, path)
    try:
        import blockcumulants as bc  # the unmodified reference, built by oracle/build_ref.sh
        return bc
    except ImportError:
        return None
    finally:
        sys.path.remove(path)


@pytest.mark.parametrize("name,t,m", [("cfg2", 20000, 4), ("cfg3", 4000, 5), ("cfg4", 1500, 6)])
def test_live_differential_against_the_reference(name, t, m):
    """The unmodified reference's cumulants_upto run live on the same seeded
    BASELINE recipe rows as ours (bc/cumulants.py:173-193): every element of
    C1..Cm within the reference's own 1e-9 criterion."""
    import paper_1701_05420_b200 as bcg
    import workloads

    bc = _reference_package()
    if bc is None:
        pytest.skip("reference not built (oracle/build_ref.sh)")
    cfg = workloads.CONFIGS[name]
    x = workloads.generate(name, t)
    want = bc.cumulants_upto(x, m, b=cfg.b)
    got = bcg.cumulants_upto(x, m, b=cfg.b)
    np.testing.assert_allclose(got[1], want[1], rtol=1e-12, atol=1e-14)
    for k in range(2, m + 1):
        lay_keys = list(want[k].blocks)
        for key in lay_keys:
            np.testing.assert_allclose(got[k].blocks[key], want[k].blocks[key], rtol=1e-9, atol=1e-12,
                                       err_msg=f"{name} C{k} block {key}")


@pytest.mark.parametrize("name,t", [("cfg2", 20000), ("cfg4", 1500)])
def test_reference_runs_on_the_gpu_through_the_dropin(name, t, monkeypatch):
    """INTEGRATION.md A for real: the unmodified reference with its compiled
    module switched to core_dropin (the one-line change at bc/_engines.py:
    26-31) runs its own cumulants_upto(engine="compiled") and its threaded
    moment_parallel_blocks(p=4) (bc/moments.py:99-131, concurrent key ranges
    into one shared buffer) on the B200; results match the unpatched reference
    at 1e-9."""
    import workloads
    from paper_1701_05420_b200 import core_dropin

    bc = _reference_package()
    if bc is None:
        pytest.skip("reference not built (oracle/build_ref.sh)")
    cfg = workloads.CONFIGS[name]
    x = workloads.generate(name, t)
    want_cs = bc.cumulants_upto(x, cfg.m, b=cfg.b, engine="compiled")
    want_pb = bc.moment_parallel_blocks(x, cfg.m, cfg.b, p=4, engine="compiled")
    engines = sys.modules[bc.__name__ + "._engines"]
    calls = []

    class Counting:
        def moment_blocks(self, *a):
            calls.append(a[-2:])
            core_dropin.moment_blocks(*a)

        naive_moment4 = staticmethod(core_dropin.naive_moment4)

    monkeypatch.setattr(engines, "_core", Counting())
    got_cs = bc.cumulants_upto(x, cfg.m, b=cfg.b, engine="compiled")
    n_cs = len(calls)
    got_pb = bc.moment_parallel_blocks(x, cfg.m, cfg.b, p=4, engine="compiled")
    assert n_cs == cfg.m - 1 and len(calls) == n_cs + 4  # one call per order; p key ranges
    np.testing.assert_allclose(got_cs[1], want_cs[1], rtol=1e-12)
    for k in range(2, cfg.m + 1):
        for key, blk in want_cs[k].blocks.items():
            np.testing.assert_allclose(got_cs[k].blocks[key], blk, rtol=1e-9, atol=1e-12, err_msg=f"C{k} {key}")
    for key, blk in want_pb.blocks.items():
        np.testing.assert_allclose(got_pb.blocks[key], blk, rtol=1e-12, atol=1e-14, err_msg=f"M{cfg.m} {key}")


def test_moment_blocks_wide_data_accumulates(rng):
    """n above the moment kernel's one-stage limit (WIDE_N): the drop-in
    routes through the variable-group decomposition with the same
    accumulate semantics and key ranges (partial last block: 745 = 106 * 7 + 3)."""
    from paper_1701_05420_b200 import core_dropin

    n, m, b, t = 745, 2, 7, 150
    x = rng.standard_normal((t, n))
    xt = np.ascontiguousarray(x.T)
    keys, col0, edges, offs = (np.asarray(a) for a in orc.block_layout(n, m, b))
    col0 = np.ascontiguousarray(col0, dtype=np.int64)
    edges = np.ascontiguousarray(edges, dtype=np.int64)
    offs = np.ascontiguousarray(offs, dtype=np.int64)
    K = col0.shape[0]
    prior = rng.standard_normal(int(offs[-1]))
    out = prior.copy()
    k0, k1 = K // 3, K - 5
    core_dropin.moment_blocks(xt, col0, edges, out, offs, k0, k1)
    want = prior.copy()
    lo, hi = int(offs[k0]), int(offs[k1])
    want[lo:hi] += orc.moment_raw_sums(x, m, b, key_range=(k0, k1))[lo:hi]
    np.testing.assert_allclose(out, want, rtol=1e-12, atol=1e-11)
    np.testing.assert_array_equal(out[:lo], prior[:lo])
    np.testing.assert_array_equal(out[hi:], prior[hi:])
