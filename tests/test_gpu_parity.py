"""GPU parity: the sm_100a path against the reference's golden vectors and the
CPU oracle, on the same seeded inputs (tolerances as the reference's own tests:
moments rtol 1e-12 atol 1e-14, pkg/tests/test_moments.py:116-126; cumulants
rtol 1e-9 atol 1e-12, pkg/tests/test_acceptance.py:44-66)."""

import ctypes
import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1701_05420_b200 as bcg  # noqa: E402
from paper_1701_05420_b200 import _native  # noqa: E402
from oracle import oracle as orc  # noqa: E402
import workloads  # noqa: E402
from conftest import random_sym_dense  # noqa: E402


def packed(t):
    return t.packed_host()


# ---------------------------------------------------------------- moments


def test_moments_match_reference_golden(golden):
    g = golden("moments.npz")
    n_cases = 0
    for key in g.files:
        if not key.startswith("shape_"):
            continue
        i = key.split("_")[1]
        n, m, b, t = map(int, g[key])
        got = bcg.moment(g[f"x_{i}"], m, b)
        np.testing.assert_allclose(packed(got), g[f"m_{i}"], rtol=1e-12, atol=1e-14)
        n_cases += 1
    assert n_cases >= 11


@pytest.mark.parametrize("n,m,b,t", [(4, 3, 2, 100), (5, 4, 2, 60), (5, 4, 3, 60), (3, 5, 2, 40),
                                     (6, 2, 4, 200), (2, 6, 1, 30), (3, 3, 5, 50), (6, 6, 2, 300),
                                     (13, 7, 3, 77), (11, 8, 5, 40), (1, 3, 1, 5), (100, 2, 7, 33),
                                     (24, 4, 4, 5000), (17, 5, 4, 4097), (9, 3, 2, 1)])
def test_moment_matches_oracle(n, m, b, t, rng):
    x = rng.standard_normal((t, n))
    got = bcg.moment(x, m, b)
    want = orc.moment(x, m, b)
    np.testing.assert_allclose(packed(got), want, rtol=1e-12, atol=1e-14)


def test_moment_kat_two_sample():
    # pkg/tests/test_moments.py:71-76
    t = bcg.moment(np.array([[1.0, 2.0], [3.0, 4.0]]), 2, 2)
    np.testing.assert_array_equal(t.blocks[(1, 1)], [[5.0, 7.0], [7.0, 10.0]])


def test_moment_constant_and_ones():
    assert bcg.moment(np.full((2, 1), 2.0), 3, 1).blocks[(1, 1, 1)][0, 0, 0] == 8.0
    t = bcg.moment(np.ones((10, 4)), 2, 2)
    np.testing.assert_array_equal(t.blocks[(1, 2)], np.ones((2, 2)))


def test_moment_order1_is_means(rng):
    x = rng.standard_normal((40, 5))
    np.testing.assert_allclose(bcg.moment(x, 1, 2).to_dense(), x.mean(axis=0), rtol=1e-14)


def test_moment_dense_against_oracle_dense(rng):
    x = rng.standard_normal((120, 5))
    np.testing.assert_allclose(bcg.moment(x, 4, 2).to_dense(), orc.dense_moment(x, 4), rtol=1e-12, atol=1e-15)


def test_moment_deterministic_bitwise(rng):
    x = rng.standard_normal((20000, 12))
    a = packed(bcg.moment(x, 4, 3))
    b = packed(bcg.moment(x, 4, 3))
    np.testing.assert_array_equal(a, b)


def test_moment_block_matches(rng):
    x = rng.standard_normal((23, 5))
    blk = bcg.moment_block(x, (1, 2), 2)
    want = orc.moment(x, 2, 2)
    lay = orc.block_layout(5, 2, 2)
    k = lay[0].index((1, 2))
    np.testing.assert_allclose(blk.ravel(), want[lay[3][k]:lay[3][k + 1]], rtol=1e-13)
    with pytest.raises(bcg.ValidationError, match="not sorted"):
        bcg.moment_block(x, (2, 1), 2)


def test_moment_validation(rng):
    with pytest.raises(bcg.ValidationError, match="row 2, column 1"):
        bcg.as_data_matrix([[1.0, 2.0], [np.nan, 3.0]])
    with pytest.raises(bcg.ValidationError, match="2-D"):
        bcg.as_data_matrix([1.0, 2.0])
    with pytest.raises(bcg.ValidationError):
        bcg.moment(rng.standard_normal((5, 2)), 0)
    with pytest.raises(bcg.ValidationError):
        bcg.moment(rng.standard_normal((5, 2)), 2, 0)
    with pytest.raises(bcg.ValidationError, match="unknown engine"):
        bcg.moment(rng.standard_normal((5, 2)), 2, 2, engine="nope")
    x = rng.standard_normal((50, 7))
    x[31, 4] = np.inf
    with pytest.raises(bcg.ValidationError, match="row 32, column 5"):
        bcg.moment(x, 3, 2)


def test_moment_torch_input_stays_on_device(rng):
    x = torch.from_numpy(rng.standard_normal((300, 6))).cuda()
    t = bcg.moment(x, 3, 2)
    assert t.data.is_cuda
    np.testing.assert_allclose(packed(t), orc.moment(x.cpu().numpy(), 3, 2), rtol=1e-12, atol=1e-14)


def test_permutation_properties(rng):
    # pkg/tests/test_moments.py:134-149
    x = rng.standard_normal((80, 4))
    a = bcg.moment(x, 3, 2).to_dense()
    b = bcg.moment(x[rng.permutation(80)], 3, 2).to_dense()
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-15)
    perm = [2, 0, 3, 1]
    c = bcg.moment(x[:, perm], 3, 2).to_dense()
    np.testing.assert_allclose(c, a[np.ix_(perm, perm, perm)], rtol=1e-12, atol=1e-15)


# ---------------------------------------------------------------- parallel


def test_moment_parallel(rng):
    x = rng.standard_normal((101, 4))
    serial = bcg.moment(x, 4, 2)
    np.testing.assert_array_equal(packed(bcg.moment_parallel(x, 4, 2, p=1)), packed(serial))
    for p in (2, 3, 4, 7, 8):
        np.testing.assert_allclose(packed(bcg.moment_parallel(x, 4, 2, p=p)), packed(serial),
                                   rtol=1e-12, atol=1e-15)
    with pytest.raises(bcg.ValidationError, match="non-empty"):
        bcg.moment_parallel(rng.standard_normal((3, 2)), 2, 2, p=5)


def test_moment_parallel_equal_chunks_bitwise(rng):
    # pkg/tests/test_moments.py:171-184: equal chunks -> exactly (1/p) sum parts
    x = rng.standard_normal((100, 3))
    par = bcg.moment_parallel(x, 3, 2, p=4)
    parts = [bcg.moment(x[lo:lo + 25], 3, 2) for lo in (0, 25, 50, 75)]
    manual = parts[0].scale(0.25)
    for part in parts[1:]:
        manual = manual + part.scale(0.25)
    np.testing.assert_array_equal(packed(par), packed(manual))


@pytest.mark.parametrize("p", [1, 2, 3, 7])
def test_moment_parallel_blocks_bitwise(p, rng):
    x = rng.standard_normal((900, 9))
    np.testing.assert_array_equal(packed(bcg.moment_parallel_blocks(x, 4, 2, p=p)), packed(bcg.moment(x, 4, 2)))


# ---------------------------------------------------------------- drop-in ABI


def test_dropin_moment_blocks_matches_oracle(rng):
    """bcg_moment_blocks with the reference's own arguments (xt, col0, edges,
    out, offs, k0, k1) and accumulate semantics (bc/_core.pyx:126-148)."""
    lib = _native.lib()
    n, m, b, t = 7, 4, 3, 513
    x = rng.standard_normal((t, n))
    keys, col0, edges, offs = orc.block_layout(n, m, b)
    dxt = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
    dc0, de, do = (torch.from_numpy(a).cuda() for a in (col0, edges, offs))
    out = torch.zeros(int(offs[-1]), dtype=torch.float64, device="cuda")
    K = len(keys)
    s = _native.stream_handle()
    for k0, k1 in ((0, K // 3), (K // 3, K)):
        _native.check(lib.bcg_moment_blocks(dxt.data_ptr(), n, t, dc0.data_ptr(), de.data_ptr(), m, K,
                                            out.data_ptr(), do.data_ptr(), k0, k1, s))
    want = orc.moment_raw_sums(x, m, b)
    np.testing.assert_allclose(out.cpu().numpy(), want, rtol=1e-12, atol=1e-12)
    # accumulate: a second full call doubles the sums (verified on the reference)
    _native.check(lib.bcg_moment_blocks(dxt.data_ptr(), n, t, dc0.data_ptr(), de.data_ptr(), m, K,
                                        out.data_ptr(), do.data_ptr(), 0, K, s))
    np.testing.assert_allclose(out.cpu().numpy(), 2 * want, rtol=1e-12, atol=1e-12)
    rc = lib.bcg_moment_blocks(dxt.data_ptr(), n, t, dc0.data_ptr(), de.data_ptr(), 17, K,
                               out.data_ptr(), do.data_ptr(), 0, K, s)
    assert rc == 1 and b"2 <= m <= 16" in lib.bcg_last_error()


# ---------------------------------------------------------------- cumulants


def test_cumulants_match_reference_golden(golden):
    g = golden("cumulants.npz")
    cases = 0
    worst = 0.0
    for key in g.files:
        if not key.startswith("shape_"):
            continue
        i = key.split("_")[1]
        n, t, m_max, b = map(int, g[key])
        cs = bcg.cumulants_upto(g[f"x_{i}"], m_max, b=b)
        np.testing.assert_allclose(cs[1], g[f"c1_{i}"], rtol=1e-12, atol=1e-15)
        for k in range(2, m_max + 1):
            got, want = packed(cs[k]), g[f"c{k}_{i}"]
            np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-12)
            worst = max(worst, float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-3))))
        cases += 1
    assert cases >= 24
    print(f"worst floored relative deviation vs reference: {worst:.2e}")


def test_cfg1_full_size_matches_reference(golden):
    g = golden("configs.npz")
    cfg = workloads.CONFIGS["cfg1"]
    x = workloads.generate("cfg1")
    np.testing.assert_allclose([x.sum(), (x * x).sum()], g["cfg1_xsum"], rtol=1e-12)
    cs = bcg.cumulants_upto(x, cfg.m, b=cfg.b)
    np.testing.assert_allclose(cs[1], g["cfg1_c1"], rtol=1e-12, atol=1e-15)
    for k in range(2, cfg.m + 1):
        flat = packed(cs[k])
        np.testing.assert_allclose(flat[g[f"cfg1_c{k}_idx"]], g[f"cfg1_c{k}_val"], rtol=1e-9, atol=1e-12)
        st = g[f"cfg1_c{k}_stats"]
        assert flat.size == int(st[2])
        np.testing.assert_allclose(flat.sum(), st[0], rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4", "cfg5"])
def test_config_shapes_match_reference(name, golden):
    g = golden("configs.npz")
    cfg = workloads.CONFIGS[name]
    x = g[f"{name}_x"]
    m_top = max(int(k.split("_")[1][1:]) for k in g.files if k.startswith(f"{name}_c") and k.endswith("_idx"))
    cs = bcg.cumulants_upto(x, m_top, b=cfg.b)
    np.testing.assert_allclose(cs[1], g[f"{name}_c1"], rtol=1e-12, atol=1e-15)
    for k in range(2, m_top + 1):
        flat = packed(cs[k])
        assert flat.size == int(g[f"{name}_c{k}_stats"][2])
        np.testing.assert_allclose(flat[g[f"{name}_c{k}_idx"]], g[f"{name}_c{k}_val"], rtol=1e-9, atol=1e-12)


def test_cumulants_match_oracle_partial_edges(rng):
    x = rng.exponential(1.0, size=(700, 7)) + rng.standard_normal((700, 7))
    c1, want = orc.cumulants_upto(x, 6, 3)
    cs = bcg.cumulants_upto(x, 6, b=3)
    for k in range(2, 7):
        np.testing.assert_allclose(packed(cs[k]), want[k], rtol=1e-9, atol=1e-12)


def test_low_orders_bitwise_equal_central_moments(rng):
    # acceptance criterion 3 (pkg/tests/test_acceptance.py:91-106)
    data = rng.standard_normal((400, 5)) + rng.standard_normal(5)
    cs = bcg.cumulants_upto(data, 4, b=2)
    centered = bcg.center(data)
    for m in (2, 3):
        np.testing.assert_array_equal(packed(cs[m]), packed(bcg.moment(centered, m, b=2)))


def test_order4_matches_direct_pairings(rng):
    x = rng.standard_normal((500, 3)) ** 3
    xc = x - x.mean(axis=0)
    m4 = orc.dense_moment(xc, 4)
    cov = xc.T @ xc / x.shape[0]
    m4 -= np.einsum("ab,cd->abcd", cov, cov) + np.einsum("ac,bd->abcd", cov, cov) + np.einsum("ad,bc->abcd", cov, cov)
    np.testing.assert_allclose(bcg.cumulants_upto(x, 4, b=2)[4].to_dense(), m4, rtol=1e-10, atol=1e-12)


def test_constant_data_exact_zeros():
    x = np.tile([2.0, -1.0, 0.5], (20, 1))
    cs = bcg.cumulants_upto(x, 4, b=2)
    np.testing.assert_array_equal(cs[1], [2.0, -1.0, 0.5])
    for k in (2, 3, 4):
        assert cs[k].max_abs() == 0.0


def test_two_point_c4():
    cs = bcg.cumulants_upto(np.array([[-1.0], [1.0]] * 5), 4, b=1)
    assert cs[4].get((1, 1, 1, 1)) == pytest.approx(-2.0, rel=1e-14)


def test_outer_prod_cum_identity_kat():
    # pkg/tests/test_cumulants.py:35-41
    c2 = bcg.BlockSymTensor.from_dense(np.eye(3), b=2)
    out = bcg.outer_prod_cum(4, 2, [c2])
    assert out.get((1, 1, 1, 1)) == 3.0
    assert out.get((1, 1, 2, 2)) == 1.0
    assert out.get((1, 2, 3, 3)) == 0.0
    assert out.get((1, 2, 3, 1)) == 0.0


@pytest.mark.parametrize("m", [4, 5, 6])
def test_outer_prod_cum_matches_oracle(m, rng):
    n, b = 5, 2
    lower = {k: bcg.BlockSymTensor.from_dense(random_sym_dense(n, k, rng), b) for k in range(2, m - 1)}
    flats = {k: t.packed_host() for k, t in lower.items()}
    for sigma in range(2, m // 2 + 1):
        got = bcg.outer_prod_cum(m, sigma, list(lower.values()))
        # same float ops in the same order as the reference einsum loop
        np.testing.assert_allclose(packed(got), orc.outer_prod_cum(m, sigma, flats, n, b), rtol=1e-14, atol=1e-15)


def test_recursion_errors(rng):
    x = bcg.center(rng.standard_normal((50, 3)))
    with pytest.raises(bcg.ValidationError, match="missing lower cumulant"):
        bcg.cumulant(x, 4, [], b=2)
    with pytest.raises(bcg.ValidationError, match="not centered"):
        bcg.cumulant(rng.standard_normal((50, 3)) + 5.0, 3, [], b=2)
    c2 = bcg.BlockSymTensor.from_dense(random_sym_dense(2, 2, rng), b=2)
    with pytest.raises(bcg.ValidationError, match="order 3"):
        bcg.outer_prod_cum(6, 2, [c2])
    with pytest.raises(bcg.ValidationError):
        bcg.outer_prod_cum(4, 3, [c2])
    with pytest.raises(bcg.ValidationError):
        bcg.cumulants_upto(rng.standard_normal((30, 2)), 13)
    with pytest.raises(bcg.ValidationError, match="two samples"):
        bcg.cumulants_upto(np.ones((1, 3)), 2)


def test_super_symmetry_of_results(rng):
    x = rng.standard_normal((150, 4))
    cs = bcg.cumulants_upto(x, 5, b=2)
    for m in range(2, 6):
        for _ in range(100):
            index = tuple(rng.integers(1, 5, size=m))
            permuted = tuple(index[q] for q in rng.permutation(m))
            assert cs[m].get(index) == cs[m].get(permuted)


def test_shift_invariance(rng):
    x = rng.standard_normal((800, 3))
    a = bcg.cumulants_upto(x, 5, b=2)
    b = bcg.cumulants_upto(x + np.array([5.0, -3.0, 10.0]), 5, b=2)
    for k in range(2, 6):
        da, db = packed(a[k]), packed(b[k])
        assert np.max(np.abs(da - db)) <= 1e-9 * max(np.max(np.abs(da)), 1e-12)


def test_cumulants_deterministic(rng):
    x = rng.standard_normal((5000, 10))
    a = bcg.cumulants_upto(x, 5, b=3)
    b = bcg.cumulants_upto(x, 5, b=3)
    for k in range(2, 6):
        np.testing.assert_array_equal(packed(a[k]), packed(b[k]))


def test_blocksymtensor_device_arithmetic(rng):
    u = bcg.BlockSymTensor.from_dense(random_sym_dense(5, 3, rng), 2)
    v = bcg.BlockSymTensor.from_dense(random_sym_dense(5, 3, rng), 2)
    np.testing.assert_array_equal((u + v).packed_host(), u.packed_host() + v.packed_host())
    np.testing.assert_array_equal((u - v).packed_host(), u.packed_host() - v.packed_host())
    np.testing.assert_array_equal(u.scale(0.3).packed_host(), u.packed_host() * 0.3)


def test_native_launches_counted(rng):
    before = _native.launch_count()
    bcg.cumulants_upto(rng.standard_normal((100, 4)), 4, b=2)
    assert _native.launch_count() > before


# ---------------------------------------------------------------- kernel variants


def test_moment_kernel_ragged_shapes_match_oracle(rng):
    for n, m, b, t in [(7, 4, 3, 1003), (13, 5, 2, 517), (9, 6, 2, 211), (24, 4, 4, 4099), (5, 2, 2, 70),
                       (30, 3, 4, 333)]:
        x = rng.standard_normal((t, n))
        np.testing.assert_allclose(packed(bcg.moment(x, m, b)), orc.moment(x, m, b), rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("n,m,b,t", [(9, 4, 3, 500), (8, 5, 2, 400), (7, 6, 1, 300), (6, 6, 2, 500), (12, 6, 3, 600),
                                     (7, 6, 3, 500), (10, 5, 4, 700)])
def test_factored_recursion_matches_oracle(n, m, b, t, rng):
    """K3 factored (full blocks) + partition kernel (partial-edge blocks) vs
    the oracle.  The kernel-vs-kernel A/B on the same moments is
    test_gpu_highorder.test_factored_recursion_matches_the_partition_sum."""
    x = rng.exponential(1.0, size=(t, n)) + rng.standard_normal((t, n))
    fact = bcg.cumulants_upto(x, m, b=b)
    _, want = orc.cumulants_upto(x, m, b)
    for k in range(2, m + 1):
        np.testing.assert_allclose(packed(fact[k]), want[k], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("tile", ["64x64", "16x128", "128x16", "32x64", "64x32", "32x32", "128x64", "64x128"])
def test_v1_tile_shapes_match_oracle_and_each_other(tile, monkeypatch, rng):
    """Every v1 CTA tile shape (BCG_TILE override of the plan's model choice)
    gives the oracle's moments and bitwise-identical results."""
    x = rng.standard_normal((20000, 13))
    monkeypatch.setenv("BCG_TILE", "64x64")
    ref = {m: packed(bcg.moment(x, m, 2)) for m in (2, 3, 4, 5)}
    monkeypatch.setenv("BCG_TILE", tile)
    for m in (2, 3, 4, 5):
        got = packed(bcg.moment(x, m, 2))
        np.testing.assert_array_equal(got, ref[m])
    for n, m, b, t in [(7, 4, 3, 1003), (13, 5, 2, 517), (9, 6, 2, 211), (30, 3, 4, 333)]:
        x2 = rng.standard_normal((t, n))
        np.testing.assert_allclose(packed(bcg.moment(x2, m, b)), orc.moment(x2, m, b), rtol=1e-12, atol=1e-14)


def _nccl_worker(rank, world, port, x, m, b, out, mode="samples"):
    import os

    import torch.distributed as dist

    from paper_1701_05420_b200.distributed import cumulants_upto_block_split, cumulants_upto_sharded, shard_bounds

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    if mode == "samples":
        lo, hi = shard_bounds(x.shape[0], world, rank)
        mean, ts = cumulants_upto_sharded(torch.from_numpy(x[lo:hi]).cuda(), m, b)
    else:
        mean, ts = cumulants_upto_block_split(torch.from_numpy(x).cuda(), m, b)
    np.savez(out, mean=mean.cpu().numpy(), **{f"c{k}": t.cpu().numpy() for k, t in enumerate(ts, 2)})
    dist.destroy_process_group()


def test_sharded_path_over_nccl_single_rank(tmp_path, rng):
    """distributed.py on the real CUDA ops + NCCL (world size 1 on this 1-GPU
    box; the 2-rank collective logic is covered with gloo in test_distributed)."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    x = rng.exponential(1.0, size=(3001, 9)) + rng.standard_normal((3001, 9))
    out = str(tmp_path / "r0.npz")
    mp.spawn(_nccl_worker, args=(1, port, x, 6, 2, out), nprocs=1, join=True)
    got = np.load(out)
    c1, want = orc.cumulants_upto(x, 6, 2)
    np.testing.assert_allclose(got["mean"], c1, rtol=1e-13)
    for k in range(2, 7):
        np.testing.assert_allclose(got[f"c{k}"], want[k], rtol=1e-9, atol=1e-12)


def test_block_split_path_over_nccl_single_rank_bitwise(tmp_path, rng):
    """The block-split multi-GPU mode on the real CUDA ops + NCCL (world size
    1 here) is bitwise identical to cumulants_upto (every key range of the
    moment kernel sums in the same order)."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    x = rng.exponential(1.0, size=(3001, 9)) + rng.standard_normal((3001, 9))
    out = str(tmp_path / "r0.npz")
    mp.spawn(_nccl_worker, args=(1, port, x, 6, 3, out, "blocks"), nprocs=1, join=True)
    got = np.load(out)
    cs = bcg.cumulants_upto(x, 6, b=3)
    np.testing.assert_array_equal(got["mean"], cs[1])
    for k in range(2, 7):
        np.testing.assert_array_equal(got[f"c{k}"], cs[k].packed_host())


_VARIANT_SHAPES = [(16, 4, 8, 300), (12, 5, 4, 400), (9, 6, 3, 300), (12, 6, 6, 200), (12, 5, 6, 300), (7, 6, 3, 250),
                   (10, 6, 5, 150), (8, 6, 4, 200)]


@pytest.mark.parametrize("env", [{"BCG_RF_VARIANT": "2", "BCG_RF_TILE": "-1"}, {"BCG_RF_VARIANT": "2", "BCG_RF_TILE": "0"},
                                 {"BCG_RF_VARIANT": "2", "BCG_RF_TILE": "1"}, {"BCG_RF_VARIANT": "3"},
                                 {"BCG_RF_VARIANT": "6"}, {"BCG_RF_VARIANT": "2", "BCG_RF_STEPS": "7"}, {}])
def test_recursion_variants_match_oracle(env, tmp_path):
    """Every factored-recursion kernel variant (the knobs are read once per
    process, so each runs in a subprocess) gives the oracle's cumulants,
    incl. b = 6 (wide register tile), b = 8, partial-edge blocks."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "c.npz"
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "import paper_1701_05420_b200 as bcg\n"
        "res = {}\n"
        "for i, (n, m, b, t) in enumerate(%r):\n"
        "    x = np.random.default_rng(i).exponential(1.0, (t, n)) + np.random.default_rng(100 + i).standard_normal((t, n))\n"
        "    cs = bcg.cumulants_upto(x, m, b=b)\n"
        "    for k in range(2, m + 1):\n"
        "        res[f'{i}_{k}'] = cs[k].packed_host()\n"
        "np.savez(%r, **res)\n" % (root, _VARIANT_SHAPES, str(out)))
    subprocess.run([sys.executable, "-c", code], check=True, env={**os.environ, **env}, timeout=600)
    got = np.load(out)
    for i, (n, m, b, t) in enumerate(_VARIANT_SHAPES):
        x = np.random.default_rng(i).exponential(1.0, (t, n)) + np.random.default_rng(100 + i).standard_normal((t, n))
        _, want = orc.cumulants_upto(x, m, b)
        for k in range(2, m + 1):
            np.testing.assert_allclose(got[f"{i}_{k}"], want[k], rtol=1e-9, atol=1e-12, err_msg=f"{env} shape {i} k={k}")


def test_concurrent_order_schedule_is_bitwise_serial(tmp_path):
    """cumulants_upto issues the per-order GEMMs on side streams; the result is
    bitwise that of the serial schedule (BCG_SERIAL_ORDERS=1, own process)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    x = np.random.default_rng(3).exponential(1.0, (50_000, 11))
    np.save(tmp_path / "x.npy", x)
    code = ("import sys, numpy as np; sys.path.insert(0, %r)\n"
            "import paper_1701_05420_b200 as bcg\n"
            "cs = bcg.cumulants_upto(np.load(%r), 6, b=3)\n"
            "np.savez(%r, **{f'c{k}': cs[k].packed_host() for k in range(2, 7)})\n"
            % (root, str(tmp_path / "x.npy"), str(tmp_path / "serial.npz")))
    subprocess.run([sys.executable, "-c", code], check=True, env={**os.environ, "BCG_SERIAL_ORDERS": "1"},
                   timeout=600)
    serial = np.load(tmp_path / "serial.npz")
    cs = bcg.cumulants_upto(x, 6, b=3)
    for k in range(2, 7):
        np.testing.assert_array_equal(cs[k].packed_host(), serial[f"c{k}"])


@pytest.mark.parametrize("n,m,b", [(12, 6, 3), (13, 5, 2), (16, 4, 4), (10, 6, 2)])
def test_recursion_key_ranges_compose_bitwise(n, m, b, rng):
    """The block-range recursion the multi-GPU paths run per rank
    (CudaOps.recursion_range -> bcg_cumulant_recursion_ex on [k0, k1)) over a
    split of the key list equals the full-range recursion bit for bit,
    incl. partial-edge blocks (n % b != 0)."""
    import torch

    from paper_1701_05420_b200.cumulants import cumulants_device
    from paper_1701_05420_b200.distributed import CudaOps, block_bounds
    from paper_1701_05420_b200.layout import layout
    from paper_1701_05420_b200.moments import _center_transposed, _moment_device_t

    x = torch.from_numpy(rng.exponential(1.0, (2000, n)) + rng.standard_normal((2000, n))).cuda()
    _, lower_t = cumulants_device(x, m - 1, b, c1_host=False)
    lower = {t.m: t.data for t in lower_t if t.m <= m - 2}
    xt = _center_transposed(x, x.mean(0))
    central = {k: _moment_device_t(xt, x.shape[0], k, b).data for k in range(4, m - 1)}
    mk = _moment_device_t(xt, x.shape[0], m, b).data
    K = layout(n, m, b).K
    ops = CudaOps()
    full = mk.clone()
    ops.recursion_range(full, n, m, b, lower, 0, K, central)
    for world in (2, 3, 5):
        part = mk.clone()
        for r in range(world):
            k0, k1 = block_bounds(K, world, r)
            ops.recursion_range(part, n, m, b, lower, k0, k1, central)
        assert torch.equal(part, full), world


@pytest.mark.parametrize("n,m,b,t", [(3, 8, 2, 300), (5, 7, 3, 400), (2, 9, 1, 200), (2, 10, 1, 200)])
def test_high_order_cumulants_match_oracle(n, m, b, t, rng):
    """Orders past the factored kernel's range (m >= 7: the partition-table
    recursion) against the oracle, including partial blocks."""
    x = rng.exponential(1.0, (t, n)) + rng.standard_normal((t, n))
    cs = bcg.cumulants_upto(x, m, b=b)
    c1, want = orc.cumulants_upto(x, m, b)
    np.testing.assert_allclose(cs[1], c1, rtol=1e-12, atol=1e-15)
    for k in range(2, m + 1):
        np.testing.assert_allclose(packed(cs[k]), want[k], rtol=1e-9, atol=1e-12, err_msg=f"k={k}")


def test_order_12_runs_with_exact_properties(rng):
    """MAX_M = 12 (bc/partitions.py:16): the partition recursion with its
    2.5e6 slots per block (plan-table lookups, not shared memory) runs, and
    the exact properties hold: constant data gives exact zeros, power-of-two
    scaling scales every order bitwise."""
    x = rng.exponential(1.0, (150, 2))
    cs = bcg.cumulants_upto(x, 12, b=1)
    cs2 = bcg.cumulants_upto(2.0 * x, 12, b=1)
    for k in range(2, 13):
        a = packed(cs[k])
        assert np.all(np.isfinite(a))
        np.testing.assert_array_equal(packed(cs2[k]), (2.0 ** k) * a)
    const = bcg.cumulants_upto(np.full((50, 2), 3.25), 12, b=1)
    for k in range(2, 13):
        assert np.max(np.abs(packed(const[k]))) == 0.0


def test_blocksymtensor_arithmetic_errors_and_bitwise_commutation(rng):
    """pkg/tests/test_symtensor.py:172-199: a + b elementwise, shape mismatch
    rejected, addition commutes bitwise (device axpby)."""
    from conftest import random_sym_dense

    a = bcg.BlockSymTensor.from_dense(random_sym_dense(4, 3, rng), b=2)
    c = bcg.BlockSymTensor.from_dense(random_sym_dense(4, 3, rng), b=2)
    np.testing.assert_array_equal((a + c).to_dense(), (c + a).to_dense())
    assert (a + c).get((1, 2, 3)) == a.get((1, 2, 3)) + c.get((1, 2, 3))
    d = bcg.BlockSymTensor.from_dense(random_sym_dense(4, 3, rng), b=1)
    with pytest.raises(bcg.ValidationError, match="mismatch"):
        a + d


def _gloo_gpu_worker(rank, world, port, x, m, b, out):
    import os

    import torch.distributed as dist

    from paper_1701_05420_b200.distributed import cumulants_upto_block_split, cumulants_upto_sharded, shard_bounds

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_bounds(x.shape[0], world, rank)
    mean, ts = cumulants_upto_sharded(torch.from_numpy(x[lo:hi]).cuda(), m, b)
    _, ts2 = cumulants_upto_block_split(torch.from_numpy(x).cuda(), m, b)
    np.savez(f"{out}_{rank}.npz", mean=mean.cpu().numpy(), **{f"c{k}": t.cpu().numpy() for k, t in enumerate(ts, 2)},
             **{f"d{k}": t.cpu().numpy() for k, t in enumerate(ts2, 2)})
    dist.destroy_process_group()


@pytest.mark.parametrize("t,n,m,b", [(5001, 9, 6, 3), (3000, 16, 4, 8), (300, 745, 2, 7)])
def test_two_ranks_on_one_gpu_over_gloo(t, n, m, b, tmp_path, rng):
    """World size 2 through the real CUDA per-rank ops (both ranks on cuda:0,
    host-staged gloo collectives, so no kernel waits on another rank): the
    sample split (all-reduce, reduce-scatter -> block-range recursion ->
    all-gather) matches cumulants_upto, the block split bit for bit."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    x = rng.exponential(1.0, (t, n)) + rng.standard_normal((t, n))
    out = str(tmp_path / "r")
    mp.spawn(_gloo_gpu_worker, args=(2, port, x, m, b, out), nprocs=2, join=True)
    cs = bcg.cumulants_upto(x, m, b=b)
    for r in range(2):
        got = np.load(f"{out}_{r}.npz")
        np.testing.assert_allclose(got["mean"], cs[1], rtol=1e-13)
        for k in range(2, m + 1):
            want = cs[k].packed_host()
            np.testing.assert_allclose(got[f"c{k}"], want, rtol=1e-9, atol=1e-12)
            np.testing.assert_array_equal(got[f"d{k}"], want)


@pytest.mark.parametrize("n,m,b,t", [(300, 2, 7, 700), (600, 2, 16, 300), (260, 3, 5, 300), (513, 2, 1, 200), (257, 3, 32, 100),
                                     (700, 2, 50, 150)])
def test_wide_data_matrices(n, m, b, t, rng):
    """n > 256 variables: the chunk is staged by several 2-D TMA boxes (256
    variables each) -- moments and cumulants against the oracle."""
    x = rng.standard_normal((t, n)) + rng.exponential(1.0, (t, n))
    np.testing.assert_allclose(packed(bcg.moment(x, m, b)), orc.moment(x, m, b), rtol=1e-12, atol=1e-12)
    cs = bcg.cumulants_upto(x, m, b=b)
    _, want = orc.cumulants_upto(x, m, b)
    np.testing.assert_allclose(packed(cs[m]), want[m], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("n,m,b,t", [(9, 6, 3, 700), (8, 6, 2, 500), (6, 7, 2, 400), (10, 5, 4, 600)])
def test_single_order_cumulant_api_matches_oracle(n, m, b, t, rng):
    """cumulant(x_centered, m, lower) (bc/cumulants.py:119-136) with the lower
    cumulants from cumulants_upto: the factored recursion (central moments
    computed on the fly for m >= 6) against the oracle and against
    cumulants_upto's own C_m."""
    x = rng.exponential(1.0, (t, n)) + rng.standard_normal((t, n))
    cs = bcg.cumulants_upto(x, m, b=b)
    xc = bcg.center(x)
    got = bcg.cumulant(xc, m, [cs[k] for k in range(2, m - 1)], b=b)
    _, want = orc.cumulants_upto(x, m, b)
    np.testing.assert_allclose(packed(got), want[m], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(packed(got), packed(cs[m]), rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("n,m,b,t", [(800, 2, 4, 300), (1500, 2, 1, 200), (760, 3, 40, 150), (731, 2, 731, 100),
                                     (731, 2, 3, 200), (745, 3, 7, 120)])
def test_wider_than_one_stage(n, m, b, t, rng):
    """n > 720 variables (one sample chunk of all of them no longer fits the
    kernel's shared-memory stage): the variable-group decomposition against
    the oracle, and bitwise consistent between moment() and cumulants_upto()."""
    x = rng.standard_normal((t, n)) + rng.exponential(1.0, (t, n))
    if b > 720 // m:
        with pytest.raises(bcg.ValidationError, match="too large"):
            bcg.moment(x, m, b)
        return
    got = packed(bcg.moment(x, m, b))
    np.testing.assert_allclose(got, orc.moment(x, m, b), rtol=1e-12, atol=1e-12)
    cs = bcg.cumulants_upto(x, m, b=b)
    np.testing.assert_array_equal(packed(cs[m]), packed(bcg.moment(bcg.center(x), m, b)))
    np.testing.assert_array_equal(packed(bcg.moment_parallel_blocks(x, m, b, p=3)), got)


@pytest.mark.parametrize("n,m,b,t", [(12, 6, 3, 700), (10, 5, 2, 500), (9, 4, 4, 400), (7, 6, 3, 300)])
def test_recursion_on_element_spans(n, m, b, t, rng):
    """bcg_cumulant_recursion_span (the per-rank step of the element-balanced
    multi-GPU split): spans that cut blocks mid-way, applied to copies of the
    same M_m, reassemble the full recursion; elements outside a span stay
    untouched."""
    import ctypes

    from paper_1701_05420_b200.layout import layout

    x = rng.exponential(1.0, (t, n)) + rng.standard_normal((t, n))
    cs = bcg.cumulants_upto(x, m - 1, b=b)
    xc = bcg.center(x)
    mom = bcg.moment(xc, m, b).data
    lower = (ctypes.c_void_p * 15)()
    for k in range(2, m - 1):
        lower[k - 2] = cs[k].data.data_ptr()
    cm = (ctypes.c_void_p * 15)()
    m4 = bcg.moment(xc, 4, b).data if m == 6 else None
    if m4 is not None:
        cm[2] = m4.data_ptr()
    plan = _native.plan(n, m, b)
    S = layout(n, m, b).size
    full = mom.clone()
    _native.check(_native.lib().bcg_cumulant_recursion_span(plan.handle, full.data_ptr(), lower, cm, 0, S,
                                                            _native.stream_handle()))
    cuts = [0, S // 3 + 1, S // 3 + 7, (2 * S) // 3 - 5, S]
    got = torch.empty_like(mom)
    for e0, e1 in zip(cuts, cuts[1:]):
        part = mom.clone()
        _native.check(_native.lib().bcg_cumulant_recursion_span(plan.handle, part.data_ptr(), lower, cm, e0, e1,
                                                                _native.stream_handle()))
        assert torch.equal(part[:e0], mom[:e0]) and torch.equal(part[e1:], mom[e1:])
        got[e0:e1] = part[e0:e1]
    np.testing.assert_allclose(got.cpu().numpy(), full.cpu().numpy(), rtol=1e-12, atol=1e-15)
    _, want = orc.cumulants_upto(x, m, b)
    np.testing.assert_allclose(got.cpu().numpy(), want[m], rtol=1e-9, atol=1e-12)
