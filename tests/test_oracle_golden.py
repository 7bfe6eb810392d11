"""Pin the CPU oracle (oracle/) against the reference's own outputs.

The golden vectors were produced by the unmodified reference package
(tests/golden/make_golden.py); these tests make the oracle a trustworthy
checker before any GPU result is compared with it.  CPU only.
"""

import json

import numpy as np
import pytest

from oracle import oracle as orc
import workloads


def test_layout_small_tables_match_reference(golden):
    g = golden("layout.npz")
    tags = sorted({k.split("_", 1)[1] for k in g.files if k.startswith("keys_")})
    assert len(tags) >= 8
    for tag in tags:
        n, m, b = map(int, tag.split("_"))
        keys, col0, edges, offs = orc.block_layout(n, m, b)
        np.testing.assert_array_equal(np.array(keys, dtype=np.int64).reshape(-1, m), g[f"keys_{tag}"])
        np.testing.assert_array_equal(col0, g[f"col0_{tag}"])
        np.testing.assert_array_equal(edges, g[f"edges_{tag}"])
        np.testing.assert_array_equal(offs, g[f"offs_{tag}"])


def test_layout_pin_5_3_2():
    # 10 keys starting (1,1,1),(1,1,2),(1,1,3),(1,2,2) ...
    keys, _, edges, offs = orc.block_layout(5, 3, 2)
    assert keys[:4] == [(1, 1, 1), (1, 1, 2), (1, 1, 3), (1, 2, 2)]
    assert list(offs[:6]) == [0, 8, 16, 20, 28, 32] and offs[-1] == 49
    assert tuple(edges[2]) == (2, 2, 1)


def test_layout_config_digests_match_reference(golden):
    import hashlib

    digests = json.loads(str(golden("layout.npz")["digests"]))
    assert len(digests) == 20  # every BASELINE config, orders 2..m
    for tag, want in digests.items():
        n, m, b = map(int, tag.split("_"))
        keys, col0, edges, offs = orc.block_layout(n, m, b)
        h = hashlib.sha256()
        for a in (np.array(keys, dtype=np.int64).reshape(-1, m), col0, edges, offs):
            h.update(np.ascontiguousarray(a).tobytes())
        assert h.hexdigest() == want, tag


def test_partitions_match_reference(golden):
    table = golden("partitions.json")
    for key, parts in table.items():
        m, sigma = map(int, key.split(","))
        got = [list(map(list, p)) for p in orc.partitions_min2(m, sigma)]
        assert got == parts, key


def test_partition_counts():
    # S'(m, sigma) values pinned by pkg/tests/test_partitions.py:115-121
    assert [len(orc.partitions_min2(*a)) for a in ((4, 2), (5, 2), (6, 2), (6, 3), (8, 2))] == [3, 10, 25, 15, 119]
    assert orc.partitions_min2(4, 2) == (((1, 2), (3, 4)), ((1, 3), (2, 4)), ((1, 4), (2, 3)))


def test_moments_match_reference(golden):
    g = golden("moments.npz")
    count = 0
    for key in g.files:
        if not key.startswith("shape_"):
            continue
        i = key.split("_")[1]
        n, m, b, t = map(int, g[key])
        got = orc.moment(g[f"x_{i}"], m, b)
        np.testing.assert_allclose(got, g[f"m_{i}"], rtol=1e-12, atol=1e-14)
        count += 1
    assert count >= 8


def test_cumulants_match_reference(golden):
    g = golden("cumulants.npz")
    count = 0
    for key in g.files:
        if not key.startswith("shape_"):
            continue
        i = key.split("_")[1]
        n, t, m_max, b = map(int, g[key])
        c1, cs = orc.cumulants_upto(g[f"x_{i}"], m_max, b)
        np.testing.assert_allclose(c1, g[f"c1_{i}"], rtol=1e-12, atol=1e-15)
        for k in range(2, m_max + 1):
            np.testing.assert_allclose(cs[k], g[f"c{k}_{i}"], rtol=1e-9, atol=1e-12)
        count += 1
    assert count >= 24


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4", "cfg5"])
def test_config_recipes_match_reference(name, golden):
    g = golden("configs.npz")
    cfg = workloads.CONFIGS[name]
    x = g[f"{name}_x"]
    # the committed input is the recipe's output (pins workloads.generate)
    np.testing.assert_allclose(workloads.generate(name, x.shape[0]), x, rtol=1e-13, atol=0)
    m_top = max(int(k.split("_")[1][1:]) for k in g.files if k.startswith(f"{name}_c") and k.endswith("_idx"))
    if name == "cfg4":
        m_top = min(m_top, 5)  # order-6 recursion in numpy is ~10 s; GPU tests cover it
    c1, cs = orc.cumulants_upto(x, m_top, cfg.b)
    np.testing.assert_allclose(c1, g[f"{name}_c1"], rtol=1e-12, atol=1e-15)
    for k in range(2, m_top + 1):
        idx = g[f"{name}_c{k}_idx"]
        np.testing.assert_allclose(cs[k][idx], g[f"{name}_c{k}_val"], rtol=1e-9, atol=1e-12)


def test_kat_two_sample_matrix():
    # pkg/tests/test_moments.py:71-76: X=[[1,2],[3,4]], key (1,1) -> [[5,7],[7,10]]
    got = orc.moment(np.array([[1.0, 2.0], [3.0, 4.0]]), 2, 2)
    np.testing.assert_array_equal(got, [5.0, 7.0, 7.0, 10.0])


def test_kat_two_point_c4():
    # pkg/tests/test_oracle.py:77-80: +-1 equally likely -> C4 = -2
    x = np.array([[-1.0], [1.0]] * 5)
    _, cs = orc.cumulants_upto(x, 4, 1)
    assert cs[4][0] == pytest.approx(-2.0, rel=1e-14)


def test_dense_roundtrip_and_dense_moment(rng):
    x = rng.standard_normal((50, 5))
    for m in (2, 3, 4):
        dense = orc.packed_to_dense(orc.moment(x, m, 2), 5, m, 2)
        np.testing.assert_allclose(dense, orc.dense_moment(x, m), rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("tag", ["cfg5s", "cfg2s"])
def test_highorder_fixture_inputs_and_low_orders(tag, golden):
    """tests/golden/highorder.npz (heavy tails to order 6, made by the
    reference): the recipe regenerates its input bit for bit, and the oracle
    matches the reference's C1..C4 there (C5/C6 are checked on the GPU,
    tests/test_gpu_highorder.py)."""
    g = golden("highorder.npz")
    spec = {"cfg5s": ("cfg5", 36, 6, 3000), "cfg2s": ("cfg2", 32, 8, 3000)}[tag]
    name, ncols, b, t = spec
    x = np.ascontiguousarray(workloads.generate(name, t)[:, :ncols])
    np.testing.assert_allclose([x.sum(), (x * x).sum(), np.abs(x).max()], g[f"{tag}_xsum"], rtol=1e-13)
    c1, cs = orc.cumulants_upto(x, 4, b)
    np.testing.assert_allclose(c1, g[f"{tag}_c1"], rtol=1e-12, atol=1e-15)
    for k in range(2, 5):
        idx = g[f"{tag}_c{k}_idx"]
        np.testing.assert_allclose(cs[k][idx], g[f"{tag}_c{k}_val"], rtol=1e-9, atol=1e-12)
