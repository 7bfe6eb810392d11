"""Host-side data type and layout helpers (no GPU): the reference's
BlockSymTensor / layout contract (pkg/tests/test_symtensor.py)."""

import itertools
import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_1701_05420_b200 import (
    BlockSymTensor,
    ValidationError,
    block_edges,
    block_keys,
    canonical_index,
    locate,
    unique_block_count,
)
from paper_1701_05420_b200.layout import enumerate_partitions_min2, layout
from conftest import random_sym_dense
from oracle import oracle as orc


def test_locate_examples():
    assert locate((1, 2, 3), 2) == ((1, 1, 2), (1, 2, 1))
    assert locate((5, 5), 2) == ((3, 3), (1, 1))
    assert block_edges((3, 3), 5, 2) == (1, 1)
    assert canonical_index((2, 2, 1)) == (1, 2, 2)


@given(st.integers(1, 6), st.lists(st.integers(1, 30), min_size=1, max_size=6))
@settings(max_examples=50, deadline=None)
def test_locate_roundtrip(b, index):
    index = tuple(sorted(index))
    j, offsets = locate(index, b)
    assert list(j) == sorted(j)
    assert tuple((jk - 1) * b + ok for jk, ok in zip(j, offsets)) == index


def test_unique_block_count():
    assert unique_block_count(2, 2) == 3
    assert unique_block_count(30, 4) == 40920
    with pytest.raises(ValidationError):
        unique_block_count(0, 2)


@pytest.mark.parametrize("n,m,b", [(5, 3, 2), (7, 4, 3), (24, 4, 4), (9, 5, 4)])
def test_layout_matches_oracle(n, m, b):
    lay = layout(n, m, b)
    keys, col0, edges, offs = orc.block_layout(n, m, b)
    assert lay.keys == keys
    np.testing.assert_array_equal(lay.col0, col0)
    np.testing.assert_array_equal(lay.edges, edges)
    np.testing.assert_array_equal(lay.offs, offs)


def test_partitions_match_golden(golden):
    for key, parts in golden("partitions.json").items():
        m, sigma = map(int, key.split(","))
        assert [list(map(list, p)) for p in enumerate_partitions_min2(m, sigma)] == parts


@pytest.mark.parametrize("n,m,b", [(4, 2, 2), (5, 3, 2), (3, 4, 2), (6, 3, 4), (5, 2, 3)])
def test_dense_roundtrip(n, m, b, rng):
    dense = random_sym_dense(n, m, rng)
    t = BlockSymTensor.from_dense(dense, b)
    np.testing.assert_array_equal(t.to_dense(), dense)
    assert t.stored_element_count == layout(n, m, b).size


def test_from_dense_rejects_asymmetric(rng):
    with pytest.raises(ValidationError, match="super-symmetric"):
        BlockSymTensor.from_dense(rng.standard_normal((3, 3)), 2)


def test_get_permutation_invariance(rng):
    t = BlockSymTensor.from_dense(random_sym_dense(6, 4, rng), 2)
    for _ in range(300):
        idx = tuple(rng.integers(1, 7, size=4))
        perm = tuple(idx[q] for q in rng.permutation(4))
        assert t.get(idx) == t.get(perm)
    with pytest.raises(ValidationError):
        t.get((1, 2, 3))
    with pytest.raises(ValidationError):
        t.get((0, 1, 2, 3))


def test_blocks_are_views_of_packed(rng):
    dense = random_sym_dense(5, 3, rng)
    t = BlockSymTensor.from_dense(dense, 2)
    flat = t.packed_host()
    lay = layout(5, 3, 2)
    for k, key in enumerate(lay.keys):
        np.testing.assert_array_equal(t.blocks[key].ravel(), flat[lay.offs[k]:lay.offs[k + 1]])
    # reference constructor from a dict packs to the same buffer
    t2 = BlockSymTensor(5, 3, 2, dict(t.blocks))
    np.testing.assert_array_equal(t2.packed_host(), flat)


def test_doc_roundtrip_and_validation(rng):
    t = BlockSymTensor.from_dense(random_sym_dense(5, 3, rng), 2)
    doc = t.to_doc()
    assert [b["j"] for b in doc["blocks"]] == [list(k) for k in sorted(t.blocks)]
    back = BlockSymTensor.from_doc(doc)
    np.testing.assert_array_equal(back.to_dense(), t.to_dense())
    bad = dict(doc, blocks=doc["blocks"][1:])
    with pytest.raises(ValidationError, match="missing block keys"):
        BlockSymTensor.from_doc(bad)
    dup = dict(doc, blocks=doc["blocks"] + doc["blocks"][:1])
    with pytest.raises(ValidationError, match="duplicate"):
        BlockSymTensor.from_doc(dup)
    with pytest.raises(ValidationError, match="malformed"):
        BlockSymTensor.from_doc({"n": 3})


def test_storage_ratio():
    # n=40, m=4, b=2: stored-element ratio 18.1 (pkg/README.md:136-137)
    ratio = 40 ** 4 / layout(40, 4, 2).size
    assert 18.0 < ratio < 18.2
    assert ratio < math.factorial(4)


def test_constructor_validation():
    with pytest.raises(ValidationError):
        BlockSymTensor(0, 2, 2, {})
    with pytest.raises(ValidationError):
        BlockSymTensor.from_packed(4, 2, 2, np.zeros(3))


def test_get_index_errors():
    """Element access errors as the reference (pkg/tests/test_symtensor.py:143-147)."""
    t = BlockSymTensor.zeros(3, 2, 2)
    with pytest.raises(ValidationError, match="out of range"):
        t.get((1, 4))
    with pytest.raises(ValidationError, match="entries"):
        t.get((1, 2, 3))
    assert BlockSymTensor.from_dense(np.ones((3, 3, 3)), b=2).get((1, 2, 2)) == 1.0
