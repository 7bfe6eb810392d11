"""Block layout of packed super-symmetric tensors (host side).

Same functions and semantics as the reference's layout helpers
(bc/symtensor.py:25-54) and its partition enumeration (bc/partitions.py:63-98).
The native plan (csrc/plan.cu) builds the identical tables in C++ for the
device; tests pin both against the reference's golden layout.
"""

from __future__ import annotations

import itertools
from functools import lru_cache
from math import comb

import numpy as np

from .errors import ValidationError

MAX_M = 12  # bc/partitions.py:16


def canonical_index(index) -> tuple[int, ...]:
    """Sorted representative of an element multi-index (bc/symtensor.py:25-27)."""
    return tuple(sorted(index))


def locate(index, b: int) -> tuple[tuple[int, ...], tuple[int, ...]]:
    """Sorted 1-based element index -> (block key, 1-based offsets)
    (bc/symtensor.py:30-37)."""
    j = tuple((i + b - 1) // b for i in index)
    offsets = tuple(i - (jk - 1) * b for i, jk in zip(index, j))
    return j, offsets


def unique_block_count(n_bar: int, m: int) -> int:
    """Stored blocks: size-m multisets over 1..n_bar (bc/symtensor.py:40-44)."""
    if n_bar < 1 or m < 1:
        raise ValidationError("n_bar and m must be >= 1")
    return comb(n_bar + m - 1, m)


def block_keys(n_bar: int, m: int):
    """All sorted block keys, lexicographic (bc/symtensor.py:47-49)."""
    return itertools.combinations_with_replacement(range(1, n_bar + 1), m)


def block_edges(key, n: int, b: int) -> tuple[int, ...]:
    """Edge along each mode of block ``key`` (bc/symtensor.py:52-54)."""
    return tuple(min(j * b, n) - (j - 1) * b for j in key)


class Layout:
    """keys / col0 / edges / offs of one (n, m, b), as bc/_engines.py:46-54."""

    __slots__ = ("n", "m", "b", "keys", "col0", "edges", "offs", "index")

    def __init__(self, n: int, m: int, b: int):
        nb = -(-n // b)
        self.n, self.m, self.b = n, m, b
        self.keys = list(block_keys(nb, m))
        K = len(self.keys)
        karr = np.array(self.keys, dtype=np.int64).reshape(K, m)
        self.col0 = (karr - 1) * b
        self.edges = np.minimum(karr * b, n) - (karr - 1) * b
        self.offs = np.zeros(K + 1, dtype=np.int64)
        np.cumsum(self.edges.prod(axis=1), out=self.offs[1:])
        self.index = None

    @property
    def K(self) -> int:
        return len(self.keys)

    @property
    def size(self) -> int:
        return int(self.offs[-1])

    def key_index(self, key) -> int:
        if self.index is None:
            self.index = {k: i for i, k in enumerate(self.keys)}
        return self.index[tuple(key)]


@lru_cache(maxsize=64)
def layout(n: int, m: int, b: int) -> Layout:
    return Layout(int(n), int(m), int(b))


@lru_cache(maxsize=None)
def enumerate_partitions_min2(m: int, sigma: int):
    """Canonical partitions of 1..m into sigma parts of size >= 2, in the
    reference's order (bc/partitions.py:63-98)."""
    if not 1 <= m <= MAX_M:
        raise ValidationError(f"m must be in 1..{MAX_M}, got {m}")
    if sigma < 1:
        raise ValidationError(f"sigma must be >= 1, got {sigma}")
    out = []
    parts: list[list[int]] = []

    def rec(e: int, short: int):
        if e > m:
            if len(parts) == sigma and short == 0:
                out.append(tuple(tuple(p) for p in parts))
            return
        if m - e + 1 < short + 2 * (sigma - len(parts)):
            return
        for p in parts:
            single = len(p) == 1
            p.append(e)
            rec(e + 1, short - single)
            p.pop()
        if len(parts) < sigma:
            parts.append([e])
            rec(e + 1, short + 1)
            parts.pop()

    rec(1, 0)
    return tuple(out)
