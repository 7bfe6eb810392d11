"""ORACLE -- CPU restatement of the reference hot path, for checking only.

Test infrastructure: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` leg may import this module, and only as the
checker.  The product package (``paper_1701_05420_b200``) never imports it and
has no CPU fallback.

Every function restates one piece of the reference package ``blockcumulants``
(``/root/reference/pkg/src/blockcumulants``; cited below as ``bc/<file>:<line>``):

* layout:      ``block_keys`` / ``block_edges`` (bc/symtensor.py:47-54) and
               ``_block_layout`` (bc/_engines.py:46-54)
* partitions:  ``enumerate_partitions_min2`` (bc/partitions.py:63-98) and
               ``enumerate_partitions`` (bc/partitions.py:26-60)
* moment:      ``moment_compiled`` (bc/_engines.py:83-100) over the C kernel in
               ``oracle/moment_blocks.c`` (restating bc/_core.pyx:60-148)
* recursion:   ``outer_prod_cum`` (bc/cumulants.py:53-84), ``cumulant``
               (bc/cumulants.py:119-136), ``cumulants_upto``
               (bc/cumulants.py:173-193)
* dense:       ``to_dense`` (bc/symtensor.py:153-174) and a literal dense
               moment (bc/oracle.py:37-66)

Parity of this restatement is PINNED: ``tests/test_oracle_golden.py`` checks it
against golden vectors produced by the reference itself
(``tests/golden/make_golden.py``).

Packed tensors are flat float64 arrays in the reference's block order: block k
(lexicographic sorted key) occupies ``flat[offs[k]:offs[k+1]]`` row-major over
its edges -- exactly the buffer ``moment_compiled`` fills before ``_pack``.
"""

from __future__ import annotations

import ctypes
import itertools
import os
import subprocess
from functools import lru_cache

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD_DIR = os.path.join(HERE, "_build")
LIB_PATH = os.path.join(BUILD_DIR, "liboracle.so")
MAX_M = 12  # bc/partitions.py:16


# -- native build --------------------------------------------------------------


def build_lib(force: bool = False) -> str:
    """Compile oracle/moment_blocks.c into oracle/_build/liboracle.so."""
    src = os.path.join(HERE, "moment_blocks.c")
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= os.path.getmtime(src)):
        return LIB_PATH
    os.makedirs(BUILD_DIR, exist_ok=True)
    subprocess.check_call(
        ["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", LIB_PATH, src]
    )
    return LIB_PATH


@lru_cache(maxsize=1)
def _lib():
    lib = ctypes.CDLL(build_lib())
    i64 = ctypes.c_int64
    ptr = ctypes.c_void_p
    lib.oracle_moment_blocks.argtypes = [ptr, i64, i64, ptr, ptr, i64, ptr, ptr, i64, i64]
    lib.oracle_moment_blocks.restype = ctypes.c_int
    return lib


# -- layout (bc/symtensor.py:47-54, bc/_engines.py:46-54) ----------------------


def n_bar(n: int, b: int) -> int:
    return -(-n // b)


def block_keys(nb: int, m: int):
    """Sorted block multi-indices, lexicographic (bc/symtensor.py:47-49)."""
    return list(itertools.combinations_with_replacement(range(1, nb + 1), m))


def block_edges(key, n: int, b: int):
    """Edge per mode; the last block is partial when b does not divide n
    (bc/symtensor.py:52-54)."""
    return tuple(min(j * b, n) - (j - 1) * b for j in key)


def block_layout(n: int, m: int, b: int):
    """(keys, col0, edges, offs) as bc/_engines.py:46-54 builds them."""
    keys = block_keys(n_bar(n, b), m)
    col0 = np.array([[(j - 1) * b for j in k] for k in keys], dtype=np.int64).reshape(len(keys), m)
    edges = np.array([block_edges(k, n, b) for k in keys], dtype=np.int64).reshape(len(keys), m)
    offs = np.zeros(len(keys) + 1, dtype=np.int64)
    np.cumsum(edges.prod(axis=1), out=offs[1:])
    return keys, col0, edges, offs


# -- partitions (bc/partitions.py:26-98) ---------------------------------------


@lru_cache(maxsize=None)
def partitions_min2(m: int, sigma: int):
    """Canonical partitions of (1..m) into sigma parts, each of size >= 2, in
    the reference's enumeration order (bc/partitions.py:63-98): element e
    first tries every open part (in opening order), then opens a new part."""
    out = []
    parts: list[list[int]] = []

    def rec(e: int, short: int):
        left = m - e + 1
        if e > m:
            if len(parts) == sigma and short == 0:
                out.append(tuple(tuple(p) for p in parts))
            return
        if left < short + 2 * (sigma - len(parts)):
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


@lru_cache(maxsize=None)
def partitions_all(m: int, sigma: int):
    """All canonical partitions into sigma parts (restricted growth strings,
    bc/partitions.py:26-60)."""
    out = []
    parts: list[list[int]] = []

    def rec(e: int):
        if e > m:
            if len(parts) == sigma:
                out.append(tuple(tuple(p) for p in parts))
            return
        if sigma - len(parts) > m - e + 1:
            return
        for p in parts:
            p.append(e)
            rec(e + 1)
            p.pop()
        if len(parts) < sigma:
            parts.append([e])
            rec(e + 1)
            parts.pop()

    rec(1)
    return tuple(out)


# -- moment (bc/_engines.py:83-100 over bc/_core.pyx:60-148) -------------------


def moment_raw_sums(x: np.ndarray, m: int, b: int, key_range=None) -> np.ndarray:
    """Packed RAW product sums (no 1/t), as the C kernel accumulates them."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    t, n = x.shape
    keys, col0, edges, offs = block_layout(n, m, b)
    k0, k1 = key_range if key_range is not None else (0, len(keys))
    out = np.zeros(int(offs[-1]))
    xt = np.ascontiguousarray(x.T)
    rc = _lib().oracle_moment_blocks(
        xt.ctypes.data, n, t, col0.ctypes.data, edges.ctypes.data, m,
        out.ctypes.data, offs.ctypes.data, k0, k1,
    )
    if rc != 0:
        raise ValueError("oracle kernel supports 2 <= m <= 16")
    return out


def moment(x: np.ndarray, m: int, b: int) -> np.ndarray:
    """Packed order-m moment (bc/moments.py:44-63; m == 1 -> column means)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if m == 1:
        return x.mean(axis=0)
    out = moment_raw_sums(x, m, b)
    out /= x.shape[0]
    return out


# -- recursion (bc/cumulants.py:53-193) ----------------------------------------

_SUB = "abcdefghijkl"


def block_views(flat: np.ndarray, n: int, m: int, b: int) -> dict:
    keys, _, edges, offs = block_layout(n, m, b)
    return {key: flat[offs[k]:offs[k + 1]].reshape(tuple(edges[k]))
            for k, key in enumerate(keys)}


def outer_prod_cum(m: int, sigma: int, lower: dict, n: int, b: int) -> np.ndarray:
    """B_sigma: per stored key and per min-2 partition, the outer product of
    the lower-cumulant sub-blocks picked by the parts (bc/cumulants.py:53-84).
    ``lower`` maps order -> packed flat array."""
    parts_list = partitions_min2(m, sigma)
    views = {k: block_views(v, n, k, b) for k, v in lower.items()}
    keys, _, edges, offs = block_layout(n, m, b)
    out = np.zeros(int(offs[-1]))
    for k, key in enumerate(keys):
        blk = out[offs[k]:offs[k + 1]].reshape(tuple(edges[k]))
        for parts in parts_list:
            expr = ",".join("".join(_SUB[q - 1] for q in p) for p in parts)
            ops = [views[len(p)][tuple(key[q - 1] for q in p)] for p in parts]
            blk += np.einsum(expr + "->" + _SUB[:m], *ops, optimize=False)
    return out


def cumulant_from_moment(mom: np.ndarray, m: int, lower: dict, n: int, b: int) -> np.ndarray:
    """C_m = (M_m - B_2) - B_3 - ... (bc/cumulants.py:119-136)."""
    if m <= 3:
        return mom
    res = mom
    for sigma in range(2, m // 2 + 1):
        res = res - outer_prod_cum(m, sigma, lower, n, b)
    return res


def cumulants_upto(x: np.ndarray, m_max: int, b: int):
    """(c1, {k: packed C_k}) as bc/cumulants.py:173-193: C1 is the raw mean,
    data centered once, C_k ascending from a fresh moment per order."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    t, n = x.shape
    c1 = x.mean(axis=0)
    out = {}
    if m_max >= 2:
        xc = x - x.mean(axis=0)
        for k in range(2, m_max + 1):
            out[k] = cumulant_from_moment(moment(xc, k, b), k, out, n, b)
    return c1, out


# -- dense helpers (bc/symtensor.py:153-174, bc/oracle.py:37-66) ---------------


def packed_to_dense(flat: np.ndarray, n: int, m: int, b: int) -> np.ndarray:
    """Dense n^m array with every permutation filled: element i reads the block
    of sorted(i) (bc/symtensor.py:143-151 applied to every index)."""
    keys, _, edges, offs = block_layout(n, m, b)
    kindex = {key: k for k, key in enumerate(keys)}
    out = np.empty((n,) * m)
    for idx in itertools.product(range(n), repeat=m):
        s = sorted(idx)
        key = tuple(i // b + 1 for i in s)
        o = [i % b for i in s]
        k = kindex[key]
        lin = 0
        for q in range(m):
            lin = lin * int(edges[k][q]) + o[q]
        out[idx] = flat[offs[k] + lin]
    return out


def dense_moment(x: np.ndarray, m: int) -> np.ndarray:
    """Literal chunked product-sum over all n^m indices (bc/oracle.py:37-66)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    t, n = x.shape
    expr = ",".join("t" + c for c in _SUB[:m]) + "->" + _SUB[:m]
    out = np.zeros((n,) * m)
    for s in range(0, t, 512):
        xs = x[s:s + 512]
        out += np.einsum(expr, *([xs] * m), optimize=True)
    return out / t
