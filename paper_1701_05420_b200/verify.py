"""GPU dense-entry oracle: full-size verification of moments and cumulants
(SURVEY §8 f row 4).

The reference verifies its engines against a dense oracle that materialises
the n^m tensor and runs the dense recursion (bc/oracle.py:89-117), so it is
limited to n^m <= 1e8 and m <= 6 (bc/oracle.py:22-34).  This module checks
single ELEMENTS instead, at any n and t:

* `subset_moments` -- one CUDA pass over the samples (csrc/dense.cu,
  `bcg_dense_subsets`) gives, for each requested element (i_1..i_m), the
  central moments M(S) of all 2^m sub-tuples S of its indices;
* `element_cumulants` -- the joint cumulant of the full tuple by the
  moment-cumulant formula over set partitions (Leonov-Shiryaev):
      C(1..m) = sum_pi (-1)^(|pi|-1) (|pi|-1)! prod_{B in pi} M(B),
  over the partitions pi of the m positions into blocks of size >= 2 (blocks
  of size 1 vanish for centered data).  Nothing here shares code with the
  product path: no block layout, no Khatri-Rao GEMM, no packed tensors, and
  not the reference's recursion C_m = M_m - sum_sigma B_sigma
  (bc/cumulants.py:119-136) either;
* `check_cumulant_set` -- samples element tuples of every order of a
  `CumulantSet` and compares its stored values with the oracle.

Verification infrastructure: cumulants_upto never calls this module.
"""

from __future__ import annotations

import math
from functools import lru_cache

import numpy as np

from . import _native
from .layout import layout, locate


@lru_cache(maxsize=None)
def partitions_min2_masks(m: int) -> tuple:
    """Set partitions of {0..m-1} into blocks of size >= 2, as tuples of
    bit masks (F(m) of them: 1, 1, 4, 11, 41, 162, 715 for m = 2..8)."""
    out = []

    def rec(rest: int, blocks: list):
        if rest == 0:
            out.append(tuple(blocks))
            return
        low = rest & -rest  # the lowest remaining position opens the next block
        others = rest ^ low
        sub = others
        while True:  # every subset of the other remaining positions joins it
            blk = low | sub
            if bin(blk).count("1") >= 2:
                rec(rest ^ blk, blocks + [blk])
            if sub == 0:
                break
            sub = (sub - 1) & others

    rec((1 << m) - 1, [])
    return tuple(out)


def subset_moments(x, idx, mean=None):
    """Central moments of every sub-tuple of each element tuple.

    x: (t, n) float64 torch CUDA tensor (or array, copied to the device);
    idx: (E, m) 0-based column indices, 1 <= m <= 8; mean: column means
    (default: the sample mean, as cumulants_upto centres).  Returns an
    (E, 2^m) float64 numpy array, column S = the central moment of the
    positions in bit mask S (column 0 = 1)."""
    torch = _native.torch_cuda()
    if not isinstance(x, torch.Tensor):
        x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    x = x.to(device="cuda", dtype=torch.float64)
    if x.dim() != 2 or x.stride(1) != 1:
        x = x.contiguous()
    t, n = x.shape
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    if idx.ndim != 2:
        raise ValueError("idx must be (E, m)")
    E, m = idx.shape
    if idx.size and (idx.min() < 0 or idx.max() >= n):
        raise ValueError("column index out of range")
    if mean is None:
        mean = x.sum(dim=0) / t
    mean = torch.as_tensor(mean, dtype=torch.float64, device="cuda").contiguous()
    d_idx = torch.from_numpy(idx).cuda()
    out = torch.empty((E, 1 << m), dtype=torch.float64, device="cuda")
    lib = _native.lib()
    ws_bytes = lib.bcg_dense_subsets_ws_bytes(E, m, t)
    ws = torch.empty(max(1, ws_bytes // 8), dtype=torch.float64, device="cuda")
    _native.check(lib.bcg_dense_subsets(x.data_ptr(), t, n, x.stride(0), mean.data_ptr(), m, d_idx.data_ptr(), E,
                                        out.data_ptr(), ws.data_ptr(), ws_bytes, _native.stream_handle()),
                  "dense subsets")
    return out.cpu().numpy() / t


def element_cumulants(moments: np.ndarray, m: int) -> np.ndarray:
    """Joint cumulant of the full m-tuple from subset_moments' output, by the
    moment-cumulant formula over set partitions into blocks of size >= 2."""
    c = np.zeros(moments.shape[0])
    for parts in partitions_min2_masks(m):
        k = len(parts)
        term = float((-1) ** (k - 1) * math.factorial(k - 1)) * np.ones(moments.shape[0])
        for blk in parts:
            term = term * moments[:, blk]
        c = c + term
    return c


def packed_values(packed: np.ndarray, n: int, b: int, idx: np.ndarray) -> np.ndarray:
    """Stored values of a packed order-m tensor at 0-based element tuples
    (any order): the block layout lookup of BlockSymTensor.get
    (bc/symtensor.py:143-151)."""
    E, m = idx.shape
    lay = layout(n, m, b)
    out = np.empty(E)
    for e in range(E):
        key, offs = locate(tuple(sorted(int(i) + 1 for i in idx[e])), b)
        k = lay.key_index(key)
        edges = lay.edges[k]
        lin = 0
        for q in range(m):
            lin = lin * int(edges[q]) + (offs[q] - 1)
        out[e] = packed[lay.offs[k] + lin]
    return out


def sample_tuples(n: int, m: int, count: int, rng) -> np.ndarray:
    """`count` element tuples of order m: uniform random indices, plus
    tuples with repeated indices (diagonal blocks, permutation fills)."""
    idx = rng.integers(0, n, size=(count, m))
    rep = count // 4
    if rep and m >= 2:
        idx[:rep, 1] = idx[:rep, 0]  # a repeated index
        idx[rep:2 * rep, :] = idx[rep:2 * rep, :1]  # all equal
    return np.sort(idx, axis=1)


def check_cumulant_set(x, cs, b: int, count: int = 64, seed: int = 0, orders=None):
    """Compare `count` sampled elements of every order k of a CumulantSet with
    the dense oracle on the same data.  Returns {k: (got, want)} arrays."""
    torch = _native.torch_cuda()
    if not isinstance(x, torch.Tensor):
        x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    x = x.cuda()
    n = x.shape[1]
    rng = np.random.default_rng(seed)
    res = {}
    for k in orders or range(2, cs.max_order + 1):
        idx = sample_tuples(n, k, count, rng)
        mom = subset_moments(x, idx)
        want = element_cumulants(mom, k)
        got = packed_values(cs[k].packed_host(), n, b, idx)
        res[k] = (got, want)
    return res
