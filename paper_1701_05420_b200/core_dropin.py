"""Drop-in for the reference's compiled module ``blockcumulants._core``
(bc/_core.pyx:126-175): the same two functions with the same arguments,
accumulate semantics and errors, the arithmetic on the B200.

The reference imports its kernel at bc/_engines.py:26-31; switching it is::

    from paper_1701_05420_b200 import core_dropin as _core

after which ``moment(..., engine="compiled")``, ``moment_parallel_blocks`` (its
``key_range`` calls map to ``k0, k1``) and the dense oracle's compiled path run
on the GPU.  Host numpy buffers in, host buffers updated
in place, as the Cython functions do; only ``out[offs[k0]:offs[k1]]`` is
touched by ``moment_blocks``.
"""

from __future__ import annotations

import numpy as np

from . import _native

__all__ = ["moment_blocks", "naive_moment4"]


def _buffer(a, dtype, ndim: int, what: str, writable: bool = False) -> np.ndarray:
    """The Cython typed-memoryview checks: dtype, dimensionality, C order."""
    if not isinstance(a, np.ndarray):
        a = np.asarray(a)
    if a.dtype != dtype:
        want = "long" if dtype == np.int64 else "double"
        raise ValueError(f"Buffer dtype mismatch, expected '{want}' but got '{a.dtype}' ({what})")
    if a.ndim != ndim:
        raise ValueError(f"Buffer has wrong number of dimensions (expected {ndim}, got {a.ndim}) ({what})")
    if not a.flags.c_contiguous:
        raise ValueError(f"ndarray is not C-contiguous ({what})")
    if writable and not a.flags.writeable:
        raise ValueError(f"buffer source array is read-only ({what})")
    return a


def moment_blocks(xt, col0, edges, out, offs, k0, k1) -> None:
    """Accumulate product sums for blocks k0..k1 into the flat buffer ``out``
    (bc/_core.pyx:126-148): out[offs[k] + rowmajor(o)] += sum_l prod_q
    xt[col0[k, q] + o_q, l]."""
    xt = _buffer(xt, np.float64, 2, "xt")
    col0 = _buffer(col0, np.int64, 2, "col0")
    edges = _buffer(edges, np.int64, 2, "edges")
    out = _buffer(out, np.float64, 1, "out", writable=True)
    offs = _buffer(offs, np.int64, 1, "offs")
    m = col0.shape[1]
    if m < 2 or m > 16:
        raise ValueError("kernel supports 2 <= m <= 16")
    K = col0.shape[0]
    k0, k1 = int(k0), int(k1)
    if k1 <= k0:
        return
    torch = _native.torch_cuda()
    n, t = xt.shape
    lo, hi = int(offs[k0]), int(offs[k1])
    from .moments import WIDE_N

    if n > WIDE_N:
        _moment_blocks_wide(xt, col0, edges, out, offs, k0, k1)
        return
    dxt = torch.from_numpy(xt).cuda()
    dc0, de, do = (torch.from_numpy(a).cuda() for a in (col0, edges, offs))
    dout = torch.from_numpy(out).cuda()
    _native.check(_native.lib().bcg_moment_blocks(dxt.data_ptr(), n, t, dc0.data_ptr(), de.data_ptr(), m, K,
                                                  dout.data_ptr(), do.data_ptr(), k0, k1, _native.stream_handle()),
                  "moment_blocks")
    out[lo:hi] = dout[lo:hi].cpu().numpy()


def _moment_blocks_wide(xt, col0, edges, out, offs, k0, k1) -> None:
    """n > WIDE_N variables (one sample chunk of all of them exceeds the
    moment kernel's shared-memory stage): the variable-group decomposition of
    moments._moment_raw_wide, each sub-problem's sums computed from zero and
    added element-wise into ``out`` -- the same accumulate semantics."""
    from .layout import layout
    from .moments import _moment_raw_wide

    torch = _native.torch_cuda()
    n, t = xt.shape
    K, m = col0.shape
    b = int(col0[1, m - 1]) if K >= 2 else n
    lay = layout(n, m, b) if b >= 1 else None
    if (lay is None or lay.K != K or not np.array_equal(np.asarray(lay.offs), offs)
            or not np.array_equal(np.asarray(lay.col0).reshape(K, m), col0)
            or not np.array_equal(np.asarray(lay.edges).reshape(K, m), edges)):
        raise ValueError("layout does not match _block_layout(n, m, b)")
    if t <= 0:
        return
    ldt = int(_native.lib().bcg_padded_t(t))
    dxt = torch.zeros((n, ldt), dtype=torch.float64, device="cuda")
    dxt[:, :t] = torch.from_numpy(xt).cuda()
    dout = torch.from_numpy(out).cuda()
    _moment_raw_wide(dxt, t, m, b, dout, key_range=(k0, k1))
    lo, hi = int(offs[k0]), int(offs[k1])
    out[lo:hi] = dout[lo:hi].cpu().numpy()


def naive_moment4(xt, out) -> None:
    """Accumulate the full order-4 product-sum tensor (bc/_core.pyx:151-175):
    out[i1, i2, i3, i4] += sum_l x[i1, l] x[i2, l] x[i3, l] x[i4, l].  Computed
    as the packed order-4 raw sums (b = 1) on the GPU, expanded to all n^4
    positions by copies."""
    from .moments import _moment_raw_into
    from .symtensor import BlockSymTensor
    from .layout import layout

    xt = _buffer(xt, np.float64, 2, "xt")
    out = _buffer(out, np.float64, 4, "out", writable=True)
    n, t = xt.shape
    if out.shape != (n, n, n, n):
        raise ValueError(f"out has shape {out.shape}, expected {(n, n, n, n)}")
    torch = _native.torch_cuda()
    X = torch.from_numpy(np.ascontiguousarray(xt.T)).cuda()
    raw = torch.zeros(layout(n, 4, 1).size, dtype=torch.float64, device="cuda")
    _moment_raw_into(X, 4, 1, raw)
    out += BlockSymTensor.from_packed(n, 4, 1, raw.cpu().numpy()).to_dense()
