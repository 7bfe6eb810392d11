"""Cumulant tensors via the central-moment recursion (the reference's bc/cumulants.py).

C_m = M_m - sum over min-2 partitions of products of lower cumulant blocks
(bc/cumulants.py:1-13).  The moment comes from the DMMA kernel, the
correction from the recursion kernel (csrc/recursion.cu) in place on the
packed M_m buffer; nothing leaves HBM until the caller asks for blocks.
"""

from __future__ import annotations

import os

import ctypes
from typing import Sequence

import numpy as np

from . import _native
from .errors import ValidationError
from .layout import MAX_M, enumerate_partitions_min2, layout
from .moments import (
    _center_transposed,
    _colstats,
    _device_matrix,
    _moment_device,
    _moment_device_t,
    _raise_if_nonfinite,
    _rowstats,
    as_data_matrix,
    resolve_engine,
)
from .symtensor import BlockSymTensor

CENTERING_RTOL = 1e-10  # bc/cumulants.py:26


def _check_centered_stats(sums, sumsq, t: int) -> None:
    """|mean| <= 1e-10 * rms per column (bc/cumulants.py:31-39)."""
    _check_centered_stats_host(sums.cpu().numpy(), sumsq.cpu().numpy(), t)


def _check_centered_stats_host(s, q, t: int) -> None:
    means = np.abs(s / t)
    rms = np.sqrt(q / t)
    bad = means > CENTERING_RTOL * np.maximum(rms, 1e-300)
    if bad.any():
        col = int(np.argmax(bad)) + 1
        raise ValidationError(f"data is not centered: column {col} has mean {means[col - 1]:.3e}")


def central_orders(m: int, b: int) -> tuple:
    """Central moments the order-m recursion reads besides the lower
    cumulants: the factored kernel (recursion_fact.cu, 4 <= m <= 6, b <= 8)
    at m = 6 reads M_4 of the complement (M_2 = C_2 and M_3 = C_3 are the
    cumulants themselves); every other (m, b) runs the partition sum."""
    return (4,) if m == 6 and b <= 8 else ()


def _check_centered(X) -> None:
    st = _colstats(X, sums=True, sumsq=True)
    _check_centered_stats(st["sums"], st["sumsq"], X.shape[0])


def _lower_by_order(lower: Sequence[BlockSymTensor], needed_orders) -> dict:
    by_order = {}
    for tensor in lower:
        by_order[tensor.m] = tensor
    for k in needed_orders:
        if k not in by_order:
            raise ValidationError(f"missing lower cumulant of order {k}")
    return by_order


def _lower_array(by_order: dict, m: int, n: int, b: int):
    """C array of device pointers lower[k-2] = packed C_k (NULL if absent)."""
    arr = (ctypes.c_void_p * 15)()
    keep = []
    for k in range(2, m - 1):
        t = by_order.get(k)
        if t is None:
            continue
        if (t.n, t.b) != (n, b):
            raise ValidationError(
                f"lower cumulant of order {k} has (n={t.n}, b={t.b}), expected (n={n}, b={b})"
            )
        d = t.data
        keep.append(d)
        arr[k - 2] = d.data_ptr()
    return arr, keep


def outer_prod_cum(m: int, sigma: int, lower: Sequence[BlockSymTensor],
                   per_element: bool = False) -> BlockSymTensor:
    """B_sigma: sum over min-2 partitions into sigma parts of the outer
    products of lower-cumulant sub-blocks (bc/cumulants.py:53-84).  The
    kernel is per-element already, so ``per_element`` selects the same path."""
    if not 2 <= sigma <= m // 2:
        raise ValidationError(f"sigma must be in 2..m//2={m // 2}, got {sigma}")
    partitions = enumerate_partitions_min2(m, sigma)
    needed = sorted({len(part) for parts in partitions for part in parts})
    by_order = _lower_by_order(lower, needed)
    ref = by_order[needed[0]]
    n, b = ref.n, ref.b
    torch = _native.torch_cuda()
    plan = _native.plan(n, m, b)
    arr, keep = _lower_array(by_order, m, n, b)
    out = torch.empty(layout(n, m, b).size, dtype=torch.float64, device="cuda")
    _native.check(_native.lib().bcg_outer_prod_cum(plan.handle, sigma, arr, out.data_ptr(),
                                                   _native.stream_handle()), "outer_prod_cum")
    del keep
    return BlockSymTensor(n, m, b, data=out)


def _recursion_inplace(result: BlockSymTensor, lower: Sequence[BlockSymTensor],
                       central: dict | None = None) -> None:
    """C_m in place on the packed M_m.  ``central`` (order -> packed central
    moment tensor, orders 4..m-2) enables the factored kernel at m = 6."""
    m, n, b = result.m, result.n, result.b
    by_order = _lower_by_order(lower, range(2, m - 1))
    plan = _native.plan(n, m, b)
    arr, keep = _lower_array(by_order, m, n, b)
    cm = (ctypes.c_void_p * 15)()
    for k, t in (central or {}).items():
        if 4 <= k <= m - 2:
            cm[k - 2] = t.data_ptr()
    _native.check(_native.lib().bcg_cumulant_recursion_ex(
        plan.handle, result.data.data_ptr(), arr, cm, 0, layout(n, m, b).K,
        _native.stream_handle()), "cumulant recursion")
    del keep


def cumulant(x_centered, m: int, lower: Sequence[BlockSymTensor], b: int = 2,
             engine: str = "auto") -> BlockSymTensor:
    """Order-m cumulant of centered data (bc/cumulants.py:119-136)."""
    X = as_data_matrix(x_centered)
    if m < 2:
        raise ValidationError(f"order must be >= 2, got {m}")
    _check_centered(X)
    resolve_engine(engine)
    if b < 1:
        raise ValidationError(f"block size must be >= 1, got {b}")
    if m <= 3:
        return _moment_device(X, m, b)
    _lower_by_order(lower, range(2, m - 1))
    result = _moment_device(X, m, b)
    # m = 6: the factored recursion needs the central moment M_4 of the
    # complement; it is a lower-order GEMM (cheap next to M_6) and replaces
    # the partition-sum kernel (bc/cumulants.py:119-136 either way)
    central = {k: _moment_device(X, k, b).data for k in central_orders(m, b)}
    _recursion_inplace(result, lower, central)
    return result


class CumulantSet:
    """Cumulants C_1..C_m sharing (n, b); 1-based (bc/cumulants.py:139-170)."""

    def __init__(self, c1: np.ndarray, tensors: Sequence[BlockSymTensor], b: int):
        self.c1 = np.asarray(c1, dtype=np.float64)
        self.tensors = list(tensors)
        self.n = self.c1.shape[0]
        self.b = b
        for k, tensor in enumerate(self.tensors, start=2):
            if tensor.m != k or tensor.n != self.n or tensor.b != b:
                raise ValidationError("inconsistent cumulant sequence")

    @property
    def max_order(self) -> int:
        return 1 + len(self.tensors)

    def __len__(self) -> int:
        return self.max_order

    def __getitem__(self, order: int):
        if order == 1:
            return self.c1
        if not 2 <= order <= self.max_order:
            raise KeyError(f"no cumulant of order {order}")
        return self.tensors[order - 2]

    def __repr__(self):
        return f"CumulantSet(n={self.n}, b={self.b}, orders=1..{self.max_order})"


def _central_kept(m_max: int, b: int) -> set:
    """Central moments cumulants_upto keeps (cloned before their own order's
    recursion overwrites them) for the recursions of the orders above."""
    return {j for k in range(4, m_max + 1) for j in central_orders(k, b)}


def cumulants_device(X, m_max: int, b: int, c1_host: bool = True, timer: dict | None = None):
    """Core of cumulants_upto on a device matrix: returns (c1, [C_2..C_m]).

    One colstats pass (means + finite scan), one pass that centers and
    transposes into the moment kernel's layout (the reference's xt,
    bc/_engines.py:95), one centering check, then per order one moment GEMM
    and one in-place recursion -- the reference's sequence
    (bc/cumulants.py:182-193) without its repeated validation scans.
    ``timer`` (bench.py) collects CUDA events around the top-order moment.
    """
    t, n = X.shape
    st = _colstats(X, mean=True, bad=True)
    tensors: list[BlockSymTensor] = []
    if m_max >= 2:
        xt = _center_transposed(X, st["mean"])
        sums, sq = _rowstats(xt, t)
        # the finite scan, the centering check and C_1 reach the host through
        # one non-blocking copy; the moment GEMMs are enqueued before the host
        # waits for it (validation errors are raised as before, and nothing is
        # returned for invalid data)
        flags = _stage_to_host(st["bad"], st["mean"], sums, sq)
        if timer is None and m_max >= 3 and not _SERIAL_ORDERS:
            tensors = _orders_concurrent(xt, t, m_max, b)
            return _validated_c1(X, flags, t, c1_host, st["mean"]), tensors
        central: dict = {}  # central moment M_4 kept for the factored order-6 recursion
        keep = _central_kept(m_max, b)
        for k in range(2, m_max + 1):
            if timer is not None and k == m_max:
                torch = _native.torch_cuda()
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                timer.setdefault("moment_top", []).append(ev)
                Mk = _moment_device_t(xt, t, k, b, events=ev)
            else:
                Mk = _moment_device_t(xt, t, k, b)
            if k in keep:
                central[k] = Mk.data.clone()
            if k >= 4:
                _recursion_inplace(Mk, tensors, central)
            tensors.append(Mk)
        return _validated_c1(X, flags, t, c1_host, st["mean"]), tensors
    _raise_if_nonfinite(X, st["bad"])
    c1 = st["mean"].cpu().numpy() if c1_host else st["mean"]
    return c1, tensors


def _stage_to_host(bad, mean, sums, sumsq):
    """[bad index, mean (n), row sums (n), row sums of squares (n)] copied to
    pinned host memory behind the current stream's work; returns (buffer, event)."""
    torch = _native.torch_cuda()
    dev = torch.cat([bad.to(torch.float64), mean, sums, sumsq])
    host = torch.empty(dev.shape, dtype=torch.float64, pin_memory=True)
    host.copy_(dev, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    return host, ev


def _validated_c1(X, flags, t: int, c1_host: bool, mean_dev):
    """Wait for the staged flags only (not for the work enqueued after them),
    raise the reference's validation errors, return C_1."""
    host, ev = flags
    ev.synchronize()
    v = host.numpy()
    n = X.shape[1]
    idx = int(v[0])
    if idx >= 0:
        raise ValidationError(f"non-finite value at row {idx // n + 1}, column {idx % n + 1}")
    _check_centered_stats_host(v[1 + n:1 + 2 * n], v[1 + 2 * n:1 + 3 * n], t)
    return v[1:1 + n].copy() if c1_host else mean_dev


# BCG_SERIAL_ORDERS=1: one order after the other on the current stream (A/B knob)
_SERIAL_ORDERS = os.environ.get("BCG_SERIAL_ORDERS", "0") not in ("", "0")
_side_streams: dict = {}


def _orders_concurrent(xt, t: int, m_max: int, b: int) -> list:
    """The per-order moment GEMMs only read xt, so orders 2..m-1 are issued
    on side streams and the top order on the current one: the GPU overlaps
    the small GEMMs with the big one (no per-GEMM wave tails, no idle SMs
    while a thin staircase drains).  The recursions then run in order on the
    current stream.  Every kernel is deterministic, so the results are
    bitwise those of the serial schedule."""
    torch = _native.torch_cuda()
    main = torch.cuda.current_stream()
    dev = xt.device.index if xt.device.index is not None else torch.cuda.current_device()
    ready = torch.cuda.Event()
    ready.record(main)
    moments: dict = {}
    done: dict = {}
    for k in range(2, m_max):
        key = (dev, k)
        if key not in _side_streams:
            _side_streams[key] = torch.cuda.Stream(device=dev)
        side = _side_streams[key]
        side.wait_event(ready)
        with torch.cuda.stream(side):
            moments[k] = _moment_device_t(xt, t, k, b)
            ev = torch.cuda.Event()
            ev.record(side)
        moments[k].data.record_stream(main)
        done[k] = ev
    moments[m_max] = _moment_device_t(xt, t, m_max, b)
    tensors: list[BlockSymTensor] = []
    central: dict = {}
    keep = _central_kept(m_max, b)
    for k in range(2, m_max + 1):
        if k in done:
            main.wait_event(done[k])
        Mk = moments[k]
        if k in keep:
            central[k] = Mk.data.clone()
        if k >= 4:
            _recursion_inplace(Mk, tensors, central)
        tensors.append(Mk)
    return tensors


def cumulants_upto(x, m_max: int, b: int = 2, engine: str = "auto") -> CumulantSet:
    """All cumulants of order 1..m_max of the raw data (bc/cumulants.py:173-193).
    C_1 is the raw column mean; the data is centered once on the GPU."""
    X = _device_matrix(x)
    if not 1 <= m_max <= MAX_M:
        raise ValidationError(f"m_max must be in 1..{MAX_M}, got {m_max}")
    if m_max >= 2 and X.shape[0] < 2:
        raise ValidationError("at least two samples are required for order >= 2")
    if b < 1:
        raise ValidationError(f"block size must be >= 1, got {b}")
    resolve_engine(engine)
    c1, tensors = cumulants_device(X, m_max, b)
    return CumulantSet(c1, tensors, b)
