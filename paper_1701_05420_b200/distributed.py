"""Multi-GPU cumulants: one process per GPU, torch.distributed over NCCL.

Two ways to split the work (SURVEY §8 e and §8 f row 3):

**Sample split** (``cumulants_upto_sharded``; the default, BASELINE cfg5).
The paper's Alg. 3 and the reference's ``moment_parallel``
(bc/moments.py:66-96) with the threads replaced by GPUs:

1. every rank holds a contiguous row shard (bounds t*s//p, bc/moments.py:66-68);
2. column sums are all-reduced (n doubles) -> the single global mean the
   reference's ``center`` uses (bc/cumulants.py:190); each rank centers its shard;
3. per order k: local packed RAW sums (the DMMA GEMM), then
   * orders the later recursions read (k <= m-2): NCCL all-reduce(SUM) ->
     / t_total -> every rank runs the (microsecond-scale) recursion on all
     blocks, so C_k (and the central moment M_k the factored recursion needs)
     is replicated without a second collective;
   * the two top orders (k >= m-1, k >= 4): the packed buffer is padded to
     world equal element spans; an in-place NCCL reduce-scatter leaves each
     rank its span fully reduced -> / t_total -> the recursion on that span
     (per element it reads only its own M_k element and the replicated lower
     orders; the at most two blocks a span cuts run with masked writes) ->
     an in-place all-gather: 2x the packed size on the wire instead of the 3x
     of all-reduce + all-gather, and no staging copy of the packed tensor
     (cfg5: C6 is 20 GB).

**Block split** (``cumulants_upto_block_split``; ``moment_parallel_blocks``,
bc/moments.py:99-131, across GPUs).  Every rank holds ALL of X; rank r
computes blocks [K r/W, K (r+1)/W) of every order (moment + recursion) and one
in-place broadcast per rank of its block range rebuilds C_k.  No moment collective, no partial M_k per
GPU (cfg5: 20 GB less per GPU), X read W times in total; results bitwise equal
to the single-GPU path (every key range of the moment kernel sums in the same
order).

The per-rank compute goes through an ``ops`` object; the default is the
sm_100a library.  (The CPU multi-process tests substitute the oracle for it to
exercise the collective logic over gloo.)
"""

from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist

from .errors import ValidationError
from .layout import MAX_M, layout


def shard_bounds(t: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row shard of rank ``rank`` (bc/moments.py:66-68)."""
    return t * rank // world, t * (rank + 1) // world


def block_bounds(K: int, world: int, rank: int) -> tuple[int, int]:
    """Block-list split of the recursion (bc/moments.py:118)."""
    return K * rank // world, K * (rank + 1) // world


class CudaOps:
    """Per-rank compute on the sm_100a library (the product path)."""

    def __init__(self):
        from . import _native

        _native.torch_cuda()

    def matrix(self, x):
        from .moments import _device_matrix

        return _device_matrix(x)

    def colstats(self, X):
        """(sums, sumsq, first_bad) of the local shard as device tensors."""
        from .moments import _colstats

        st = _colstats(X, sums=True, sumsq=True, bad=True)
        return st["sums"], st["sumsq"], st["bad"]

    def colmean(self, X):
        """(mean, first_bad) of the whole matrix, as cumulants_upto computes them."""
        from .moments import _colstats

        st = _colstats(X, mean=True, bad=True)
        return st["mean"], st["bad"]

    def center(self, X, mean):
        """Centered data in the moment kernel's transposed layout: (xt, t)."""
        from .moments import _center_transposed

        return _center_transposed(X, mean), X.shape[0]

    def centered_stats(self, centered):
        from .moments import _rowstats

        return _rowstats(*centered)

    def moment_raw(self, centered, k: int, b: int, key_range=None, size=None):
        """Packed RAW order-k sums (all blocks, or blocks [k0, k1) only; the
        rest of the buffer stays zero) in a buffer of ``size`` >= S_k
        elements (zero past S_k: padding for the equal-span collectives)."""
        from . import _native

        from .moments import WIDE_N, _moment_raw_wide

        xt, t = centered
        n, ldt = xt.shape
        S = layout(n, k, b).size
        out = torch.zeros(max(S, size or 0), dtype=torch.float64, device=xt.device)
        if n > WIDE_N:
            _moment_raw_wide(xt, t, k, b, out[:S], key_range)
            return out
        plan = _native.plan(n, k, b)
        wsb = plan.t_ws_bytes(t)  # split-K partials only: xt is already transposed
        ws = torch.empty(wsb, dtype=torch.uint8, device=xt.device) if wsb else None
        wsp = ws.data_ptr() if ws is not None else None
        lib = _native.lib()
        if key_range is None:
            rc = lib.bcg_moment_raw_t(plan.handle, xt.data_ptr(), t, ldt, out.data_ptr(), wsp, wsb,
                                      _native.stream_handle())
        else:
            rc = lib.bcg_moment_raw_t_range(plan.handle, xt.data_ptr(), t, ldt, out.data_ptr(), wsp, wsb,
                                            int(key_range[0]), int(key_range[1]), _native.stream_handle())
        _native.check(rc, "moment")
        return out

    def divide(self, buf, t: int):
        from .moments import _divide

        _divide(buf, t)

    @staticmethod
    def _pointer_arrays(lower: dict, central, k: int):
        import ctypes

        arr = (ctypes.c_void_p * 15)()
        for j, t in lower.items():
            arr[j - 2] = t.data_ptr()
        cm = (ctypes.c_void_p * 15)()
        for j, t in (central or {}).items():
            if 4 <= j <= k - 2:
                cm[j - 2] = t.data_ptr()
        return arr, cm

    def recursion_span(self, mk, n: int, k: int, b: int, lower: dict, e0: int, e1: int, central=None):
        """C_k in place on the ELEMENTS mk[e0:e1) (bcg_cumulant_recursion_span)."""
        from . import _native

        plan = _native.plan(n, k, b)
        arr, cm = self._pointer_arrays(lower, central, k)
        _native.check(_native.lib().bcg_cumulant_recursion_span(
            plan.handle, mk.data_ptr(), arr, cm, int(e0), int(e1), _native.stream_handle()), "recursion")

    def recursion_range(self, mk, n: int, k: int, b: int, lower: dict, k0: int, k1: int, central=None):
        """C_k in place on blocks [k0, k1) of the packed M_k.  ``central``
        (order -> packed central moment, orders 4..k-2) selects the factored
        kernel at k >= 6 (bcg_cumulant_recursion_ex)."""
        import ctypes

        from . import _native

        plan = _native.plan(n, k, b)
        arr = (ctypes.c_void_p * 15)()
        for j, t in lower.items():
            arr[j - 2] = t.data_ptr()
        cm = (ctypes.c_void_p * 15)()
        for j, t in (central or {}).items():
            if 4 <= j <= k - 2:
                cm[j - 2] = t.data_ptr()
        _native.check(_native.lib().bcg_cumulant_recursion_ex(
            plan.handle, mk.data_ptr(), arr, cm, int(k0), int(k1), _native.stream_handle()), "recursion")


def _central_kept(m_max: int, b: int) -> set:
    from .cumulants import _central_kept as kept

    return kept(m_max, b)


def _check_centered(sums, sumsq, t: int):
    from .cumulants import _check_centered_stats

    _check_centered_stats(sums, sumsq, t)


def cumulants_upto_sharded(x_local, m_max: int, b: int = 2, group=None, ops=None,
                           timer: Optional[dict] = None):
    """Cumulants C_1..C_m of the row-concatenation of every rank's shard.

    Collective: every rank must call it with its own contiguous shard (same
    n, m_max, b).  Returns (c1, [C_2..C_m]) as tensors on the rank's device,
    identical on every rank; wrap with ``CumulantSet`` via
    ``to_cumulant_set``.  ``timer`` (optional) collects CUDA events around the
    top-order moment launches for bench.py.
    """
    if not 1 <= m_max <= MAX_M:
        raise ValidationError(f"m_max must be in 1..{MAX_M}, got {m_max}")
    ops = ops or CudaOps()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    X = ops.matrix(x_local)
    t_local, n = X.shape
    sums, _, bad = ops.colstats(X)
    # one small all-reduce: column sums, row count and a non-finite flag
    # (the flag stays on the device: no host sync before the collective)
    head = torch.cat([sums, torch.tensor([float(t_local)], dtype=torch.float64, device=sums.device),
                      (bad.reshape(-1)[:1] >= 0).to(device=sums.device, dtype=torch.float64)])
    dist.all_reduce(head, group=group)
    if head[n + 1].item() > 0:
        raise ValidationError(f"non-finite value in the data shard of some rank (this rank: {int(bad.item()) >= 0})")
    t_total = int(round(head[n].item()))
    if m_max >= 2 and t_total < 2:
        raise ValidationError("at least two samples are required for order >= 2")
    mean = head[:n] / t_total if not isinstance(ops, CudaOps) else _device_div(head[:n].contiguous(), t_total, ops)
    tensors = []
    if m_max >= 2:
        Xc = ops.center(X, mean)
        csum, csq = ops.centered_stats(Xc)
        both = torch.cat([csum, csq])
        dist.all_reduce(both, group=group)
        _check_centered(both[:n], both[n:], t_total)
        lower: dict = {}
        central: dict = {}  # central moment M_4 (factored order-6 recursion)
        keep = _central_kept(m_max, b)
        # all moment GEMMs only read Xc: issue them up front (lower orders on
        # side streams), so each order's collective overlaps the GEMMs still
        # running -- the top order's in particular
        # the two top orders (k >= 4) are split by element span: their
        # buffers are padded to world x span so the collectives run in place
        S = {k: layout(n, k, b).size for k in range(2, m_max + 1)}
        split = {k for k in range(4, m_max + 1) if world > 1 and k >= m_max - 1 and k not in keep}
        size = {k: (_padded(S[k], world) if k in split else S[k]) for k in S}
        early = _issue_moments(ops, Xc, m_max, b, size) if timer is None else {}
        for k in range(2, m_max + 1):
            top = k == m_max and timer is not None
            if top:
                ev0 = torch.cuda.Event(enable_timing=True)
                ev1 = torch.cuda.Event(enable_timing=True)
                ev0.record()
            if k in early:
                mk, ev = early[k]
                if ev is not None:
                    torch.cuda.current_stream().wait_event(ev)
            else:
                mk = ops.moment_raw(Xc, k, b, size=size[k])
            if top:
                ev1.record()
                timer.setdefault("moment_top", []).append((ev0, ev1))
            if k in split:
                # reduce-scatter (in place) -> this rank's element span fully
                # reduced -> / t -> recursion on the span -> all-gather (in place)
                c = size[k] // world
                e0, e1 = rank * c, min((rank + 1) * c, S[k])
                _reduce_scatter_inplace(mk, c, rank, group)
                ops.divide(mk[e0:e1], t_total)
                ops.recursion_span(mk, n, k, b, lower, e0, e1, central)
                _all_gather_inplace(mk, c, rank, group)
                mk = mk[:S[k]]
            else:
                if world > 1:
                    dist.all_reduce(mk, group=group)
                ops.divide(mk, t_total)
                if k in keep:
                    central[k] = mk.clone()
                if k >= 4:
                    ops.recursion_range(mk, n, k, b, lower, 0, layout(n, k, b).K, central)
            lower[k] = mk
            tensors.append(mk)
    return mean, tensors


def cumulants_upto_block_split(x_full, m_max: int, b: int = 2, group=None, ops=None,
                               timer: Optional[dict] = None):
    """Cumulants C_1..C_m of ``x_full`` (the SAME full matrix on every rank),
    split by block list across ranks: rank r computes the moments and the
    recursion of blocks [K r/W, K (r+1)/W) of every order; an all-gather per
    order rebuilds C_k on every rank.  Collective; returns (c1, [C_2..C_m]),
    bitwise identical to the single-GPU ``cumulants_upto``."""
    if not 1 <= m_max <= MAX_M:
        raise ValidationError(f"m_max must be in 1..{MAX_M}, got {m_max}")
    ops = ops or CudaOps()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    X = ops.matrix(x_full)
    t, n = X.shape
    mean, bad = ops.colmean(X)
    if int(bad.item()) >= 0:
        i = int(bad.item())
        raise ValidationError(f"non-finite value at row {i // n + 1}, column {i % n + 1}")
    if m_max >= 2 and t < 2:
        raise ValidationError("at least two samples are required for order >= 2")
    tensors = []
    if m_max >= 2:
        Xc = ops.center(X, mean)
        csum, csq = ops.centered_stats(Xc)
        _check_centered(csum, csq, t)
        lower: dict = {}
        central: dict = {}
        keep = _central_kept(m_max, b)
        for k in range(2, m_max + 1):
            lay = layout(n, k, b)
            k0, k1 = block_bounds(lay.K, world, rank)
            top = k == m_max and timer is not None
            if top:
                ev0 = torch.cuda.Event(enable_timing=True)
                ev1 = torch.cuda.Event(enable_timing=True)
                ev0.record()
            mk = ops.moment_raw(Xc, k, b, key_range=(k0, k1))
            if top:
                ev1.record()
                timer.setdefault("moment_top", []).append((ev0, ev1))
            lo, hi = int(lay.offs[k0]), int(lay.offs[k1])
            ops.divide(mk[lo:hi], t)
            if k in keep:
                # the factored recursion of higher orders reads the central
                # moment of every block: gather it before correcting in place
                if world > 1:
                    _broadcast_block_ranges(mk, lay, world, group)
                central[k] = mk.clone()
            if k >= 4:
                ops.recursion_range(mk, n, k, b, lower, k0, k1, central)
            if world > 1:
                _broadcast_block_ranges(mk, lay, world, group)
            lower[k] = mk
            tensors.append(mk)
    return mean, tensors


def _issue_moments(ops, centered, m_max: int, b: int, size: dict) -> dict:
    """Orders 2..m-1 on per-order side streams, the top order on the current
    stream; returns {k: (raw sums, event or None)}.  CUDA ops only (the CPU
    test ops run serially); BCG_SERIAL_ORDERS=1 disables it."""
    from .cumulants import _SERIAL_ORDERS, _side_streams

    if not isinstance(ops, CudaOps) or m_max < 3 or _SERIAL_ORDERS:
        return {}
    main = torch.cuda.current_stream()
    dev = centered[0].device.index if centered[0].device.index is not None else torch.cuda.current_device()
    ready = torch.cuda.Event()
    ready.record(main)
    out: dict = {}
    for k in range(2, m_max):
        key = (dev, k)
        if key not in _side_streams:
            _side_streams[key] = torch.cuda.Stream(device=dev)
        side = _side_streams[key]
        side.wait_event(ready)
        with torch.cuda.stream(side):
            mk = ops.moment_raw(centered, k, b, size=size[k])
            ev = torch.cuda.Event()
            ev.record(side)
        mk.record_stream(main)
        out[k] = (mk, ev)
    out[m_max] = (ops.moment_raw(centered, m_max, b, size=size[m_max]), None)
    return out


def _device_div(v, t, ops):
    ops.divide(v, t)
    return v


def _padded(S: int, world: int) -> int:
    """Packed size rounded up to world equal element spans."""
    return -(-S // world) * world


def _nccl(group) -> bool:
    return dist.get_backend(group) == "nccl"


def _reduce_scatter_inplace(buf, c: int, rank: int, group) -> None:
    """Sum ``buf`` (world x c elements) over ranks into this rank's span
    buf[rank c : (rank + 1) c].  NCCL runs it in place (receive buffer = send
    buffer + rank x count): no staging copy of the packed tensor.  (gloo, the
    CPU tests' backend, gets a staging buffer.)"""
    own = buf[rank * c:(rank + 1) * c]
    if _nccl(group):
        dist.reduce_scatter_tensor(own, buf, group=group)
    else:
        tmp = torch.empty_like(own)
        dist.reduce_scatter_tensor(tmp, buf, group=group)
        own.copy_(tmp)


def _all_gather_inplace(buf, c: int, rank: int, group) -> None:
    """Every rank's span of ``buf`` to every rank; NCCL in place (send
    buffer = receive buffer + rank x count)."""
    own = buf[rank * c:(rank + 1) * c]
    if _nccl(group):
        dist.all_gather_into_tensor(buf, own, group=group)
    else:
        tmp = torch.empty_like(buf)
        dist.all_gather_into_tensor(tmp, own.clone(), group=group)
        buf.copy_(tmp)


def _broadcast_block_ranges(mk, lay, world: int, group) -> None:
    """Rebuild the full packed tensor from each rank's block range: one
    in-place broadcast per rank of its contiguous range (uneven ranges, no
    padding, no staging copies)."""
    for r in range(world):
        k0, k1 = block_bounds(lay.K, world, r)
        lo, hi = int(lay.offs[k0]), int(lay.offs[k1])
        if hi > lo:
            src = r if group is None else dist.get_global_rank(group, r)
            dist.broadcast(mk[lo:hi], src=src, group=group)


def to_cumulant_set(mean, tensors, n: int, b: int):
    from .cumulants import CumulantSet
    from .symtensor import BlockSymTensor

    ts = [BlockSymTensor(n, k, b, data=t) if t.is_cuda else BlockSymTensor(n, k, b, host=t.numpy())
          for k, t in enumerate(tensors, start=2)]
    return CumulantSet(mean.cpu().numpy(), ts, b)
