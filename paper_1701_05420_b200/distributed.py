"""Multi-GPU cumulants: the sample axis t sharded across ranks (one process per
GPU, torch.distributed over NCCL).

This is the paper's Alg. 3 and the reference's
sample-split ``moment_parallel`` (bc/moments.py:66-96) with the threads
replaced by GPUs and the Python reduction loop by collectives:

1. every rank holds a contiguous row shard (bounds t*s//p, bc/moments.py:66-68);
2. column sums are all-reduced (n doubles) -> the single global mean the
   reference's ``center`` uses (bc/cumulants.py:190); each rank centers its shard;
3. per order k: local packed RAW sums (the DMMA GEMM) -> NCCL all-reduce(SUM)
   -> / t_total, i.e. the global central moment M_k on every rank;
4. the recursion is split by block list (bc/moments.py:114-131): rank r
   corrects blocks [K r/W, K (r+1)/W) in place and an all-gather rebuilds C_k
   everywhere (the next order's recursion reads every block of it).

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

    def center(self, X, mean):
        """Centered data in the moment kernel's transposed layout: (xt, t)."""
        from .moments import _center_transposed

        return _center_transposed(X, mean), X.shape[0]

    def centered_stats(self, centered):
        from .moments import _rowstats

        return _rowstats(*centered)

    def moment_raw(self, centered, k: int, b: int):
        from .moments import _moment_raw_t_into

        xt, t = centered
        out = torch.zeros(layout(xt.shape[0], k, b).size, dtype=torch.float64, device=xt.device)
        _moment_raw_t_into(xt, t, k, b, out)
        return out

    def divide(self, buf, t: int):
        from .moments import _divide

        _divide(buf, t)

    def recursion_range(self, mk, n: int, k: int, b: int, lower: dict, k0: int, k1: int):
        import ctypes

        from . import _native

        plan = _native.plan(n, k, b)
        arr = (ctypes.c_void_p * 15)()
        for j, t in lower.items():
            arr[j - 2] = t.data_ptr()
        _native.check(_native.lib().bcg_cumulant_recursion_range(
            plan.handle, mk.data_ptr(), arr, int(k0), int(k1), _native.stream_handle()), "recursion")


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
    head = torch.cat([sums, torch.tensor([float(t_local), 0.0], dtype=torch.float64, device=sums.device)])
    head[n + 1] = float(int(bad.item()) >= 0)
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
        for k in range(2, m_max + 1):
            top = k == m_max and timer is not None
            if top:
                ev0 = torch.cuda.Event(enable_timing=True)
                ev1 = torch.cuda.Event(enable_timing=True)
                ev0.record()
            mk = ops.moment_raw(Xc, k, b)
            if top:
                ev1.record()
                timer.setdefault("moment_top", []).append((ev0, ev1))
            if world > 1:
                dist.all_reduce(mk, group=group)
            ops.divide(mk, t_total)
            if k >= 4:
                lay = layout(n, k, b)
                if world == 1:
                    ops.recursion_range(mk, n, k, b, lower, 0, lay.K)
                else:
                    k0, k1 = block_bounds(lay.K, world, rank)
                    ops.recursion_range(mk, n, k, b, lower, k0, k1)
                    _allgather_blocks(mk, lay, world, group)
            lower[k] = mk
            tensors.append(mk)
    return mean, tensors


def _device_div(v, t, ops):
    ops.divide(v, t)
    return v


def _allgather_blocks(mk, lay, world: int, group) -> None:
    """Rebuild the full packed tensor from each rank's block range."""
    spans = []
    for r in range(world):
        k0, k1 = block_bounds(lay.K, world, r)
        spans.append((int(lay.offs[k0]), int(lay.offs[k1])))
    width = max(hi - lo for lo, hi in spans)
    rank = dist.get_rank(group)
    lo, hi = spans[rank]
    send = torch.zeros(width, dtype=mk.dtype, device=mk.device)
    send[: hi - lo] = mk[lo:hi]
    recv = torch.empty(width * world, dtype=mk.dtype, device=mk.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    for r, (a, z) in enumerate(spans):
        if r != rank:
            mk[a:z] = recv[r * width: r * width + (z - a)]


def to_cumulant_set(mean, tensors, n: int, b: int):
    from .cumulants import CumulantSet
    from .symtensor import BlockSymTensor

    ts = [BlockSymTensor(n, k, b, data=t) if t.is_cuda else BlockSymTensor(n, k, b, host=t.numpy())
          for k, t in enumerate(tensors, start=2)]
    return CumulantSet(mean.cpu().numpy(), ts, b)
