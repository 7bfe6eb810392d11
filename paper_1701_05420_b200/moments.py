"""Centering and packed moment tensors on the GPU (the reference's bc/moments.py).

Same entry points, arguments and errors as the reference; the data matrix
lives in HBM as a C-contiguous (t x n) float64 torch tensor and every pass
over it is one of our sm_100a kernels (csrc/), reached through the C ABI
(include/bcgpu.h).  All estimators normalise by the raw sample count t
(bc/moments.py:1-7).
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import ValidationError
from .symtensor import BlockSymTensor
from .layout import layout

ENGINES = ("auto", "compiled", "gram", "blockwise", "cuda")
PARALLEL_STRATEGIES = ("none", "samples", "blocks")


def resolve_engine(engine: str) -> str:
    """The reference's engine names (bc/_engines.py:33-43) are accepted for
    signature compatibility; all of them run the single sm_100a backend."""
    if engine not in ENGINES:
        raise ValidationError(f"unknown engine {engine!r}, expected one of {ENGINES}")
    return "cuda"


# -- data matrix ---------------------------------------------------------------


def _device_matrix(x):
    """(t, n) C-contiguous float64 CUDA tensor of x (shape checks of
    bc/moments.py:25-29, no finite scan)."""
    torch = _native.torch_cuda()
    if isinstance(x, torch.Tensor):
        if x.ndim != 2:
            raise ValidationError(f"data must be 2-D (t x n), got shape {tuple(x.shape)}")
        t = x.to(device="cuda", dtype=torch.float64)
        if not t.is_contiguous():
            t = t.contiguous()
    else:
        arr = np.ascontiguousarray(x, dtype=np.float64)
        if arr.ndim != 2:
            raise ValidationError(f"data must be 2-D (t x n), got shape {arr.shape}")
        t = torch.from_numpy(arr).to("cuda")
    if t.shape[0] < 1 or t.shape[1] < 1:
        raise ValidationError(f"data must be non-empty, got shape {tuple(t.shape)}")
    return t


def _colstats(X, sums=False, mean=False, sumsq=False, bad=False):
    """One deterministic pass over X (bcg_colstats): column sums / means /
    sums of squares and the first non-finite position."""
    torch = _native.torch_cuda()
    t, n = X.shape
    outs = {}
    for name, want in (("sums", sums), ("mean", mean), ("sumsq", sumsq)):
        outs[name] = torch.empty(n, dtype=torch.float64, device=X.device) if want else None
    outs["bad"] = torch.empty(1, dtype=torch.int64, device=X.device) if bad else None
    lib = _native.lib()
    wsb = lib.bcg_colstats_ws_bytes(t, n)
    ws = torch.empty(wsb, dtype=torch.uint8, device=X.device)
    p = lambda v: v.data_ptr() if v is not None else None  # noqa: E731
    _native.check(lib.bcg_colstats(
        X.data_ptr(), t, n, n, p(outs["sums"]), p(outs["mean"]), p(outs["sumsq"]), p(outs["bad"]),
        ws.data_ptr(), wsb, _native.stream_handle()), "colstats")
    return outs


def _raise_if_nonfinite(X, bad) -> None:
    idx = int(bad.item())
    if idx >= 0:
        n = X.shape[1]
        raise ValidationError(f"non-finite value at row {idx // n + 1}, column {idx % n + 1}")


def as_data_matrix(x):
    """Validate and coerce a t x n observation matrix of finite float64
    (bc/moments.py:23-35).  Returns the CUDA tensor the kernels read."""
    X = _device_matrix(x)
    st = _colstats(X, bad=True)
    _raise_if_nonfinite(X, st["bad"])
    return X


def _center_device(X, mean):
    torch = _native.torch_cuda()
    t, n = X.shape
    out = torch.empty_like(X)
    _native.check(_native.lib().bcg_center(X.data_ptr(), t, n, n, mean.data_ptr(), out.data_ptr(),
                                           _native.stream_handle()), "center")
    return out


def center(x):
    """Subtract each column's mean (bc/moments.py:38-41); returns a CUDA tensor."""
    X = _device_matrix(x)
    st = _colstats(X, mean=True, bad=True)
    _raise_if_nonfinite(X, st["bad"])
    return _center_device(X, st["mean"])


# -- moments ---------------------------------------------------------------------


# The moment kernel stages a sample chunk of ALL variables in shared memory,
# which bounds n (K2).  Wider data is decomposed by variable groups:
# the key set splits by which groups its blocks fall in; every set S of at
# most m groups is one sub-problem over the columns of S's blocks (<= WIDE_N
# variables), whose keys that touch exactly the groups of S are scattered into
# the global packed buffer.  Per element the products, their association and
# the sample order are those of a kernel launch over the sub-matrix, so the
# result is deterministic and the same for every caller (moment, cumulants_upto,
# the multi-GPU paths) -- the bitwise invariants hold.
WIDE_N = 720


def _multiset_ranks(keys: np.ndarray, N: int) -> np.ndarray:
    """Lexicographic rank of sorted 1-based keys (rows) among all size-m
    multisets over 1..N: sum over positions of the multisets that branch off
    below (hockey-stick sums of C(N - v + L, L))."""
    K, m = keys.shape
    comb = np.zeros((N + m + 2, m + 1), dtype=np.int64)
    cap = 1 << 62  # entries this large are never reached by a layout that fits in memory
    for a in range(N + m + 2):
        comb[a, 0] = 1
        for k in range(1, min(a, m) + 1):
            comb[a, k] = min(cap, int(comb[a - 1, k - 1]) + int(comb[a - 1, k]))
    rank = np.zeros(K, dtype=np.int64)
    prev = np.ones(K, dtype=np.int64)
    for q in range(m):
        L = m - q - 1
        j = keys[:, q]
        rank += comb[N - prev + L + 1, L + 1] - comb[N - j + L + 1, L + 1]
        prev = j
    return rank


def _ranges(starts: np.ndarray, lengths: np.ndarray) -> np.ndarray:
    """Concatenation of arange(s, s + l) over (s, l) pairs."""
    total = int(lengths.sum())
    first = np.repeat(np.cumsum(lengths) - lengths, lengths)
    return np.repeat(starts, lengths) + (np.arange(total, dtype=np.int64) - first)


def _moment_raw_wide(xt, t: int, m: int, b: int, out, key_range=None) -> None:
    """Accumulate packed RAW order-m sums of the transposed data xt (n > WIDE_N)
    into out, via variable-group sub-problems (keys in ``key_range`` only)."""
    import itertools

    torch = _native.torch_cuda()
    n = xt.shape[0]
    nb = -(-n // b)
    gsz = WIDE_N // (m * b)
    if gsz < 1:
        raise ValidationError(f"block size b={b} too large for order {m} on {n} variables "
                              f"(m * b must be <= {WIDE_N})")
    groups = [np.arange(g0 + 1, min(nb, g0 + gsz) + 1) for g0 in range(0, nb, gsz)]
    goffs = layout(n, m, b).offs
    k0, k1 = (0, len(goffs) - 1) if key_range is None else (int(key_range[0]), int(key_range[1]))
    for size in range(1, m + 1):
        for S in itertools.combinations(range(len(groups)), size):
            blocks = np.concatenate([groups[g] for g in S])          # ascending global block ids
            group_of = np.concatenate([np.full(len(groups[g]), i) for i, g in enumerate(S)])
            cols = np.concatenate([np.arange((j - 1) * b, min(j * b, n)) for j in blocks])
            slay = layout(len(cols), m, b)
            skeys = np.asarray(slay.keys, dtype=np.int64).reshape(-1, m)
            gkeys = blocks[skeys - 1]
            # keys touching every group of S (fewer: another sub-problem's)
            gsets = np.sort(group_of[skeys - 1], axis=1)
            ndist = 1 + (np.diff(gsets, axis=1) != 0).sum(axis=1)
            gk = _multiset_ranks(gkeys, nb)
            keep = (ndist == size) & (gk >= k0) & (gk < k1)
            if not keep.any():
                continue
            sk = np.nonzero(keep)[0]
            lengths = slay.offs[sk + 1] - slay.offs[sk]
            src = torch.from_numpy(_ranges(slay.offs[sk], lengths)).to(xt.device)
            dst = torch.from_numpy(_ranges(goffs[gk[keep]], lengths)).to(xt.device)
            sub_xt = xt[torch.from_numpy(cols).to(xt.device)]
            sub = torch.zeros(slay.size, dtype=torch.float64, device=xt.device)
            _moment_raw_t_into(sub_xt, t, m, b, sub)
            out.index_put_((dst,), sub[src], accumulate=True)  # unique targets: deterministic


def _moment_raw_into(X, m: int, b: int, out, key_range=None) -> None:
    """Accumulate packed RAW order-m sums of X into out (bcg_moment_raw)."""
    torch = _native.torch_cuda()
    t, n = X.shape
    if n > WIDE_N:
        _moment_raw_wide(_center_transposed(X, None), t, m, b, out, key_range)
        return
    plan = _native.plan(n, m, b)
    wsb = plan.ws_bytes(t)
    ws = torch.empty(wsb, dtype=torch.uint8, device=X.device) if wsb else None
    lib = _native.lib()
    wsp = ws.data_ptr() if ws is not None else None
    if key_range is None:
        rc = lib.bcg_moment_raw(plan.handle, X.data_ptr(), t, n, out.data_ptr(), wsp, wsb,
                                _native.stream_handle())
    else:
        rc = lib.bcg_moment_raw_range(plan.handle, X.data_ptr(), t, n, out.data_ptr(), wsp, wsb,
                                      int(key_range[0]), int(key_range[1]), _native.stream_handle())
    _native.check(rc, "moment")


def _center_transposed(X, mean):
    """Xc^T: centered (mean may be None) and transposed into the moment
    kernel's padded layout (n x padded_t(t)) in one pass (bcg_transpose_pad)."""
    torch = _native.torch_cuda()
    t, n = X.shape
    lib = _native.lib()
    ldt = int(lib.bcg_padded_t(t))
    xt = torch.empty((n, ldt), dtype=torch.float64, device=X.device)
    _native.check(lib.bcg_transpose_pad(X.data_ptr(), t, n, n, mean.data_ptr() if mean is not None else None,
                                        xt.data_ptr(), ldt, _native.stream_handle()), "center")
    return xt


def _rowstats(xt, t: int):
    """Column sums / sums of squares of the data from its transposed layout."""
    torch = _native.torch_cuda()
    n, ldt = xt.shape
    lib = _native.lib()
    wsb = int(lib.bcg_rowstats_ws_bytes(n, t))
    buf = torch.empty(2 * n + wsb // 8, dtype=torch.float64, device=xt.device)
    sums, sq, ws = buf[:n], buf[n:2 * n], buf[2 * n:]
    _native.check(lib.bcg_rowstats_ws(xt.data_ptr(), n, t, ldt, sums.data_ptr(), sq.data_ptr(), ws.data_ptr(), wsb,
                                      _native.stream_handle()), "rowstats")
    return sums, sq


def _moment_raw_t_into(xt, t: int, m: int, b: int, out) -> None:
    """Accumulate packed RAW order-m sums from the transposed layout."""
    torch = _native.torch_cuda()
    n, ldt = xt.shape
    if n > WIDE_N:
        _moment_raw_wide(xt, t, m, b, out)
        return
    plan = _native.plan(n, m, b)
    wsb = plan.t_ws_bytes(t)  # split-K partials only: xt is already transposed
    ws = torch.empty(wsb, dtype=torch.uint8, device=xt.device) if wsb else None
    _native.check(_native.lib().bcg_moment_raw_t(plan.handle, xt.data_ptr(), t, ldt, out.data_ptr(),
                                                 ws.data_ptr() if ws is not None else None, wsb,
                                                 _native.stream_handle()), "moment")


def _moment_device_t(xt, t: int, m: int, b: int, events=None) -> BlockSymTensor:
    """Order-m moment from the transposed layout (m >= 2)."""
    torch = _native.torch_cuda()
    n = xt.shape[0]
    out = torch.zeros(layout(n, m, b).size, dtype=torch.float64, device=xt.device)
    if events is not None:
        events[0].record()
    _moment_raw_t_into(xt, t, m, b, out)
    if events is not None:
        events[1].record()
    _divide(out, t)
    return BlockSymTensor(n, m, b, data=out)


def _divide(buf, t: int) -> None:
    _native.check(_native.lib().bcg_div(buf.numel(), buf.data_ptr(), float(t), buf.data_ptr(),
                                        _native.stream_handle()), "scale")


def _moment_device(X, m: int, b: int, events=None) -> BlockSymTensor:
    """Order-m moment of a validated device matrix (m >= 2).  ``events``:
    optional (start, end) CUDA events recorded around the GEMM launch(es)."""
    torch = _native.torch_cuda()
    t, n = X.shape
    out = torch.zeros(layout(n, m, b).size, dtype=torch.float64, device=X.device)
    if events is not None:
        events[0].record()
    _moment_raw_into(X, m, b, out)
    if events is not None:
        events[1].record()
    _divide(out, t)  # the reference's `out /= t` (bc/_engines.py:99)
    return BlockSymTensor(n, m, b, data=out)


def _means_tensor(X, b: int) -> BlockSymTensor:
    st = _colstats(X, mean=True)
    return BlockSymTensor(X.shape[1], 1, b, data=st["mean"])


def moment(x, m: int, b: int = 2, engine: str = "auto") -> BlockSymTensor:
    """Order-m moment tensor in block storage (bc/moments.py:44-63)."""
    X = as_data_matrix(x)
    if m < 1:
        raise ValidationError(f"order must be >= 1, got {m}")
    if b < 1:
        raise ValidationError(f"block size must be >= 1, got {b}")
    if m == 1:
        return _means_tensor(X, b)
    resolve_engine(engine)
    if m > 16:
        raise ValidationError("kernel supports 2 <= m <= 16")
    return _moment_device(X, m, b)


def moment_block(x, key, b: int) -> np.ndarray:
    """One dense block of the moment tensor (bc/_engines.py:216-232), from
    the same kernel restricted to that block."""
    X = as_data_matrix(x)
    t, n = X.shape
    m = len(key)
    if list(key) != sorted(key):
        raise ValidationError(f"block index {tuple(key)} is not sorted")
    n_bar = -(-n // b)
    if any(j < 1 or j > n_bar for j in key):
        raise ValidationError(f"block index {tuple(key)} out of range 1..{n_bar}")
    if m == 1:
        means = _means_tensor(X, b).packed_host()
        return means[(key[0] - 1) * b:min(key[0] * b, n)].copy()
    torch = _native.torch_cuda()
    lay = layout(n, m, b)
    k = lay.key_index(tuple(key))
    out = torch.zeros(lay.size, dtype=torch.float64, device=X.device)
    _moment_raw_into(X, m, b, out, key_range=(k, k + 1))
    blk = out[int(lay.offs[k]):int(lay.offs[k + 1])].clone()
    _divide(blk, t)
    return blk.cpu().numpy().reshape(tuple(lay.edges[k]))


def _chunk_bounds(t: int, p: int):
    bounds = [t * s // p for s in range(p + 1)]
    return [(bounds[s], bounds[s + 1]) for s in range(p)]


def moment_parallel(x, m: int, b: int = 2, p: int = 1, engine: str = "auto") -> BlockSymTensor:
    """Sample-split moment (bc/moments.py:71-96): contiguous chunks t*s//p,
    each chunk's moment, combined as sum_s part_s * (t_s / t) in chunk order.
    p = 1 is exactly `moment`.  (Across GPUs: see distributed.py.)"""
    X = as_data_matrix(x)
    t = X.shape[0]
    if p < 1:
        raise ValidationError(f"worker count must be >= 1, got {p}")
    if p > t:
        raise ValidationError(f"cannot split {t} rows into {p} non-empty chunks")
    if p == 1:
        return moment(X, m, b, engine)
    chunks = _chunk_bounds(t, p)
    parts = [moment(X[lo:hi], m, b, engine) for lo, hi in chunks]
    total = parts[0].scale((chunks[0][1] - chunks[0][0]) / t)
    for (lo, hi), part in zip(chunks[1:], parts[1:]):
        total = total._axpby(1.0, (hi - lo) / t, part)  # total + part.scale(w), same roundings
    return total


def moment_parallel_blocks(x, m: int, b: int = 2, p: int = 1, engine: str = "auto") -> BlockSymTensor:
    """Block-split moment (bc/moments.py:99-131): p disjoint key ranges
    filling one packed buffer; bitwise identical to `moment`."""
    X = as_data_matrix(x)
    if p < 1:
        raise ValidationError(f"worker count must be >= 1, got {p}")
    if m == 1 or p == 1:
        return moment(X, m, b, engine)
    resolve_engine(engine)
    torch = _native.torch_cuda()
    t, n = X.shape
    lay = layout(n, m, b)
    out = torch.zeros(lay.size, dtype=torch.float64, device=X.device)
    bounds = [lay.K * s // p for s in range(p + 1)]
    for s in range(p):
        if bounds[s] < bounds[s + 1]:
            _moment_raw_into(X, m, b, out, key_range=(bounds[s], bounds[s + 1]))
    _divide(out, t)
    return BlockSymTensor(n, m, b, data=out)
