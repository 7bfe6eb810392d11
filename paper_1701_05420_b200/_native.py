"""ctypes binding of libbcgpu.so (include/bcgpu.h) -- the C-ABI boundary.

This is the only door to compute: there is no CPU fallback.  If the library
or a CUDA device is missing, the call raises NativeUnavailableError.
"""

from __future__ import annotations

import ctypes
import os
import threading
from functools import lru_cache

import numpy as np

from .errors import NativeUnavailableError, ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
# BCG_LIB=checks selects the bounds-checked debug build (_build.py --checks)
_LIB_ENV = os.environ.get("BCG_LIB", "")
LIB_PATH = (os.path.join(_HERE, "libbcgpu_checks.so") if _LIB_ENV == "checks"
            else _LIB_ENV if _LIB_ENV.endswith(".so") else os.path.join(_HERE, "libbcgpu.so"))

_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_dbl = ctypes.c_double
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t

# (name, restype, argtypes) -- every symbol include/bcgpu.h declares
SIGNATURES = [
    ("bcg_last_error", ctypes.c_char_p, []),
    ("bcg_version", ctypes.c_int, []),
    ("bcg_launch_count", _i64, []),
    ("bcg_moment_blocks", ctypes.c_int, [_vp, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _i64, _i64, _vp]),
    ("bcg_plan_create", ctypes.c_int, [_i64, _i32, _i32, ctypes.POINTER(_vp)]),
    ("bcg_plan_create_ex", ctypes.c_int, [_i64, _i32, _i32, _i32, ctypes.POINTER(_vp)]),
    ("bcg_plan_create_flags", ctypes.c_int, [_i64, _i32, _i32, _i32, ctypes.POINTER(_vp)]),
    ("bcg_plan_output", ctypes.c_int, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    ("bcg_plan_tiled", ctypes.c_int, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    ("bcg_plan_waste", ctypes.c_int, [_vp, ctypes.POINTER(_i64)]),
    ("bcg_plan_kernel", ctypes.c_int, [_vp, ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32),
                                       ctypes.POINTER(_i64)]),
    ("bcg_plan_gemm", ctypes.c_int, [_vp, _i32, ctypes.POINTER(_i32), ctypes.POINTER(_i32), _vp,
                                     ctypes.POINTER(_i64)]),
    ("bcg_plan_create_host", ctypes.c_int, [_i64, _i32, _i32, ctypes.POINTER(_vp)]),
    ("bcg_plan_destroy", ctypes.c_int, [_vp]),
    ("bcg_plan_selfcheck", ctypes.c_int, [_vp]),
    ("bcg_plan_sizes", ctypes.c_int, [_vp, _i32, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    ("bcg_plan_layout", ctypes.c_int, [_vp, _i32, _vp, _vp, _vp, _vp]),
    ("bcg_moment_ws_bytes", ctypes.c_int, [_vp, _i64, ctypes.POINTER(_sz)]),
    ("bcg_moment_t_ws_bytes", ctypes.c_int, [_vp, _i64, ctypes.POINTER(_sz)]),
    ("bcg_colstats", ctypes.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    ("bcg_colstats_ws_bytes", _sz, [_i64, _i64]),
    ("bcg_center", ctypes.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    ("bcg_moment_raw", ctypes.c_int, [_vp, _vp, _i64, _i64, _vp, _vp, _sz, _vp]),
    ("bcg_moment_raw_t", ctypes.c_int, [_vp, _vp, _i64, _i64, _vp, _vp, _sz, _vp]),
    ("bcg_padded_t", _i64, [_i64]),
    ("bcg_dense_subsets_ws_bytes", _sz, [_i64, _i32, _i64]),
    ("bcg_dense_subsets", ctypes.c_int, [_vp, _i64, _i64, _i64, _vp, _i32, _vp, _i64, _vp, _vp, _sz, _vp]),
    ("bcg_transpose_pad", ctypes.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp]),
    ("bcg_rowstats", ctypes.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    ("bcg_rowstats_ws_bytes", _sz, [_i64, _i64]),
    ("bcg_rowstats_ws", ctypes.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    ("bcg_moment_raw_range", ctypes.c_int, [_vp, _vp, _i64, _i64, _vp, _vp, _sz, _i64, _i64, _vp]),
    ("bcg_moment_raw_t_range", ctypes.c_int, [_vp, _vp, _i64, _i64, _vp, _vp, _sz, _i64, _i64, _vp]),
    ("bcg_cumulant_recursion", ctypes.c_int, [_vp, _vp, _vp, _vp]),
    ("bcg_cumulant_recursion_range", ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _vp]),
    ("bcg_cumulant_recursion_ex", ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, _vp]),
    ("bcg_cumulant_recursion_span", ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, _vp]),
    ("bcg_outer_prod_cum", ctypes.c_int, [_vp, _i32, _vp, _vp, _vp]),
    ("bcg_axpby", ctypes.c_int, [_i64, _dbl, _vp, _dbl, _vp, _vp, _vp]),
    ("bcg_div", ctypes.c_int, [_i64, _vp, _dbl, _vp, _vp]),
]

_lock = threading.Lock()


@lru_cache(maxsize=1)
def lib() -> ctypes.CDLL:
    """Load libbcgpu.so (building it in-tree first if nvcc is available)."""
    if not os.path.exists(LIB_PATH):
        try:
            from . import _build

            _build.build()
        except Exception as exc:  # pragma: no cover - depends on toolchain
            raise NativeUnavailableError(f"libbcgpu.so is not built ({exc})") from exc
    try:
        handle = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        raise NativeUnavailableError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, res, args in SIGNATURES:
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    return handle


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = lib().bcg_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == 1:
        raise ValidationError(msg)
    if rc == 3:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def torch_cuda():
    """torch with a usable CUDA device, or NativeUnavailableError."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailableError(
            "a CUDA device is required: this framework has no CPU fallback"
        )
    return torch


def stream_handle() -> int:
    torch = torch_cuda()
    return torch.cuda.current_stream().cuda_stream


def ptr(tensor) -> int:
    return tensor.data_ptr()


PLAN_FULL = 1  # BCG_PLAN_FULL: every stored element computed directly
PLAN_HOST = 2  # BCG_PLAN_HOST: tables only


class Plan:
    """Host-built index tables for one (n, m, b) (bcg_plan_create_flags).
    ``full``: the moment GEMM computes every stored element directly instead
    of the sorted ones within runs of equal block indices plus the fill."""

    def __init__(self, n: int, m: int, b: int, host_only: bool = False, variant: int = -1,
                 full: bool = False):
        self.n, self.m, self.b = int(n), int(m), int(b)
        self.host_only = host_only
        self.variant = int(variant)
        self.full = bool(full)
        if self.variant > 0:
            raise ValidationError(f"unknown moment kernel variant {self.variant}")
        h = _vp()
        flags = (PLAN_FULL if full else 0) | (PLAN_HOST if host_only else 0)
        check(lib().bcg_plan_create_flags(self.n, self.m, self.b, flags, ctypes.byref(h)), "plan")
        self._h = h
        self._lib = lib()

    @property
    def handle(self):
        return self._h

    def sizes(self, order: int):
        k, s = _i64(), _i64()
        check(self._lib.bcg_plan_sizes(self._h, order, ctypes.byref(k), ctypes.byref(s)))
        return k.value, s.value

    def layout(self, order: int):
        """(keys, col0, edges, offs) as int64 arrays (bc/_engines.py:46-54)."""
        K, _ = self.sizes(order)
        keys = np.empty((K, order), dtype=np.int64)
        col0 = np.empty((K, order), dtype=np.int64)
        edges = np.empty((K, order), dtype=np.int64)
        offs = np.empty(K + 1, dtype=np.int64)
        check(self._lib.bcg_plan_layout(self._h, order, keys.ctypes.data, col0.ctypes.data,
                                        edges.ctypes.data, offs.ctypes.data))
        return keys, col0, edges, offs

    def output(self):
        """(S_out, produced): output size of bcg_moment_raw and the number of
        elements the moment GEMMs compute (S_out for a full plan)."""
        S, prod = _i64(), _i64()
        check(self._lib.bcg_plan_output(self._h, ctypes.byref(S), ctypes.byref(prod)))
        return S.value, prod.value

    def kernel(self):
        """(variant, tm, tn, ntiles) of the moment GEMM this plan launches."""
        v, tm, tn, nt = _i32(), _i32(), _i32(), _i64()
        check(self._lib.bcg_plan_kernel(self._h, ctypes.byref(v), ctypes.byref(tm), ctypes.byref(tn),
                                        ctypes.byref(nt)))
        return v.value, tm.value, tn.value, nt.value

    def gemms(self):
        """(split_T, [(h, r, tm, tn, ntiles), ...]) of the plan's moment GEMMs."""
        ng, T = _i32(), _i32()
        check(self._lib.bcg_plan_gemm(self._h, -1, ctypes.byref(ng), ctypes.byref(T), None, None))
        out = []
        for i in range(ng.value):
            info, nt = (_i32 * 4)(), _i64()
            check(self._lib.bcg_plan_gemm(self._h, i, None, None, info, ctypes.byref(nt)))
            out.append((*info, nt.value))
        return T.value, out

    def ws_bytes(self, t: int) -> int:
        """Workspace of the row-major entries (transposed copy + split-K)."""
        out = _sz()
        check(self._lib.bcg_moment_ws_bytes(self._h, int(t), ctypes.byref(out)))
        return out.value

    def t_ws_bytes(self, t: int) -> int:
        """Workspace of the transposed-input entries (split-K partials only)."""
        out = _sz()
        check(self._lib.bcg_moment_t_ws_bytes(self._h, int(t), ctypes.byref(out)))
        return out.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.bcg_plan_destroy(h)
            except Exception:
                pass


_plans: dict = {}


def moment_variant() -> int:
    """Moment-kernel variant for new plans: $BCG_MOMENT_VARIANT or the
    library default (-1)."""
    v = os.environ.get("BCG_MOMENT_VARIANT", "")
    return int(v) if v.strip() else -1


def full_blocks() -> bool:
    """$BCG_MOMENT_FULL=1: plans compute every stored element directly (A/B knob)."""
    return os.environ.get("BCG_MOMENT_FULL", "0") not in ("", "0")


def plan(n: int, m: int, b: int, full: bool | None = None) -> Plan:
    """Cached device plan for (n, m, b) and the current kernel knobs."""
    torch = torch_cuda()
    full = full_blocks() if full is None else bool(full)
    # plans hold device tables: one per (device, n, m, b, kernel knobs)
    key = (torch.cuda.current_device(), int(n), int(m), int(b), moment_variant(), full,
           os.environ.get("BCG_TILE", ""), os.environ.get("BCG_NO_HYBRID", ""))
    with _lock:
        p = _plans.get(key)
        if p is None:
            p = _plans[key] = Plan(key[1], key[2], key[3], variant=key[4], full=full)
        return p


def launch_count() -> int:
    return int(lib().bcg_launch_count())
