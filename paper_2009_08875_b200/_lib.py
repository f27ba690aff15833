"""ctypes binding of libhwgpu.so (include/heatwave_b200.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing, every entry point raises instead of computing something else.
Return codes map onto the reference's exceptions:
HWG_EINVAL -> ValueError, HWG_ENOTSPD -> RuntimeError,
HWG_EMAXIT -> IterationLimitError, HWG_EKEY -> KeyError,
HWG_ENOMEM -> MemoryError, HWG_ECUDA -> RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhwgpu.so")

HWG_OK, HWG_EINVAL, HWG_ENOTSPD, HWG_EMAXIT, HWG_ECUDA, HWG_ENOMEM, HWG_EKEY = range(7)
COEF_STRIDE = 8

# every symbol include/heatwave_b200.h declares
EXPORTS = ("hwg_last_error", "hwg_version", "hwg_create", "hwg_destroy",
           "hwg_workspace_bytes", "hwg_wavelet", "hwg_spatial", "hwg_schur_apply",
           "hwg_kx_apply", "hwg_mg_rows", "hwg_rhs", "hwg_dot", "hwg_pcg",
           "hwg_solve_host", "hwg_launch_count", "hwg_profile_enable", "hwg_profile_read",
           "hwg_syn_stage", "hwg_ana_stage", "hwg_bside_rows", "hwg_bt_rows", "hwg_mg_rows_dev",
           "hwg_mg_rows_dev_dot", "hwg_grid_scatter", "hwg_grid_gather", "hwg_set_schur_form",
           "hwg_row_partials", "hwg_tree_sum", "hwg_axpy", "hwg_xpay", "hwg_temporal_rows",
           "hwg_pcg_scalar", "hwg_pcg_update_wr", "hwg_pcg_update_wp", "hwg_sub",
           "hwg_any_nonzero")

_P = C.c_void_p
_D = C.c_double
_I32 = C.c_int32
_I64 = C.c_int64


class HwgDesc(C.Structure):
    _fields_ = [("dim", _I32), ("J", _I32), ("K", _I32), ("vcycles", _I32),
                ("smooth", _I32), ("device", _I32), ("alpha", _D),
                ("coef", _P), ("stencil_M", _P), ("stencil_A", _P),
                ("temporal", _P), ("wavelet_scale", _P), ("rows_max", _I64),
                ("domain", _I32), ("reserved", _I32), ("coarse_inv", _P)]


class HwgPcgStats(C.Structure):
    _fields_ = [("iterations", _I32), ("capacity", _I32),
                ("residual_norms", _P), ("alphas", _P), ("betas", _P),
                ("ms_schur", _D), ("ms_precond", _D), ("ms_vector", _D),
                ("ms_total", _D), ("epsilon_used", _D)]


class IterationLimitError(RuntimeError):
    """PCG hit the iteration cap; carries the residual-norm history
    (solver.py:132-137)."""

    def __init__(self, message, residual_norms):
        super().__init__(message)
        self.residual_norms = residual_norms


_lib = None


def load(build_if_missing=True):
    """Load libhwgpu.so (building it first if it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    alt = os.environ.get("HWG_LIB_PATH")      # A/B measurements of two builds
    if alt:
        _lib = _bind(C.CDLL(alt))
        return _lib
    if not os.path.exists(LIB_PATH):
        if not build_if_missing:
            raise OSError(f"{LIB_PATH} is missing; run python -m paper_2009_08875_b200.build")
        from . import build
        build.build()
    _lib = _bind(C.CDLL(LIB_PATH))
    return _lib


def _bind(L):
    """Declare the ctypes signatures of every exported entry point."""
    L.hwg_last_error.restype = C.c_char_p
    L.hwg_version.restype = C.c_int
    L.hwg_create.argtypes = [C.POINTER(HwgDesc), C.POINTER(_P)]
    L.hwg_destroy.argtypes = [_P]
    L.hwg_workspace_bytes.argtypes = [_P]
    L.hwg_workspace_bytes.restype = _I64
    L.hwg_launch_count.argtypes = [_P]
    L.hwg_launch_count.restype = _I64
    L.hwg_wavelet.argtypes = [_P, _P, _P, C.c_int, _P]
    L.hwg_spatial.argtypes = [_P, C.c_int, _P, _P, _I64, _P]
    L.hwg_schur_apply.argtypes = [_P, _P, _P, _P]
    L.hwg_kx_apply.argtypes = [_P, _P, _P, _P]
    L.hwg_mg_rows.argtypes = [_P, _I32, _P, _P, _P, _I64, _P]
    L.hwg_rhs.argtypes = [_P, _P, _P, _P, _P, _P]
    L.hwg_dot.argtypes = [_P, _P, _P, _I64, C.POINTER(_D), _P]
    L.hwg_pcg.argtypes = [_P, _P, _P, _D, _D, _I32, _I32, C.POINTER(HwgPcgStats), _P]
    L.hwg_profile_enable.argtypes = [_P, C.c_int]
    L.hwg_profile_read.argtypes = [_P, C.c_int, C.POINTER(_D), C.POINTER(_D), C.POINTER(_I64)]
    L.hwg_syn_stage.argtypes = [_P, C.c_int, _P, _I64, _P, _I64, _P, _P, _I64, _I64, _P]
    L.hwg_ana_stage.argtypes = [_P, C.c_int, _P, _I64, _P, _I64, _I64, _P, _I64, _I64, _P]
    L.hwg_bside_rows.argtypes = [_P, _P, _I64, _I64, _P, _P, _I64, _I64, _P, _P]
    L.hwg_bt_rows.argtypes = [_P, _P, _P, _P, _P, _I64, _P]
    L.hwg_mg_rows_dev.argtypes = [_P, _P, _P, _P, _I64, _P]
    L.hwg_mg_rows_dev_dot.argtypes = [_P, _P, _P, _P, _I64, _P, _P, _P]
    L.hwg_grid_scatter.argtypes = [_P, _P, _P, _I64, _P]
    L.hwg_set_schur_form.argtypes = [_P, C.c_int]
    L.hwg_grid_gather.argtypes = [_P, _P, _P, _I64, _P]
    L.hwg_row_partials.argtypes = [_P, _P, _P, _I64, _P, _P]
    L.hwg_tree_sum.argtypes = [_P, _P, _I64, _P, _P]
    L.hwg_axpy.argtypes = [_P, _D, _P, _P, _I64, _P]
    L.hwg_xpay.argtypes = [_P, _D, _P, _P, _I64, _P]
    L.hwg_temporal_rows.argtypes = [_P, C.c_int, _P, _I64, _P, _I64, _I64, _P]
    L.hwg_pcg_scalar.argtypes = [_P, C.c_int, _P, _P]
    L.hwg_pcg_update_wr.argtypes = [_P, _P, _P, _P, _P, _P, _I64, C.c_int, C.c_int, _P]
    L.hwg_pcg_update_wp.argtypes = [_P, _P, _P, _P, _P, _I64, C.c_int, _P]
    L.hwg_sub.argtypes = [_P, _P, _P, _P, _I64, _P]
    L.hwg_any_nonzero.argtypes = [_P, _P, _I64, _P, _P]
    L.hwg_solve_host.argtypes = [_P, _P, _P, _D, _D, _I32, _I32, C.POINTER(HwgPcgStats), _P]
    for name in EXPORTS:
        if name not in ("hwg_last_error", "hwg_version", "hwg_workspace_bytes",
                        "hwg_launch_count"):
            getattr(L, name).restype = C.c_int
    return L


def check(rc, history=None):
    """Raise the reference's exception for a non-zero return code."""
    if rc == HWG_OK:
        return
    msg = load().hwg_last_error().decode(errors="replace")
    if rc == HWG_EINVAL:
        raise ValueError(msg)
    if rc == HWG_ENOTSPD:
        raise RuntimeError(msg)
    if rc == HWG_EMAXIT:
        raise IterationLimitError(msg, history or [])
    if rc == HWG_EKEY:
        raise KeyError(msg)
    if rc == HWG_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"CUDA failure: {msg}")
