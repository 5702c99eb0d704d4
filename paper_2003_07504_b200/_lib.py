"""ctypes binding of the C ABI in include/ils_b200.h (libils_b200.so).

This is the reference-facing boundary: every product call goes through
these foreign functions.  There is no CPU fallback -- if the library or a
CUDA device is missing, the calls raise.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import NumericalError

HERE = os.path.dirname(os.path.abspath(__file__))
# ILS_LIB: an alternative build of the same library (tuning variants, tools/build_variant.py)
LIB_PATH = os.environ.get("ILS_LIB") or os.path.join(HERE, "libils_b200.so")

ILS_OK, ILS_EINVAL, ILS_ENONFINITE_INPUT, ILS_ENONFINITE, ILS_ECUDA, ILS_EUNSUPPORTED = range(6)
ILS_CHARBONNIER, ILS_WELSCH, ILS_SOFT = 0, 1, 2
ILS_F32, ILS_F64 = 0, 1
STATUS_CLEAN = 0x7F7F7F7F

EXPORTS = (
    "ils_plan_create", "ils_hqs_plan_create", "ils_plan_destroy", "ils_workspace_size", "ils_smooth", "ils_smooth_host", "ils_smooth_u8",
    "ils_smooth_host_u8", "ils_smooth_epilogue", "ils_gaussian_blur",
    "ils_host_io_size", "ils_launch_pass", "ils_slab_plan_create", "ils_slab_get_layout", "ils_slab_row_pass",
    "ils_slab_col_pass",
    "ils_solve_ls", "ils_rfft2", "ils_irfft2", "ils_rgb_yuv", "ils_plan_get_info", "ils_last_error",
    "ils_abi_version", "ils_grad", "ils_adjoint_accumulate", "ils_aux_update", "ils_energy",
    "ils_convert", "ils_denominator", "ils_hermitian_full", "ils_tonemap_workspace_size", "ils_tonemap",
    "ils_detail_boost", "ils_nccl_get_unique_id", "ils_nccl_comm_create", "ils_nccl_comm_destroy",
    "ils_dist_workspace_size", "ils_smooth_dist",
)


class Params(C.Structure):
    _fields_ = [("kind", C.c_int32), ("p", C.c_double), ("eps", C.c_double), ("gamma", C.c_double),
                ("lam", C.c_double), ("c", C.c_double), ("iters", C.c_int32)]


class HqsParams(C.Structure):
    _fields_ = [("lam", C.c_double), ("beta0", C.c_double), ("kappa", C.c_double), ("iters", C.c_int32)]


class TonemapParamsC(C.Structure):
    _fields_ = [("nscales", C.c_int32), ("lam", C.c_double * 3), ("weights", C.c_double * 3),
                ("target_range", C.c_double), ("saturation", C.c_double), ("log_offset", C.c_double)]


class NcclId(C.Structure):
    _fields_ = [("internal", C.c_char * 128)]


class Epilogue(C.Structure):
    _fields_ = [("kind", C.c_int32), ("k", C.c_double)]


ILS_EPI_NONE, ILS_EPI_DETAIL = 0, 1


class PlanInfo(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "batch", "height", "width", "dtype", "packed",
        "row_band", "row_threads", "row_grid", "row_smem",
        "col_cols", "col_threads", "col_grid", "col_smem",
        "row_passes", "col_passes", "row_group", "col_group", "row_spec", "col_spec", "row_swz", "col_swz")] + [
        ("row_radix", C.c_int32 * 16), ("col_radix", C.c_int32 * 16),
        ("spec_pitch", C.c_int64), ("launches_per_call", C.c_int32),
        ("col2_spec", C.c_int32), ("col2_n1", C.c_int32), ("col2_n2", C.c_int32), ("col2_cols", C.c_int32),
        ("col3_spec", C.c_int32), ("col3_n1", C.c_int32), ("col3_n2", C.c_int32), ("col3_n3", C.c_int32),
        ("col3_cols", C.c_int32), ("row_roll_rows", C.c_int32)]

    def as_dict(self):
        d = {n: getattr(self, n) for n, _ in self._fields_ if n not in ("row_radix", "col_radix")}
        d["row_radix"] = [r for r in self.row_radix[: self.row_passes]]
        d["col_radix"] = [r for r in self.col_radix[: self.col_passes]]
        return d


_lib = None
_lock = threading.Lock()

_P = C.c_void_p
_SIGS = {
    "ils_plan_create": (C.c_int, [C.POINTER(_P), C.c_int32, C.c_int32, C.c_int32, C.POINTER(Params), C.c_int32,
                                  C.c_int32]),
    "ils_hqs_plan_create": (C.c_int, [C.POINTER(_P), C.c_int32, C.c_int32, C.c_int32, C.POINTER(HqsParams),
                                      C.c_int32, C.c_int32]),
    "ils_plan_destroy": (None, [_P]),
    "ils_workspace_size": (C.c_int, [_P, C.POINTER(C.c_size_t)]),
    "ils_smooth": (C.c_int, [_P, _P, _P, C.c_int64, _P, _P, _P, _P]),
    "ils_smooth_host": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int32, _P, _P, _P, C.POINTER(C.c_int32)]),
    "ils_smooth_u8": (C.c_int, [_P, _P, _P, C.c_int32, _P, _P, _P]),
    "ils_smooth_host_u8": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, _P, _P, _P, C.POINTER(C.c_int32)]),
    "ils_smooth_epilogue": (C.c_int, [_P, _P, _P, C.c_int64, _P, _P, _P, C.POINTER(Epilogue)]),
    "ils_gaussian_blur": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_double, C.c_int32,
                                    _P]),
    "ils_host_io_size": (C.c_int, [_P, C.POINTER(C.c_size_t)]),
    "ils_launch_pass": (C.c_int, [_P, C.c_int32, _P, _P, C.c_int64, _P, _P, _P]),
    "ils_solve_ls": (C.c_int, [_P, _P, _P, _P, _P, C.c_int64, _P, _P, _P]),
    "ils_rfft2": (C.c_int, [_P, _P, C.c_int64, _P, C.c_int64, _P]),
    "ils_irfft2": (C.c_int, [_P, _P, C.c_int64, _P, C.c_int64, _P]),
    "ils_rgb_yuv": (C.c_int, [_P, C.c_int32, C.c_int64, C.c_int64, C.c_int32, C.c_int32, _P]),
    "ils_plan_get_info": (C.c_int, [_P, C.POINTER(PlanInfo)]),
    "ils_slab_plan_create": (C.c_int, [C.POINTER(_P), C.c_int32, C.c_int32, C.POINTER(Params), C.c_int32, C.c_int32,
                                       C.c_int32, C.c_int32]),
    "ils_slab_get_layout": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int64)]),
    "ils_slab_row_pass": (C.c_int, [_P, C.c_int32, _P, _P, _P, _P, C.c_int32, _P, _P]),
    "ils_slab_col_pass": (C.c_int, [_P, _P, _P, _P]),
    "ils_grad": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32, _P]),
    "ils_adjoint_accumulate": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32, _P]),
    "ils_aux_update": (C.c_int, [C.POINTER(Params), _P, _P, C.c_int64, C.c_int32, _P]),
    "ils_energy": (C.c_int, [C.POINTER(Params), _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32, _P,
                             _P, _P]),
    "ils_convert": (C.c_int, [_P, C.c_int32, _P, C.c_int32, C.c_int64, _P]),
    "ils_denominator": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_double, C.c_double, _P]),
    "ils_hermitian_full": (C.c_int, [_P, C.c_int64, _P, C.c_int32, C.c_int32, _P]),
    "ils_tonemap_workspace_size": (C.c_int, [_P, C.POINTER(C.c_size_t)]),
    "ils_tonemap": (C.c_int, [_P, _P, _P, _P, C.POINTER(TonemapParamsC), _P, _P, _P, _P]),
    "ils_detail_boost": (C.c_int, [_P, _P, _P, C.c_int64, C.c_double, C.c_int32, _P]),
    "ils_nccl_get_unique_id": (C.c_int, [C.POINTER(NcclId)]),
    "ils_nccl_comm_create": (C.c_int, [C.POINTER(_P), C.c_int32, C.POINTER(NcclId), C.c_int32, C.c_int32]),
    "ils_nccl_comm_destroy": (C.c_int, [_P]),
    "ils_dist_workspace_size": (C.c_int, [_P, C.POINTER(C.c_size_t)]),
    "ils_smooth_dist": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int64, C.c_int64, _P, _P, _P, _P]),
    "ils_last_error": (C.c_char_p, []),
    "ils_abi_version": (C.c_int32, []),
}


def lib():
    """Load (building first if this checkout has no .so yet) the C library."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    from .build import build

                    build()
                handle = C.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


def last_error() -> str:
    return lib().ils_last_error().decode("utf-8", "replace")


def check(status: int, what: str = "") -> None:
    """Map an ils_status to the reference's exception types (errors.py:10-15)."""
    if status == ILS_OK:
        return
    msg = last_error() or what
    if status in (ILS_EINVAL, ILS_ENONFINITE_INPUT, ILS_EUNSUPPORTED):
        raise ValueError(msg)
    if status == ILS_ENONFINITE:
        raise NumericalError(msg)
    raise RuntimeError(f"CUDA failure in {what}: {msg}")
