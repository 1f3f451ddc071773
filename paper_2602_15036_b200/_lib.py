"""ctypes binding of the in-tree native library (include/lithogpu.h).

This is the reference-side binding a maintainer would add (the ctypes stub of
INTEGRATION.md).  It fails loudly when liblithogpu.so is missing: there is no
CPU fallback of the hot path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# LITHOGPU_LIB: alternative build of the same library (A/B timing variants, tools/)
LIB_PATH = os.environ.get("LITHOGPU_LIB") or os.path.join(_HERE, "liblithogpu.so")

OK, ERR_DOMAIN, ERR_USAGE = 0, 1, 2
F32, F64, U8 = 0, 1, 2


class LithoError(RuntimeError):
    """Raised for LITHOGPU_ERR_DOMAIN (reference: std::runtime_error / invalid_argument)."""


class LithoUsageError(ValueError):
    """Raised for LITHOGPU_ERR_USAGE (null pointers, bad enums, out-of-range indices)."""


class Grid(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("pitch_nm", C.c_double),
                ("origin_x_nm", C.c_double), ("origin_y_nm", C.c_double)]


class IltParams(C.Structure):
    _fields_ = [("mask_steepness", C.c_double), ("resist_beta", C.c_double),
                ("threshold", C.c_double), ("resist_sigma_nm", C.c_double),
                ("dose", C.c_double), ("step", C.c_double),
                ("focus_weights", C.POINTER(C.c_double))]


_lib = None

_vp = C.c_void_p
_SIGS = {
    "lithogpu_last_error": (C.c_char_p, []),
    "lithogpu_host_last_error": (C.c_char_p, []),
    "lithogpu_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "lithogpu_ctx_destroy": (None, [_vp]),
    "lithogpu_ctx_set_stream": (C.c_int, [_vp, _vp]),
    "lithogpu_ctx_synchronize": (C.c_int, [_vp]),
    "lithogpu_ctx_launch_count": (C.c_longlong, [_vp]),
    "lithogpu_ctx_set_profiling": (C.c_int, [_vp, C.c_int]),
    "lithogpu_ctx_profile_report": (C.c_int, [_vp, C.c_char_p, C.c_size_t, C.c_int]),
    "lithogpu_fp32_peak": (C.c_int, [_vp, C.POINTER(C.c_double)]),
    "lithogpu_rasterize": (C.c_int, [_vp, C.POINTER(Grid), _vp, _vp, C.c_int, C.c_double, _vp]),
    "lithogpu_kernels_create": (C.c_int, [_vp, C.POINTER(Grid), C.c_int, C.c_int, C.c_int, _vp,
                                          C.c_int, _vp, _vp, C.POINTER(_vp)]),
    "lithogpu_kernels_destroy": (None, [_vp]),
    "lithogpu_kernels_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                        C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "lithogpu_kernels_fast_order": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "lithogpu_kernels_fast_stacks": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "lithogpu_image_socs": (C.c_int, [_vp, C.c_int, _vp, C.c_int, C.c_double, _vp, C.c_int]),
    "lithogpu_image_resist": (C.c_int, [_vp, C.c_int, _vp, C.c_int, C.c_double, C.c_double,
                                        C.c_double, _vp, _vp, C.c_int, _vp]),
    "lithogpu_gaussian_blur": (C.c_int, [_vp, C.POINTER(Grid), _vp, C.c_int, C.c_double, _vp]),
    "lithogpu_threshold": (C.c_int, [_vp, C.c_size_t, _vp, C.c_int, C.c_double, _vp, C.c_int]),
    "lithogpu_fft2": (C.c_int, [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int]),
    "lithogpu_intensity_gradient": (C.c_int, [_vp, C.c_int, _vp, C.c_int, _vp, C.c_int,
                                              C.c_double, _vp, C.c_int]),
    "lithogpu_ilt_create": (C.c_int, [_vp, C.POINTER(IltParams), C.c_int, C.POINTER(_vp)]),
    "lithogpu_ilt_destroy": (None, [_vp]),
    "lithogpu_ilt_set_tile": (C.c_int, [_vp, C.c_int, _vp, _vp, C.c_int]),
    "lithogpu_ilt_set_tiles": (C.c_int, [_vp, _vp, _vp, C.c_int]),
    "lithogpu_ilt_run": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "lithogpu_ilt_gradient": (C.c_int, [_vp, _vp, _vp, C.c_int]),
    "lithogpu_ilt_get_window": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _vp, C.c_int64,
                                          C.c_int]),
    "lithogpu_ilt_get_window_async": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _vp, C.c_int64,
                                                C.c_int]),
    "lithogpu_ilt_get_tile": (C.c_int, [_vp, C.c_int, _vp, _vp, C.c_int]),
    "lithogpu_ilt_get_tiles": (C.c_int, [_vp, _vp, _vp, C.c_int]),
    "lithogpu_marching_squares": (C.c_int, [_vp, C.POINTER(Grid), _vp, C.c_double, C.POINTER(_vp)]),
    "lithogpu_contours_size": (C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "lithogpu_contours_get": (C.c_int, [_vp, _vp, _vp, _vp]),
    "lithogpu_contours_destroy": (None, [_vp]),
    "lithogpu_measure_epe": (C.c_int, [_vp, _vp, C.c_int64, C.c_double, _vp, _vp]),
    "lithogpu_measure_epe_loops": (C.c_int, [_vp, _vp, C.c_int64, _vp, _vp, _vp, C.c_int64, C.c_double, _vp,
                                             _vp]),
    "lithogpu_evaluate_epe": (C.c_int, [_vp, C.c_int, C.c_int, _vp, C.c_int, C.c_double, C.c_double, C.c_double,
                                        _vp, C.c_int64, C.c_double, _vp, _vp, _vp]),
    "lithogpu_socs_kernels_gpu": (C.c_int, [_vp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                            _vp, C.c_int, C.c_int, _vp, C.c_int, _vp, C.c_int, C.c_double, C.c_int,
                                            _vp, _vp, _vp, _vp]),
    "lithogpu_layout_load": (C.c_int, [C.c_char_p, C.POINTER(_vp)]),
    "lithogpu_layout_destroy": (None, [_vp]),
    "lithogpu_layout_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "lithogpu_layout_layer": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int64)]),
    "lithogpu_layout_get": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "lithogpu_write_aimg": (C.c_int, [_vp, C.POINTER(Grid), C.c_int, _vp, _vp, C.c_int]),
    "lithogpu_read_aimg": (C.c_int, [_vp, C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double),
                                     _vp]),
    "lithogpu_source_annular": (C.c_int, [C.c_double, C.c_double, C.c_int, C.POINTER(C.c_int), _vp]),
    "lithogpu_tcc_support": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                       C.c_double, C.POINTER(C.c_int), _vp]),
    "lithogpu_socs_kernels": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                        C.c_int, _vp, C.c_int, C.c_double, C.c_int, _vp, C.c_int,
                                        C.c_double, C.c_int, C.POINTER(C.c_int),
                                        C.POINTER(C.c_double), _vp, _vp]),
}

EXPORTED = tuple(_SIGS)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"native library missing: {LIB_PATH} — build it with "
                "`python -m paper_2602_15036_b200.build` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, host: bool = False) -> None:
    if rc == OK:
        return
    msg = (lib().lithogpu_host_last_error() if host else lib().lithogpu_last_error()) or b""
    msg = msg.decode()
    if rc == ERR_USAGE:
        raise LithoUsageError(msg)
    raise LithoError(msg)
