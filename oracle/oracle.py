"""TEST INFRASTRUCTURE ONLY: ctypes binding of oracle/liblitho_oracle.so, the
plain-C fp64 restatement of the reference hot path (oracle/litho_oracle.c).

Parity pinned against the reference itself (oracle/_ref) and the golden
vectors in tests/golden/ by tests/test_oracle.py. Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline may import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblitho_oracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"oracle not built: {LIB_PATH} (make -C oracle)")
        _lib = C.CDLL(LIB_PATH)
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _check(rc, what):
    if rc != 0:
        raise ValueError(f"oracle {what}: invalid argument")


def set_threads(n: int) -> None:
    lib().orc_set_threads(C.c_int(n))


def _poly_arrays(polys):
    if polys:
        xy = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int64).reshape(-1, 2) for p in polys]))
    else:
        xy = np.zeros((0, 2), np.int64)
    starts = np.zeros(len(polys) + 1, np.int64)
    starts[1:] = np.cumsum([len(p) for p in polys])
    return xy, starts


def rasterize(polys, nx, ny, pitch=1.0, ox=0.0, oy=0.0, dbu_per_nm=1.0):
    """Healed polygons -> fp64 coverage (raster.cpp:53-95 without heal)."""
    xy, starts = _poly_arrays(polys)
    out = np.zeros(nx * ny)
    _check(lib().orc_rasterize(_p(xy, C.c_int64), _p(starts, C.c_int64), C.c_int(len(polys)), C.c_int(nx),
                               C.c_int(ny), C.c_double(pitch), C.c_double(ox), C.c_double(oy),
                               C.c_double(dbu_per_nm), _p(out, C.c_double)), "rasterize")
    return out.reshape(ny, nx)


def _kargs(weights, support, values):
    w = np.ascontiguousarray(weights, np.float64)
    s = np.ascontiguousarray(support, np.int32)
    v = np.ascontiguousarray(np.stack([np.real(values), np.imag(values)], -1), np.float64)
    return w, s, v


def image_socs(mask, weights, support, values, dose=1.0):
    ny, nx = mask.shape
    m = np.ascontiguousarray(mask, np.float64)
    w, s, v = _kargs(weights, support, values)
    out = np.zeros(nx * ny)
    lib().orc_image_socs(C.c_int(nx), C.c_int(ny), _p(m, C.c_double), C.c_int(len(w)), _p(w, C.c_double),
                         C.c_int(len(s)), _p(s, C.c_int32), _p(v, C.c_double), C.c_double(dose),
                         _p(out, C.c_double))
    return out.reshape(ny, nx)


def gaussian_blur(img, sigma_nm, pitch=1.0):
    ny, nx = img.shape
    m = np.ascontiguousarray(img, np.float64)
    out = np.zeros(nx * ny)
    _check(lib().orc_gaussian_blur(C.c_int(nx), C.c_int(ny), C.c_double(pitch), _p(m, C.c_double),
                                   C.c_double(sigma_nm), _p(out, C.c_double)), "gaussian_blur")
    return out.reshape(ny, nx)


def weighted_gradient(mask, weights, support, values, W=None, dose=1.0):
    ny, nx = mask.shape
    m = np.ascontiguousarray(mask, np.float64)
    w, s, v = _kargs(weights, support, values)
    out = np.zeros(nx * ny)
    if W is None:
        wp = None
    else:
        ww = np.ascontiguousarray(W, np.float64)
        wp = _p(ww, C.c_double)
    lib().orc_weighted_gradient(C.c_int(nx), C.c_int(ny), _p(m, C.c_double), C.c_int(len(w)),
                                _p(w, C.c_double), C.c_int(len(s)), _p(s, C.c_int32), _p(v, C.c_double),
                                C.c_double(dose), wp, _p(out, C.c_double))
    return out.reshape(ny, nx)


def ilt_iteration(theta, target, weights, support, values, focus_weight, params, pitch=1.0):
    """One ILT step (see litho_oracle.c); theta (float64, C-contig) updated in place."""
    ny, nx = theta.shape
    assert theta.dtype == np.float64 and theta.flags.c_contiguous
    t = np.ascontiguousarray(target, np.float64)
    w = np.ascontiguousarray(weights, np.float64)
    F, K = w.shape
    s = np.ascontiguousarray(support, np.int32)
    v = np.ascontiguousarray(np.stack([np.real(values), np.imag(values)], -1), np.float64)
    fw = np.ascontiguousarray(focus_weight, np.float64)
    pr = np.ascontiguousarray(params, np.float64)
    cost = C.c_double()
    grad = np.zeros(nx * ny)
    lib().orc_ilt_iteration(C.c_int(nx), C.c_int(ny), C.c_double(pitch), C.c_int(F), C.c_int(K),
                            _p(w, C.c_double), C.c_int(len(s)), _p(s, C.c_int32), _p(v, C.c_double),
                            _p(fw, C.c_double), _p(pr, C.c_double), _p(t, C.c_double), _p(theta, C.c_double),
                            C.byref(cost), _p(grad, C.c_double))
    return cost.value, grad.reshape(ny, nx)


def threshold(img, tau):
    """z_print / ResistImage threshold semantics (ai.cpp:90-92): v >= tau -> 1."""
    return (np.asarray(img) >= tau).astype(np.float64)
