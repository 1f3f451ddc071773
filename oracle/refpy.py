"""TEST INFRASTRUCTURE ONLY: ctypes binding of oracle/_ref/libref_litho.so, the
reference's UNMODIFIED sources compiled by oracle/build_ref.sh (see
oracle/ref_capi.cpp for the symbol list and reference file:line anchors).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
reference) may import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libref_litho.so")
_lib = None
# the same reference sources with FFTW resolved by NVIDIA cuFFTW (GPU FFTs,
# host memory): oracle/build_ref_cufftw.sh; select with use_variant("cufftw")
VARIANTS = {"cpu": LIB_PATH, "cufftw": os.path.join(_HERE, "_ref", "libref_litho_cufftw.so")}


def use_variant(name: str) -> None:
    """switch the reference build ("cpu": FFT stand-in on host cores,
    "cufftw": cuFFT through its FFTW interface)."""
    global LIB_PATH, _lib
    LIB_PATH = VARIANTS[name]
    _lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run oracle/build_ref.sh)")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _check(rc):
    if rc != 0:
        raise RuntimeError("reference: " + lib().ref_last_error().decode())


def set_threads(n: int) -> None:
    lib().ref_set_threads(C.c_int(n))


def _poly_arrays(polys):
    xy = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int64).reshape(-1, 2) for p in polys]) if polys else np.zeros((0, 2), np.int64))
    starts = np.zeros(len(polys) + 1, np.int64)
    starts[1:] = np.cumsum([len(p) for p in polys])
    return xy, starts


def rasterize(polys, nx, ny, pitch=1.0, ox=0.0, oy=0.0, dbu_per_nm=1.0):
    xy, starts = _poly_arrays(polys)
    out = np.zeros(nx * ny, np.float64)
    _check(lib().ref_rasterize(_p(xy, C.c_int64), _p(starts, C.c_int64), C.c_int(len(polys)),
                               C.c_int(nx), C.c_int(ny), C.c_double(pitch), C.c_double(ox),
                               C.c_double(oy), C.c_double(dbu_per_nm), _p(out, C.c_double)))
    return out.reshape(ny, nx)


def heal(polys):
    xy, starts = _poly_arrays(polys)
    npoly = C.c_int64()
    nvert = C.c_int64()
    _check(lib().ref_heal(_p(xy, C.c_int64), _p(starts, C.c_int64), C.c_int(len(polys)),
                          C.byref(npoly), C.byref(nvert), None, None))
    oxy = np.zeros((max(nvert.value, 1), 2), np.int64)
    ost = np.zeros(npoly.value + 1, np.int64)
    _check(lib().ref_heal(_p(xy, C.c_int64), _p(starts, C.c_int64), C.c_int(len(polys)),
                          C.byref(npoly), C.byref(nvert), _p(oxy, C.c_int64), _p(ost, C.c_int64)))
    return [oxy[ost[i]:ost[i + 1]].copy() for i in range(npoly.value)]


def pupil(fx, fy, focus, lam=13.5, na=0.33, high_na=False):
    out = np.zeros(2)
    _check(lib().ref_pupil(C.c_double(lam), C.c_double(na), C.c_int(int(high_na)), C.c_double(fx),
                           C.c_double(fy), C.c_double(focus), _p(out, C.c_double)))
    return complex(out[0], out[1])


def source(sigma_in, sigma_out, grid_n):
    n = C.c_int()
    _check(lib().ref_source(C.c_double(sigma_in), C.c_double(sigma_out), C.c_int(grid_n), C.byref(n), None))
    out = np.zeros((n.value, 3))
    _check(lib().ref_source(C.c_double(sigma_in), C.c_double(sigma_out), C.c_int(grid_n), C.byref(n),
                            _p(out, C.c_double)))
    return out


class RefKernels:
    """build_tcc + decompose_tcc (reference imaging.cpp:113-216)."""

    def __init__(self, nx, ny, pitch, focus=0.0, lam=13.5, na=0.33, sigma_in=0.4, sigma_out=0.8,
                 grid_n=7, high_na=False, energy_floor=0.995, k_fixed=0, full_rank=False):
        h = C.c_void_p()
        _check(lib().ref_kernels_build(C.c_int(nx), C.c_int(ny), C.c_double(pitch), C.c_double(lam),
                                       C.c_double(na), C.c_double(sigma_in), C.c_double(sigma_out),
                                       C.c_int(grid_n), C.c_int(int(high_na)), C.c_double(focus),
                                       C.c_double(energy_floor), C.c_int(k_fixed),
                                       C.c_int(int(full_rank)), C.byref(h)))
        self._h = h
        self.nx, self.ny, self.pitch = nx, ny, pitch
        K, S, cap = C.c_int(), C.c_int(), C.c_double()
        lib().ref_kernels_info(h, C.byref(K), C.byref(S), C.byref(cap))
        self.K, self.S, self.captured = K.value, S.value, cap.value
        self.weights = np.zeros(self.K)
        self.support = np.zeros((self.S, 2), np.int32)
        vals = np.zeros((self.K, self.S, 2))
        self.tcc = np.zeros((self.S, self.S, 2))
        lib().ref_kernels_get(h, _p(self.weights, C.c_double), _p(self.support, C.c_int32),
                              _p(vals, C.c_double), _p(self.tcc, C.c_double))
        self.values = vals[..., 0] + 1j * vals[..., 1]
        self.tcc = self.tcc[..., 0] + 1j * self.tcc[..., 1]

    def hopkins(self, mask, dose=1.0):
        m = np.ascontiguousarray(mask, np.float64)
        out = np.zeros(self.nx * self.ny)
        _check(lib().ref_image_hopkins(self._h, _p(m, C.c_double), C.c_double(dose), _p(out, C.c_double)))
        return out.reshape(self.ny, self.nx)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ref_kernels_free(self._h)
            self._h = None


def _kargs(weights, support, values):
    w = np.ascontiguousarray(weights, np.float64)
    s = np.ascontiguousarray(support, np.int32)
    v = np.ascontiguousarray(np.stack([np.real(values), np.imag(values)], -1), np.float64)
    return w, s, v


def image_socs(mask, weights, support, values, pitch=1.0, dose=1.0):
    ny, nx = mask.shape
    m = np.ascontiguousarray(mask, np.float64)
    w, s, v = _kargs(weights, support, values)
    out = np.zeros(nx * ny)
    _check(lib().ref_image_socs(C.c_int(nx), C.c_int(ny), C.c_double(pitch), _p(m, C.c_double),
                                C.c_int(len(w)), _p(w, C.c_double), C.c_int(len(s)), _p(s, C.c_int32),
                                _p(v, C.c_double), C.c_double(dose), _p(out, C.c_double)))
    return out.reshape(ny, nx)


def gaussian_blur(img, sigma_nm, pitch=1.0):
    ny, nx = img.shape
    m = np.ascontiguousarray(img, np.float64)
    out = np.zeros(nx * ny)
    _check(lib().ref_gaussian_blur(C.c_int(nx), C.c_int(ny), C.c_double(pitch), _p(m, C.c_double),
                                   C.c_double(sigma_nm), _p(out, C.c_double)))
    return out.reshape(ny, nx)


def intensity_gradient(mask, weights, support, values, pitch=1.0, dose=1.0):
    ny, nx = mask.shape
    m = np.ascontiguousarray(mask, np.float64)
    w, s, v = _kargs(weights, support, values)
    out = np.zeros(nx * ny)
    _check(lib().ref_intensity_gradient(C.c_int(nx), C.c_int(ny), C.c_double(pitch), _p(m, C.c_double),
                                        C.c_int(len(w)), _p(w, C.c_double), C.c_int(len(s)),
                                        _p(s, C.c_int32), _p(v, C.c_double), C.c_double(dose),
                                        _p(out, C.c_double)))
    return out.reshape(ny, nx)


def weighted_gradient(mask, weights, support, values, W, pitch=1.0, dose=1.0):
    ny, nx = mask.shape
    m = np.ascontiguousarray(mask, np.float64)
    ww = np.ascontiguousarray(W, np.float64)
    w, s, v = _kargs(weights, support, values)
    out = np.zeros(nx * ny)
    _check(lib().ref_weighted_gradient(C.c_int(nx), C.c_int(ny), C.c_double(pitch), _p(m, C.c_double),
                                       C.c_int(len(w)), _p(w, C.c_double), C.c_int(len(s)),
                                       _p(s, C.c_int32), _p(v, C.c_double), C.c_double(dose),
                                       _p(ww, C.c_double), _p(out, C.c_double)))
    return out.reshape(ny, nx)


def z_print(field, weights, support, values, tau, pitch=1.0, dose=1.0):
    ny, nx = field.shape
    m = np.ascontiguousarray(field, np.float64)
    w, s, v = _kargs(weights, support, values)
    out = np.zeros(nx * ny)
    _check(lib().ref_z_print(C.c_int(nx), C.c_int(ny), C.c_double(pitch), _p(m, C.c_double),
                             C.c_int(len(w)), _p(w, C.c_double), C.c_int(len(s)), _p(s, C.c_int32),
                             _p(v, C.c_double), C.c_double(dose), C.c_double(tau), _p(out, C.c_double)))
    return out.reshape(ny, nx)


def z_round(raster, sigma_nm, tau, pitch=1.0):
    ny, nx = raster.shape
    m = np.ascontiguousarray(raster, np.float64)
    out = np.zeros(nx * ny)
    _check(lib().ref_z_round(C.c_int(nx), C.c_int(ny), C.c_double(pitch), _p(m, C.c_double),
                             C.c_double(sigma_nm), C.c_double(tau), _p(out, C.c_double)))
    return out.reshape(ny, nx)


def ilt_iteration(theta, target, weights, support, values, focus_weight, params, pitch=1.0):
    """theta updated in place; returns (cost, grad_theta). weights [F,K], values [F,K,S]."""
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
    _check(lib().ref_ilt_iteration(C.c_int(nx), C.c_int(ny), C.c_double(pitch), C.c_int(F), C.c_int(K),
                                   _p(w, C.c_double), C.c_int(len(s)), _p(s, C.c_int32), _p(v, C.c_double),
                                   _p(fw, C.c_double), _p(pr, C.c_double), _p(t, C.c_double),
                                   _p(theta, C.c_double), C.byref(cost), _p(grad, C.c_double)))
    return cost.value, grad.reshape(ny, nx)


def marching_squares(field, threshold, pitch=1.0, ox=0.0, oy=0.0):
    """reference marching_squares (contour.cpp:58-168): list of (xs, ys) loops."""
    f = np.ascontiguousarray(field, dtype=np.float64)
    ny, nx = f.shape
    nl, npnt = C.c_int64(), C.c_int64()
    _check(lib().ref_marching_squares(nx, ny, C.c_double(pitch), C.c_double(ox), C.c_double(oy),
                                      _p(f, C.c_double), C.c_double(threshold), C.byref(nl), C.byref(npnt)))
    st = np.zeros(nl.value + 1, np.int64)
    xs = np.zeros(max(npnt.value, 1))
    ys = np.zeros(max(npnt.value, 1))
    lib().ref_ms_get(_p(st, C.c_int64), _p(xs, C.c_double), _p(ys, C.c_double))
    return st, xs[:npnt.value], ys[:npnt.value]


def measure_epe(gauges, radius):
    """reference measure_epe (contour.cpp:181-201) on the last marching_squares result."""
    g = np.ascontiguousarray(gauges, dtype=np.float64).reshape(-1, 4)
    n = g.shape[0]
    epe = np.zeros(max(n, 1))
    op = np.zeros(max(n, 1), np.uint8)
    _check(lib().ref_measure_epe(_p(g, C.c_double), C.c_int64(n), C.c_double(radius), _p(epe, C.c_double),
                                 _p(op, C.c_uint8)))
    return epe[:n], op[:n].astype(bool)


def write_aimg(path, values, pitch=1.0):
    """reference write_aimg (io.cpp:317-330)."""
    v = np.ascontiguousarray(values, np.float64)
    ny, nx = v.shape
    _check(lib().ref_write_aimg(path.encode(), nx, ny, C.c_double(pitch), _p(v, C.c_double)))


def read_aimg(path, cap=1 << 26):
    """reference read_aimg (io.cpp:332-350): (nx, ny, pitch, values)."""
    nx, ny, p = C.c_int(), C.c_int(), C.c_double()
    _check(lib().ref_read_aimg(path.encode(), C.byref(nx), C.byref(ny), C.byref(p), None, C.c_int64(0)))
    out = np.zeros((ny.value, nx.value))
    _check(lib().ref_read_aimg(path.encode(), C.byref(nx), C.byref(ny), C.byref(p), _p(out, C.c_double),
                               C.c_int64(out.size)))
    return nx.value, ny.value, p.value, out
