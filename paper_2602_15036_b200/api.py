"""Host-side mirror of the reference `litho` imaging / ILT interface, over the
C ABI in include/lithogpu.h.

Names, argument meaning and error behaviour follow the reference C++ API
(proj/src/core/raster.hpp, imaging.hpp, ai.hpp): `rasterize_layer`,
`image_socs`, `resist_filter`, `gaussian_blur`, `intensity_gradient`,
`z_print`, `z_round`, `make_annular_source`, `Grid`, `OpticalModel`,
`SocsKernelSet`.  Preconditions raise ValueError (reference
std::invalid_argument), computational failures RuntimeError.

Arrays may be numpy (host; results come back as numpy) or torch CUDA tensors
(device-resident; results are torch tensors on the same device, computed on
the context stream without a host round trip).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import F32, F64, U8, LithoError, LithoUsageError, check, lib

try:  # torch is plumbing only (device memory / streams); optional for host use
    import torch
except Exception:  # pragma: no cover
    torch = None


# ---------------------------------------------------------------------------
# geometry / optics value types (reference raster.hpp:10-20, imaging.hpp:15-47)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Grid:
    nx: int
    ny: int
    pitch_nm: float = 1.0
    origin_x_nm: float = 0.0
    origin_y_nm: float = 0.0

    def size(self) -> int:
        return self.nx * self.ny

    def index(self, ix: int, iy: int) -> int:
        return iy * self.nx + ix

    def c(self) -> _lib.Grid:
        return _lib.Grid(self.nx, self.ny, self.pitch_nm, self.origin_x_nm, self.origin_y_nm)


def make_annular_source(sigma_in: float, sigma_out: float, grid_n: int = 21) -> np.ndarray:
    """(n, 3) array of (sx, sy, weight), weights sum to 1 (imaging.cpp:50-64)."""
    if sigma_out <= sigma_in or sigma_out <= 0:
        raise ValueError("annular source: need 0 <= sigma_in < sigma_out")
    n = C.c_int()
    check(lib().lithogpu_source_annular(sigma_in, sigma_out, grid_n, C.byref(n), None), host=True)
    out = np.zeros((n.value, 3))
    check(lib().lithogpu_source_annular(sigma_in, sigma_out, grid_n, C.byref(n),
                                        out.ctypes.data), host=True)
    return out


def make_circular_source(sigma_out: float, grid_n: int = 21) -> np.ndarray:
    return make_annular_source(0.0, sigma_out, grid_n)


def make_point_source() -> np.ndarray:
    return np.array([[0.0, 0.0, 1.0]])


@dataclass
class OpticalModel:
    """reference OpticalModel (imaging.hpp:32-47)."""
    wavelength_nm: float = 13.5
    na: float = 0.33
    source: np.ndarray = field(default_factory=make_point_source)
    high_na_defocus: bool = False
    resist_sigma_nm: float = 2.0
    t_eff: float = 0.25
    tau_print: float = 0.25
    tau_round: float = 0.5
    dose: float = 1.0

    def pupil_cutoff(self) -> float:
        return self.na / self.wavelength_nm

    def max_source_radius(self) -> float:
        return float(np.max(np.hypot(self.source[:, 0], self.source[:, 1]))) if len(self.source) else 0.0


@dataclass
class SocsKernelSet:
    """Band-sparse SOCS kernel stacks (reference SocsKernelSet, imaging.hpp:78-87,
    one per focus plane as build_optics, opc.cpp:114-124).

    weights [F, K] (descending per focus), support [S, 2] signed (kx, ky),
    values [F, K, S] complex = kernels_freq at the support indices.
    """
    grid: Grid
    focus_nm: Sequence[float]
    weights: np.ndarray
    support: np.ndarray
    values: np.ndarray
    captured_energy: Sequence[float] = ()

    @property
    def n_focus(self) -> int:
        return self.weights.shape[0]

    def order(self) -> int:
        return self.weights.shape[1]

    def focus_stack(self, f: int) -> "SocsKernelSet":
        return SocsKernelSet(self.grid, [self.focus_nm[f]], self.weights[f:f + 1],
                             self.support, self.values[f:f + 1])

    @staticmethod
    def from_full_grid(grid: Grid, weights, kernels_freq, focus_nm=0.0) -> "SocsKernelSet":
        """From reference-style full-grid spectra [K, ny, nx] (nonzeros = support)."""
        kf = np.asarray(kernels_freq)
        nz = np.any(kf != 0, axis=0)
        ky, kx = np.nonzero(nz)
        skx = np.where(kx <= grid.nx // 2, kx, kx - grid.nx)
        sky = np.where(ky <= grid.ny // 2, ky, ky - grid.ny)
        support = np.stack([skx, sky], 1).astype(np.int32)
        vals = kf[:, ky, kx]
        return SocsKernelSet(grid, [focus_nm], np.asarray(weights, float)[None], support, vals[None])


def tcc_support(model: OpticalModel, grid: Grid) -> np.ndarray:
    n = C.c_int()
    args = (grid.nx, grid.ny, grid.pitch_nm, model.wavelength_nm, model.na, model.max_source_radius())
    check(lib().lithogpu_tcc_support(*args, C.byref(n), None), host=True)
    out = np.zeros((n.value, 2), np.int32)
    check(lib().lithogpu_tcc_support(*args, C.byref(n), out.ctypes.data), host=True)
    return out


def build_socs_kernels(model: OpticalModel, grid: Grid, focus_nm: Sequence[float] = (0.0,),
                       k_fixed: int = 0, energy_floor: float = 0.995, backend: str = "host",
                       ctx: Optional["Context"] = None) -> SocsKernelSet:
    """build_tcc + decompose_tcc (imaging.cpp:113-216) for each focus plane,
    via the TCC = Q Q^H factorisation (fp64).  backend "host" (OpenMP, Jacobi
    eigensolve) or "gpu" (cuBLAS Gram + cuSOLVER eigensolve, all foci in one
    call).  All stacks are padded to the same order K (the max over foci;
    missing kernels have weight 0)."""
    support = tcc_support(model, grid)
    S = len(support)
    if S == 0:
        raise ValueError("decompose_tcc: empty support")
    src = np.ascontiguousarray(model.source, np.float64)
    cap = k_fixed if k_fixed > 0 else len(src)
    if backend == "gpu":
        ctx = ctx or default_context()
        nf = len(focus_nm)
        foc = np.ascontiguousarray(focus_nm, np.float64)
        order = np.zeros(nf, np.int32)
        capd = np.zeros(nf)
        w = np.zeros((nf, cap))
        v = np.zeros((nf, cap, S, 2))
        check(lib().lithogpu_socs_kernels_gpu(ctx.handle, grid.nx, grid.ny, grid.pitch_nm, model.wavelength_nm,
                                              model.na, int(model.high_na_defocus), src.ctypes.data, len(src), nf,
                                              foc.ctypes.data, S, support.ctypes.data, int(k_fixed),
                                              float(energy_floor), cap, order.ctypes.data, capd.ctypes.data,
                                              w.ctypes.data, v.ctypes.data))
        K = int(order.max())
        V = v[:, :K, :, 0] + 1j * v[:, :K, :, 1]
        W = w[:, :K].copy()
        for f in range(nf):  # padding kernels of lower-rank stacks: weight 0
            W[f, order[f]:] = 0.0
            V[f, order[f]:] = 0.0
        return SocsKernelSet(grid, list(focus_nm), W, support, V, list(capd))
    if backend != "host":
        raise ValueError("build_socs_kernels: backend must be 'host' or 'gpu'")
    ws, vs, caps = [], [], []
    for f in focus_nm:
        K = C.c_int()
        capd = C.c_double()
        w = np.zeros(cap)
        v = np.zeros((cap, S, 2))
        check(lib().lithogpu_socs_kernels(grid.nx, grid.ny, grid.pitch_nm, model.wavelength_nm, model.na,
                                          int(model.high_na_defocus), src.ctypes.data, len(src), float(f),
                                          S, support.ctypes.data, int(k_fixed), float(energy_floor), cap,
                                          C.byref(K), C.byref(capd), w.ctypes.data, v.ctypes.data), host=True)
        ws.append(w[:K.value])
        vs.append(v[:K.value, :, 0] + 1j * v[:K.value, :, 1])
        caps.append(capd.value)
    K = max(len(w) for w in ws)
    W = np.zeros((len(ws), K))
    V = np.zeros((len(ws), K, S), np.complex128)
    for i, (w, v) in enumerate(zip(ws, vs)):
        W[i, :len(w)] = w
        V[i, :len(w)] = v
    return SocsKernelSet(grid, list(focus_nm), W, support, V, caps)


# ---------------------------------------------------------------------------
# context / buffers
# ---------------------------------------------------------------------------
class Context:
    """One CUDA device + stream (lithogpu_ctx)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        h = C.c_void_p()
        check(lib().lithogpu_ctx_create(device, C.byref(h)))
        self._h = h
        self.device = device
        if stream is not None:
            self.set_stream(stream)

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream) -> None:
        ptr = stream if isinstance(stream, int) else getattr(stream, "cuda_stream", stream)
        check(lib().lithogpu_ctx_set_stream(self._h, C.c_void_p(ptr)))

    def synchronize(self) -> None:
        check(lib().lithogpu_ctx_synchronize(self._h))

    def launch_count(self) -> int:
        return int(lib().lithogpu_ctx_launch_count(self._h))

    def set_profiling(self, on: bool) -> None:
        check(lib().lithogpu_ctx_set_profiling(self._h, int(bool(on))))

    def profile_report(self, reset: bool = True) -> dict:
        """{kernel name: (launches, total ms)} from per-launch CUDA events."""
        buf = C.create_string_buffer(1 << 16)
        check(lib().lithogpu_ctx_profile_report(self._h, buf, len(buf), int(reset)))
        out = {}
        for line in buf.value.decode().splitlines():
            name, n, ms = line.split()
            out[name] = (int(n), float(ms))
        return out

    def fp32_peak_tflops(self) -> float:
        v = C.c_double()
        check(lib().lithogpu_fp32_peak(self._h, C.byref(v)))
        return v.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().lithogpu_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: dict = {}


def default_context(device: int = 0) -> Context:
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


def _is_torch(a) -> bool:
    return torch is not None and isinstance(a, torch.Tensor)


_NP2DT = {np.dtype(np.float32): F32, np.dtype(np.float64): F64, np.dtype(np.uint8): U8}


def _buf(a):
    """(pointer, dtype code, keepalive) for a numpy array or torch tensor."""
    if _is_torch(a):
        if not a.is_contiguous():
            a = a.contiguous()
        m = {torch.float32: F32, torch.float64: F64, torch.uint8: U8}
        if a.dtype not in m:
            a = a.to(torch.float64)
        return a.data_ptr(), m[a.dtype], a
    a = np.ascontiguousarray(a)
    if a.dtype not in _NP2DT:
        a = a.astype(np.float64)
    return a.ctypes.data, _NP2DT[a.dtype], a


def _empty_like(ref, shape, dt):
    if _is_torch(ref):
        tdt = {F32: torch.float32, F64: torch.float64, U8: torch.uint8}[dt]
        return torch.empty(shape, dtype=tdt, device=ref.device)
    ndt = {F32: np.float32, F64: np.float64, U8: np.uint8}[dt]
    return np.empty(shape, ndt)


# ---------------------------------------------------------------------------
# device kernel stacks
# ---------------------------------------------------------------------------
class DeviceKernels:
    """Kernel stacks uploaded to one GPU (lithogpu_kernels), fp32 or fp64."""

    def __init__(self, kernels: SocsKernelSet, precision: str = "f32", ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.kernels = kernels
        self.grid = kernels.grid
        self.precision = precision
        w = np.ascontiguousarray(kernels.weights, np.float64)
        F, K = w.shape
        s = np.ascontiguousarray(kernels.support, np.int32)
        v = np.ascontiguousarray(np.stack([kernels.values.real, kernels.values.imag], -1), np.float64)
        assert v.shape == (F, K, len(s), 2)
        h = C.c_void_p()
        g = self.grid.c()
        check(lib().lithogpu_kernels_create(self.ctx.handle, C.byref(g), F32 if precision == "f32" else F64,
                                            F, K, w.ctypes.data, len(s), s.ctypes.data, v.ctypes.data,
                                            C.byref(h)))
        self._h = h
        self.F, self.K = F, K

    @property
    def handle(self):
        return self._h

    def info(self):
        a, b, c, d = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        check(lib().lithogpu_kernels_info(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
        k, fs = C.c_int(), C.c_int()
        check(lib().lithogpu_kernels_fast_order(self._h, C.byref(k)))
        check(lib().lithogpu_kernels_fast_stacks(self._h, C.byref(fs)))
        return {"nx_sub": a.value, "ny_sub": b.value, "band_x": c.value, "band_y": d.value,
                "fast_order": k.value, "fast_stacks": fs.value}

    def close(self):
        if getattr(self, "_h", None):
            lib().lithogpu_kernels_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- imaging ------------------------------------------------------------
    def image(self, mask, dose: float = 1.0, focus: int = 0, sigma_nm: float = 0.0,
              threshold: float = 0.0, want=("intensity",), out_dtype=None):
        """Fused forward; returns dict with requested 'intensity' / 'resist' / 'print'."""
        mp, mdt, keep = _buf(mask)
        odt = out_dtype if out_dtype is not None else (F32 if self.precision == "f32" else F64)
        shape = (self.grid.ny, self.grid.nx)
        res = {}
        I = _empty_like(mask, shape, odt) if "intensity" in want else None
        R = _empty_like(mask, shape, odt) if "resist" in want else None
        P = _empty_like(mask, shape, U8) if "print" in want else None
        ptr = lambda a: None if a is None else (a.data_ptr() if _is_torch(a) else a.ctypes.data)
        check(lib().lithogpu_image_resist(self._h, focus, mp, mdt, dose, sigma_nm, threshold,
                                          ptr(I), ptr(R), odt, ptr(P)))
        if I is not None:
            res["intensity"] = I
        if R is not None:
            res["resist"] = R
        if P is not None:
            res["print"] = P
        return res

    def gradient(self, mask, dose: float = 1.0, weight=None, focus: int = 0, out_dtype=None):
        mp, mdt, k1 = _buf(mask)
        wp, wdt, k2 = (None, F64, None) if weight is None else _buf(weight)
        odt = out_dtype if out_dtype is not None else (F32 if self.precision == "f32" else F64)
        out = _empty_like(mask, (self.grid.ny, self.grid.nx), odt)
        optr = out.data_ptr() if _is_torch(out) else out.ctypes.data
        check(lib().lithogpu_intensity_gradient(self._h, focus, mp, mdt, wp, wdt, dose, optr, odt))
        return out


# ---------------------------------------------------------------------------
# reference-named functions
# ---------------------------------------------------------------------------
def _kernels_on_device(kernels, precision, ctx):
    if isinstance(kernels, DeviceKernels):
        return kernels
    return DeviceKernels(kernels, precision, ctx)


def image_socs(mask, kernels, dose: float = 1.0, focus: int = 0, precision: str = "f64",
               ctx: Optional[Context] = None):
    """image_socs (imaging.cpp:218-241): I = dose sum_k w_k |O (x) Phi_k|^2."""
    dk = _kernels_on_device(kernels, precision, ctx)
    return dk.image(mask, dose, focus, want=("intensity",))["intensity"]


def fft2(values, inverse: bool = False, precision: str = "f64", ctx: Optional[Context] = None) -> np.ndarray:
    """fft2 (imaging.hpp:124, imaging.cpp:17-31): unnormalized 2-D DFT of a
    [ny][nx] complex grid (x contiguous), forward e^{-i}, backward e^{+i}.
    O(L log L) at every size (power-of-two Stockham, mixed radix 2/3/5/7,
    Bluestein otherwise).  Returns a new complex128 array."""
    a = np.asarray(values)
    if a.ndim != 2:
        raise ValueError("fft2: size mismatch")
    ny, nx = a.shape
    rt = np.float32 if precision == "f32" else np.float64
    buf = np.ascontiguousarray(np.stack([a.real, a.imag], -1), rt)
    ctx = ctx or default_context()
    check(lib().lithogpu_fft2(ctx.handle, buf.ctypes.data, F32 if precision == "f32" else F64, nx, ny,
                              1 if inverse else 0))
    return buf[..., 0].astype(np.float64) + 1j * buf[..., 1].astype(np.float64)


def gaussian_blur(grid: Grid, values, sigma_nm: float, ctx: Optional[Context] = None):
    """gaussian_blur (imaging.cpp:287-314): cyclic unit-sum truncated Gaussian."""
    if sigma_nm < 0:
        raise ValueError("gaussian_blur: negative sigma")
    ctx = ctx or default_context()
    p, dt, keep = _buf(values)
    if dt == U8:
        raise ValueError("gaussian_blur: real input required")
    out = _empty_like(values, (grid.ny, grid.nx), dt)
    optr = out.data_ptr() if _is_torch(out) else out.ctypes.data
    g = grid.c()
    check(lib().lithogpu_gaussian_blur(ctx.handle, C.byref(g), p, dt, sigma_nm, optr))
    return out


@dataclass
class ResistImage:
    grid: Grid
    focus_nm: float
    threshold: float
    values: object


def resist_filter(grid: Grid, aerial, sigma_nm: float, threshold: float, focus_nm: float = 0.0,
                  ctx: Optional[Context] = None) -> ResistImage:
    """resist_filter (imaging.cpp:316-323)."""
    return ResistImage(grid, focus_nm, threshold, gaussian_blur(grid, aerial, sigma_nm, ctx))


def threshold(values, tau: float, ctx: Optional[Context] = None):
    ctx = ctx or default_context()
    p, dt, keep = _buf(values)
    shape = tuple(values.shape)
    out = _empty_like(values, shape, F64)
    optr = out.data_ptr() if _is_torch(out) else out.ctypes.data
    n = int(np.prod(shape))
    check(lib().lithogpu_threshold(ctx.handle, n, p, dt, tau, optr, F64))
    return out


def z_print(field_values, kernels, dose: float, tau_print: float, precision: str = "f64",
            ctx: Optional[Context] = None):
    """z_print (ai.cpp:85-94): threshold of the best-focus image, {0,1}."""
    return threshold(image_socs(field_values, kernels, dose, 0, precision, ctx), tau_print, ctx)


def z_round(grid: Grid, target_raster, sigma_nm: float, tau_round: float, ctx: Optional[Context] = None):
    """z_round (ai.cpp:76-83): blur then threshold, {0,1}."""
    if not (0 < tau_round < 1):
        raise ValueError("z_round: tau outside (0,1)")
    return threshold(gaussian_blur(grid, target_raster, sigma_nm, ctx), tau_round, ctx)


def intensity_gradient(mask, kernels, dose: float, weight=None, focus: int = 0, precision: str = "f64",
                       ctx: Optional[Context] = None):
    """intensity_gradient (ai.cpp:11-42); `weight` W generalises it to
    d(sum_r W(r) I(r))/dM (W=None: the reference's uniform case)."""
    dk = _kernels_on_device(kernels, precision, ctx)
    return dk.gradient(mask, dose, weight, focus)


def rasterize_layer(polygons, grid: Grid, dbu_per_nm: float, ctx: Optional[Context] = None):
    """rasterize_layer (raster.cpp:53-95), fp64 bit-exact, on HEALED polygons
    (list of (n,2) int64 vertex arrays in the reference heal() output order)."""
    if grid.pitch_nm <= 0:
        raise ValueError("rasterize_layer: nonpositive pitch")
    if grid.nx <= 0 or grid.ny <= 0:
        raise ValueError("rasterize_layer: empty grid")
    ctx = ctx or default_context()
    if polygons:
        xy = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int64).reshape(-1, 2) for p in polygons]))
    else:
        xy = np.zeros((1, 2), np.int64)
    starts = np.zeros(len(polygons) + 1, np.int64)
    starts[1:] = np.cumsum([len(p) for p in polygons])
    out = np.empty((grid.ny, grid.nx), np.float64)
    g = grid.c()
    check(lib().lithogpu_rasterize(ctx.handle, C.byref(g), xy.ctypes.data, starts.ctypes.data,
                                   len(polygons), dbu_per_nm, out.ctypes.data))
    return out


# ---------------------------------------------------------------------------
# contours and EPE (reference contour.hpp / contour.cpp:58-201)
# ---------------------------------------------------------------------------
class ContourSet:
    """marching_squares result (reference ContourSet, contour.hpp:13-27):
    loops[i] = (xs, ys) closed polyline in nm, CCW around printed regions.
    Keeps the device crossing graph for measure_epe."""

    def __init__(self, handle, ctx):
        self._h = handle
        self.ctx = ctx
        nl, npnt = C.c_int64(), C.c_int64()
        check(lib().lithogpu_contours_size(self._h, C.byref(nl), C.byref(npnt)))
        self.loop_start = np.zeros(nl.value + 1, np.int64)
        self.xs = np.zeros(npnt.value, np.float64)
        self.ys = np.zeros(npnt.value, np.float64)
        check(lib().lithogpu_contours_get(self._h, self.loop_start.ctypes.data,
                                          self.xs.ctypes.data if npnt.value else None,
                                          self.ys.ctypes.data if npnt.value else None))

    @property
    def loops(self):
        st = self.loop_start
        return [(self.xs[st[i]:st[i + 1]], self.ys[st[i]:st[i + 1]]) for i in range(len(st) - 1)]

    def close(self):
        if getattr(self, "_h", None):
            lib().lithogpu_contours_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def marching_squares(field, grid: Grid, threshold: float, ctx: Optional[Context] = None) -> ContourSet:
    """marching_squares (contour.cpp:58-168) of a resist image (ny x nx f64,
    numpy or CUDA tensor) at `threshold`; bit-identical loops."""
    ctx = ctx or default_context()
    if _is_torch(field):
        field = field.to(torch.float64)
    else:
        field = np.ascontiguousarray(field, np.float64)
    if tuple(field.shape) != (grid.ny, grid.nx):
        raise ValueError("marching_squares: field shape does not match the grid")
    finite = bool(torch.isfinite(field).all()) if _is_torch(field) else bool(np.isfinite(field).all())
    if not finite:  # reference std::invalid_argument (contour.cpp:62-63)
        raise ValueError("marching_squares: non-finite field")
    buf, _, keep = _buf(field)
    h = C.c_void_p()
    g = grid.c()
    check(lib().lithogpu_marching_squares(ctx.handle, C.byref(g), buf, threshold, C.byref(h)))
    return ContourSet(h, ctx)


def measure_epe(contours: ContourSet, gauges, search_radius_nm: float):
    """measure_epe (contour.cpp:181-201): gauges (n, 4) = x, y, nx, ny (site and
    unit outward normal, nm).  Returns (epe_nm[n], open[n] bool)."""
    g = np.ascontiguousarray(gauges, np.float64).reshape(-1, 4)
    n = g.shape[0]
    epe = np.zeros(max(n, 1), np.float64)
    op = np.zeros(max(n, 1), np.uint8)
    check(lib().lithogpu_measure_epe(contours._h, g.ctypes.data, n, search_radius_nm, epe.ctypes.data,
                                     op.ctypes.data))
    return epe[:n], op[:n].astype(bool)


def evaluate_epe(masks, kernels, gauges, dose: float, sigma_nm: float, t_eff: float, search_radius_nm: float,
                 focus: int = 0, precision: str = "f64", ctx: Optional[Context] = None, want_resist: bool = False):
    """evaluate_epe (opc.cpp:140-151) on the device for one mask raster or a
    batch (m, ny, nx) — e.g. the MEEF probe batches of estimate_meef
    (opc.cpp:153-202): image -> resist_filter -> marching_squares ->
    measure_epe, imaged in one batched launch sequence.
    Returns (epe [m, n], open [m, n] bool[, resist [m, ny, nx]])."""
    dk = _kernels_on_device(kernels, precision, ctx)
    single = len(tuple(masks.shape) if hasattr(masks, "shape") else np.shape(masks)) == 2
    if _is_torch(masks):  # device-resident masks stay on the device
        m = masks[None] if single else masks
        finite = bool(torch.isfinite(m).all())
    else:
        m = np.ascontiguousarray(masks, np.float64)
        if single:
            m = m[None]
        finite = bool(np.isfinite(m).all())
    if not finite:  # the resist field would be non-finite (reference contour.cpp:62-63)
        raise ValueError("evaluate_epe: non-finite mask")
    mp, mdt, keep = _buf(m)
    nm = m.shape[0]
    g = np.ascontiguousarray(gauges, np.float64).reshape(-1, 4)
    n = g.shape[0]
    epe = np.zeros((nm, max(n, 1)), np.float64)
    op = np.zeros((nm, max(n, 1)), np.uint8)
    res = np.zeros(tuple(m.shape), np.float64) if want_resist else None
    check(lib().lithogpu_evaluate_epe(dk.handle, focus, nm, mp, mdt, dose, sigma_nm, t_eff,
                                      g.ctypes.data if n else None, n, search_radius_nm, epe.ctypes.data,
                                      op.ctypes.data, res.ctypes.data if want_resist else None))
    out = (epe[:, :n], op[:, :n].astype(bool))
    if single:
        out = (out[0][0], out[1][0])
    if want_resist:
        out = out + ((res[0] if single else res),)
    return out


# ---------------------------------------------------------------------------
# AIMG tile I/O (reference io.hpp:39-43 / io.cpp:317-350)
# ---------------------------------------------------------------------------
def write_aimg(paths, grid: Grid, values, ctx: Optional[Context] = None) -> None:
    """write_aimg for one image (path str, (ny, nx)) or a batch of tiles
    (list of paths, (t, ny, nx)); numpy or CUDA tensors (f32/f64).  Device
    tiles stream through a pinned double buffer."""
    ctx = ctx or default_context()
    single = isinstance(paths, (str, bytes))
    plist = [paths] if single else list(paths)
    ptr, dt, keep = _buf(values)
    arr = (C.c_char_p * len(plist))(*[p.encode() if isinstance(p, str) else p for p in plist])
    g = grid.c()
    check(lib().lithogpu_write_aimg(ctx.handle, C.byref(g), len(plist), C.cast(arr, C.c_void_p), ptr, dt))


def read_aimg(path: str, ctx: Optional[Context] = None):
    """read_aimg: (Grid (origin 0, as the reference), values (ny, nx) f64)."""
    ctx = ctx or default_context()
    nx, ny, p = C.c_int(), C.c_int(), C.c_double()
    check(lib().lithogpu_read_aimg(ctx.handle, path.encode(), C.byref(nx), C.byref(ny), C.byref(p), None))
    out = np.empty((ny.value, nx.value), np.float64)
    check(lib().lithogpu_read_aimg(ctx.handle, path.encode(), C.byref(nx), C.byref(ny), C.byref(p),
                                   out.ctypes.data))
    return Grid(nx.value, ny.value, p.value), out


# ---------------------------------------------------------------------------
# layout JSON (reference io.hpp load_layout / io.cpp:53-116)
# ---------------------------------------------------------------------------
@dataclass
class Layout:
    """load_layout result: dbu per nm as num/den, layers = [(name, [polygon (n, 2) int64, ...])]."""
    dbu_num: int
    dbu_den: int
    layers: list

    def dbu_per_nm(self) -> float:
        return self.dbu_num / self.dbu_den


def load_layout(path: str, device=None) -> Layout:
    """Reference layout JSON -> polygons (lithogpu_layout_load / _get).  With
    `device` (a torch device), each layer instead comes back as flattened
    device buffers (xy [V, 2] int64, poly_start [P + 1] int64) ready for
    lithogpu_rasterize."""
    h = C.c_void_p()
    check(lib().lithogpu_layout_load(path.encode(), C.byref(h)))
    try:
        nl, num, den = C.c_int(), C.c_int64(), C.c_int64()
        check(lib().lithogpu_layout_info(h, C.byref(nl), C.byref(num), C.byref(den)))
        layers = []
        for li in range(nl.value):
            name, npoly, nvert = C.c_char_p(), C.c_int64(), C.c_int64()
            check(lib().lithogpu_layout_layer(h, li, C.byref(name), C.byref(npoly), C.byref(nvert)))
            if device is not None:
                xy = torch.empty((nvert.value, 2), dtype=torch.int64, device=device)
                st = torch.empty(npoly.value + 1, dtype=torch.int64, device=device)
                check(lib().lithogpu_layout_get(h, li, xy.data_ptr() if nvert.value else None, st.data_ptr()))
                layers.append((name.value.decode(), (xy, st)))
                continue
            xy = np.empty((nvert.value, 2), np.int64)
            st = np.empty(npoly.value + 1, np.int64)
            check(lib().lithogpu_layout_get(h, li, xy.ctypes.data if nvert.value else None, st.ctypes.data))
            layers.append((name.value.decode(), [xy[st[i]:st[i + 1]] for i in range(npoly.value)]))
        return Layout(num.value, den.value, layers)
    finally:
        lib().lithogpu_layout_destroy(h)


# ---------------------------------------------------------------------------
# ILT
# ---------------------------------------------------------------------------
@dataclass
class IltParams:
    mask_steepness: float = 4.0
    resist_beta: float = 30.0
    threshold: float = 0.25
    resist_sigma_nm: float = 2.0
    dose: float = 1.0
    step: float = 1.0
    focus_weights: Optional[Sequence[float]] = None


class IltSolver:
    """Pixel ILT over `n_tiles` halo-padded tiles sharing one kernel stack set."""

    def __init__(self, kernels, params: IltParams, n_tiles: int = 1, precision: str = "f32",
                 ctx: Optional[Context] = None):
        self.dk = _kernels_on_device(kernels, precision, ctx)
        F = self.dk.F
        fw = params.focus_weights if params.focus_weights is not None else [1.0 / F] * F
        if len(fw) != F:
            raise ValueError(f"IltParams.focus_weights: {len(fw)} weights for {F} focus stacks")
        if not all(math.isfinite(float(c)) and float(c) >= 0 for c in fw):
            raise ValueError("IltParams.focus_weights: weights must be finite and >= 0")
        self._fw = (C.c_double * F)(*fw)
        self.params = params
        p = _lib.IltParams(params.mask_steepness, params.resist_beta, params.threshold,
                           params.resist_sigma_nm, params.dose, params.step,
                           C.cast(self._fw, C.POINTER(C.c_double)))
        h = C.c_void_p()
        check(lib().lithogpu_ilt_create(self.dk.handle, C.byref(p), n_tiles, C.byref(h)))
        self._h = h
        self.n_tiles = n_tiles
        self.grid = self.dk.grid

    def set_tiles(self, target, theta0=None):
        tp, tdt, k1 = _buf(target)
        if theta0 is None:
            check(lib().lithogpu_ilt_set_tiles(self._h, tp, None, tdt))
        else:
            hp, hdt, k2 = _buf(theta0)
            if hdt != tdt:
                raise ValueError("target and theta0 dtypes differ")
            check(lib().lithogpu_ilt_set_tiles(self._h, tp, hp, tdt))

    def run(self, iterations: int, with_gmax: bool = False):
        cost = np.zeros((iterations, self.n_tiles))
        gmax = np.zeros((iterations, self.n_tiles)) if with_gmax else None
        check(lib().lithogpu_ilt_run(self._h, iterations, cost.ctypes.data,
                                     gmax.ctypes.data if with_gmax else None))
        return (cost, gmax) if with_gmax else cost

    def gradient(self, like=None, dtype=None):
        """(cost [n_tiles], dcost/dtheta [n_tiles, ny, nx]) at the current
        theta, theta unchanged (lithogpu_ilt_gradient).  `like`: a CUDA tensor
        to allocate the gradient next to (device-resident result)."""
        dt = dtype if dtype is not None else (F32 if self.dk.precision == "f32" else F64)
        shape = (self.n_tiles, self.grid.ny, self.grid.nx)
        g = _empty_like(like if like is not None else np.empty(0), shape, dt)
        cost = np.zeros(self.n_tiles)
        gp = g.data_ptr() if _is_torch(g) else g.ctypes.data
        check(lib().lithogpu_ilt_gradient(self._h, cost.ctypes.data, gp, dt))
        return cost, g

    def run_device(self, iterations: int, cost_dev=None, gmax_dev=None):
        """Enqueue without host sync of results (cost_dev / gmax_dev: device
        f64 [iters, tiles] or None; gmax = max |dL/dtheta| per tile)."""
        ptr = cost_dev.data_ptr() if cost_dev is not None else None
        gptr = gmax_dev.data_ptr() if gmax_dev is not None else None
        check(lib().lithogpu_ilt_run(self._h, iterations, ptr, gptr))

    def get_tiles(self, like=None, dtype=F64):
        shape = (self.n_tiles, self.grid.ny, self.grid.nx)
        theta = _empty_like(like if like is not None else np.empty(0), shape, dtype)
        mask = _empty_like(like if like is not None else np.empty(0), shape, dtype)
        ptr = lambda a: a.data_ptr() if _is_torch(a) else a.ctypes.data
        check(lib().lithogpu_ilt_get_tiles(self._h, ptr(theta), ptr(mask), dtype))
        return theta, mask

    def get_window(self, tile: int, x0: int, y0: int, w: int, h: int, out=None, dtype=F32, async_: bool = False):
        """Mask window of one tile (lithogpu_ilt_get_window) into `out`
        (numpy / CUDA tensor view with unit column stride, e.g. a block of
        the stitched chip mask) or a new (h, w) host array.  async_: stream-
        ordered without waiting (lithogpu_ilt_get_window_async; `out` must be
        device or pinned host memory, valid after the context synchronizes)."""
        if out is None:
            out = np.empty((h, w), np.float32 if dtype == F32 else np.float64)
        if _is_torch(out):
            ptr, stride = out.data_ptr(), out.stride(0)
            dt = {torch.float32: F32, torch.float64: F64}[out.dtype]
        else:
            if out.strides[1] != out.itemsize:
                raise ValueError("get_window: out needs unit column stride")
            ptr, stride = out.ctypes.data, out.strides[0] // out.itemsize
            dt = _NP2DT[out.dtype]
        fn = lib().lithogpu_ilt_get_window_async if async_ else lib().lithogpu_ilt_get_window
        check(fn(self._h, tile, x0, y0, w, h, ptr, stride, dt))
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib().lithogpu_ilt_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
