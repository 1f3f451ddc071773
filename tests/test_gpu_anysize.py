"""Arbitrary transform lengths on the GPU (fft.cuh: mixed radix 2/3/5/7 and
Bluestein) against numpy's FFT and the CPU oracle.

The reference fft2 (imaging.cpp:17-31, FFTW) is O(L log L) at every size and
make_window (opc.cpp:97-112) produces arbitrary window sizes; the reference
tests image 74x49 windows (test_opc_ai.cpp:116-117).  Tolerances: fp32 rel
L-inf <= 1e-4 (north star), fp64 at the reference's test_imaging.cpp bars.
"""
import time

import numpy as np
import pytest

import paper_2602_15036_b200 as L
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def rel_linf(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    s = np.abs(b).max()
    return np.abs(a - b).max() / (s if s > 0 else 1.0)


# (nx, ny): primes, 2*prime, 7^2, 3*7*47, the C-window sizes, tiny lengths
FFT_SIZES = [(1, 5), (2, 3), (12, 16), (74, 49), (97, 61), (125, 343), (1234, 987), (617, 2), (2048, 1536)]


@pytest.mark.parametrize("nx,ny", FFT_SIZES)
@pytest.mark.parametrize("prec,tol", [("f32", 2e-6), ("f64", 1e-13)])
@pytest.mark.parametrize("inverse", [False, True])
def test_fft2_any_size_vs_numpy(ctx, nx, ny, prec, tol, inverse):
    rng = np.random.default_rng(nx * 1000 + ny)
    a = rng.standard_normal((ny, nx)) + 1j * rng.standard_normal((ny, nx))
    got = L.fft2(a, inverse=inverse, precision=prec, ctx=ctx)
    want = np.fft.ifft2(a) * (nx * ny) if inverse else np.fft.fft2(a)
    # fp32 error of an O(L log L) transform grows ~ log L: bound by tol * log2(L)
    scale = max(1.0, np.log2(nx * ny)) if prec == "f32" else 1.0
    assert rel_linf(got, want) < tol * scale


def _kernels(nx, ny, pitch, K, gn=21, focus=(0.0,)):
    model = L.OpticalModel(source=L.make_annular_source(0.4, 0.8, gn))
    return L.build_socs_kernels(model, L.Grid(nx, ny, pitch), list(focus), k_fixed=K)


@pytest.mark.parametrize("nx,ny,pitch,K,gn", [(74, 49, 4.0, 0, 7), (1234, 987, 1.0, 8, 21)])
@pytest.mark.parametrize("prec,tol", [("f32", 1e-4), ("f64", 1e-10)])
def test_image_and_gradient_any_size_vs_oracle(ctx, nx, ny, pitch, K, gn, prec, tol):
    rng = np.random.default_rng(nx + 3 * ny)
    ks = _kernels(nx, ny, pitch, K, gn, focus=(20.0,))
    mask = (rng.random((ny, nx)) > 0.5).astype(np.float64)
    want = O.image_socs(mask, ks.weights[0], ks.support, ks.values[0], dose=1.1)
    dk = L.DeviceKernels(ks, prec, ctx)
    got = dk.image(mask, dose=1.1)["intensity"]
    assert rel_linf(got, want) < tol, dk.info()
    W = rng.standard_normal((ny, nx))
    gw = O.weighted_gradient(mask, ks.weights[0], ks.support, ks.values[0], W, dose=1.1)
    gg = L.intensity_gradient(mask, dk, 1.1, weight=W, precision=prec, ctx=ctx)
    assert rel_linf(gg, gw) < (tol if prec == "f64" else 1e-4)


def test_any_size_is_n_log_n(ctx):
    """A prime-length window costs about what the next power of two costs
    (Bluestein), not the O(L^2) of a direct DFT: 1234x987 vs 2048x2048."""
    import torch
    rng = np.random.default_rng(5)

    def t(nx, ny):
        a = rng.standard_normal((ny, nx)) + 1j * rng.standard_normal((ny, nx))
        buf = torch.tensor(np.stack([a.real, a.imag], -1), dtype=torch.float32, device="cuda")
        from paper_2602_15036_b200._lib import F32, check, lib
        for _ in range(3):
            check(lib().lithogpu_fft2(ctx.handle, buf.data_ptr(), F32, nx, ny, 0))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            check(lib().lithogpu_fft2(ctx.handle, buf.data_ptr(), F32, nx, ny, 0))
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / 10
    t_odd, t_pow2 = t(1234, 987), t(2048, 2048)
    print(f"fft2 f32 device: 1234x987 {t_odd * 1e3:.3f} ms, 2048x2048 {t_pow2 * 1e3:.3f} ms")
    assert t_odd < 4 * t_pow2
