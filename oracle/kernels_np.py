"""TEST INFRASTRUCTURE ONLY: numpy restatement of the reference SOCS kernel
source (build_tcc + decompose_tcc, /root/reference/proj/src/core/imaging.cpp
:46-216) for the oracle side of the harness — the reference arm of bench.py
and the CPU tests — so that nothing there loads the product library.

The reference's dense S x S eigensolve throws above S = 6000
(imaging.cpp:130-134), i.e. at every BASELINE tile size.  Its nonzero
eigenpairs are computed here through the same factorisation the product
generator uses (TCC = Q Q^H, Q[i][s] = sqrt(w_s) P(f_i + s fc; F);
G = Q^H Q = V L V^H, u = Q v / sqrt(l)), with the reference's semantics:
support order (imaging.cpp:115-129), descending eigenvalues clamped at 0,
k_fixed / energy-floor truncation (:183-191), and the largest-|.| component
made real positive (:192-196).  Pinned against the reference's own
decompose_tcc (oracle/_ref) at S <= 6000 in tests/test_oracle.py.
"""
from __future__ import annotations

import numpy as np


def annular_source(sigma_in: float, sigma_out: float, grid_n: int) -> np.ndarray:
    """make_annular_source (imaging.cpp:50-64): (n, 3) = sx, sy, weight (sum 1)."""
    c = -1.0 + (np.arange(grid_n) + 0.5) * 2.0 / grid_n
    sx, sy = np.meshgrid(c, c)  # iy outer, ix inner (row-major as the reference loop)
    sx, sy = sx.ravel(), sy.ravel()
    r = np.hypot(sx, sy)
    keep = (r >= sigma_in) & (r <= sigma_out)
    out = np.stack([sx[keep], sy[keep], np.ones(int(keep.sum()))], 1)
    out[:, 2] /= out[:, 2].sum()
    return out


def tcc_support(nx: int, ny: int, pitch: float, wavelength: float, na: float, max_src_r: float) -> np.ndarray:
    """(S, 2) signed (kx, ky) in the reference's row-major scan order (imaging.cpp:115-129)."""
    fmax = (1.0 + max_src_r) * na / wavelength
    kx = np.arange(nx)
    ky = np.arange(ny)
    skx = np.where(kx <= nx // 2, kx, kx - nx)
    sky = np.where(ky <= ny // 2, ky, ky - ny)
    KX, KY = np.meshgrid(skx, sky)
    fx = KX / (nx * pitch)
    fy = KY / (ny * pitch)
    m = fx * fx + fy * fy <= fmax * fmax * (1.0 + 1e-12)
    return np.stack([KX[m], KY[m]], 1).astype(np.int32)


def pupil(fx, fy, focus, wavelength, na):
    """paraxial pupil (imaging.cpp:72-84)."""
    f2 = fx * fx + fy * fy
    fc = na / wavelength
    return np.where(f2 <= fc * fc, np.exp(1j * (-np.pi * wavelength * focus * f2)), 0.0)


def socs_kernels(nx, ny, pitch, source, focus_nm, k_fixed=0, energy_floor=0.995, wavelength=13.5, na=0.33,
                 support=None):
    """One focus plane: (weights [K], support [S, 2], values [K, S] complex)."""
    src = np.asarray(source, np.float64)
    if support is None:
        support = tcc_support(nx, ny, pitch, wavelength, na, float(np.max(np.hypot(src[:, 0], src[:, 1]))))
    fc = na / wavelength
    fx = support[:, 0] / (nx * pitch)
    fy = support[:, 1] / (ny * pitch)
    Q = pupil(fx[:, None] + src[None, :, 0] * fc, fy[:, None] + src[None, :, 1] * fc, focus_nm, wavelength, na)
    Q = Q * np.sqrt(src[:, 2])[None, :]
    G = Q.conj().T @ Q
    lam, V = np.linalg.eigh(G)
    order = np.argsort(-lam, kind="stable")
    lam = np.maximum(lam[order], 0.0)
    V = V[:, order]
    total = lam.sum()
    S = len(support)
    ws, us = [], []
    captured = 0.0
    for r in range(len(lam)):
        if k_fixed > 0:
            if r >= k_fixed:
                break
        elif total > 0 and captured >= energy_floor * total and r > 0:
            break
        if r > 0 and (lam[r] <= 0 or r >= S or lam[r] <= 1e-13 * lam[0]):
            break
        u = Q @ V[:, r] / np.sqrt(lam[r]) if lam[r] > 0 else np.zeros(S, complex)
        i = int(np.argmax(np.abs(u)))
        if abs(u[i]) > 0:
            u = u * (np.conj(u[i]) / abs(u[i]))
        ws.append(lam[r])
        us.append(u)
        captured += lam[r]
    return np.asarray(ws), support, np.asarray(us)


def socs_kernel_stacks(n, pitch, foci, k_fixed, sigma_in=0.4, sigma_out=0.8, grid_n=21, wavelength=13.5, na=0.33):
    """Per-focus stacks padded to one order K (build_optics, opc.cpp:114-124):
    (weights [F, K], support [S, 2], values [F, K, S])."""
    src = annular_source(sigma_in, sigma_out, grid_n)
    out = [socs_kernels(n, n, pitch, src, f, k_fixed, wavelength=wavelength, na=na) for f in foci]
    K = max(len(w) for w, _, _ in out)
    S = len(out[0][1])
    W = np.zeros((len(foci), K))
    V = np.zeros((len(foci), K, S), complex)
    for i, (w, _, v) in enumerate(out):
        W[i, :len(w)] = w
        V[i, :len(w)] = v
    return W, out[0][1], V
