"""Library baseline: the same band-limited decimated SOCS ILT iteration as
liblithogpu.so, written with cuFFT (torch.fft) — batched plans over tiles,
every field resident in HBM, the iteration captured in a CUDA graph.

It exists to show what the hand-written kernels buy over a competent
library implementation of the SAME algorithm: decimated
n-grid coherent fields, band-limited intensity / resist / adjoint spectra,
full-resolution sigmoid resist and mask update.  It is NOT on the product
path (bench.py reports it as `library_cufft`); torch.fft is cuFFT.

Semantics per iteration (oracle/litho_oracle.c orc_ilt_iteration, itself
the chain rule through imaging.cpp:218-241 / 287-323 and ai.cpp:11-42):
  M = sig(a theta);  for each focus stack f:
    I_f = dose sum_k w_fk |IFFT(M^ H_fk)|^2,  R_f = blur(I_f),
    Z_f = sig(beta (R_f - thr)),  cost += c_f sum (Z_f - Zt)^2,
    W_f = blur(2 c_f (Z_f - Zt) beta Z_f (1 - Z_f)),
    g_M += sum_k 2 dose w_fk Re IFFT(FFT(W_f E_fk) conj(H_fk) / N^2)
  theta -= step * g_M * a M (1 - M)
No kernel pairs and no mirror-stack merging (those are structural savings
of the hand-written path).
"""
from __future__ import annotations

import math

import numpy as np
import torch


def _gauss_hat(N, sigma_px):
    """DFT of the reference's truncated unit-sum Gaussian (imaging.cpp:292-305)."""
    if sigma_px <= 0:
        return np.ones(N)
    r = min(N // 2, int(math.ceil(6 * sigma_px)) + 1)
    d = np.arange(-r, r + 1)
    g = np.exp(-0.5 * d * d / (sigma_px * sigma_px))
    g /= g.sum()
    p = np.arange(N)
    return (g[None, :] * np.cos(2 * np.pi * p[:, None] * d[None, :] / N)).sum(1)


class CufftIlt:
    def __init__(self, kernels, params, n_sub=None, device="cuda"):
        """kernels: api.SocsKernelSet (F stacks x K, band-sparse support);
        params: api.IltParams."""
        ks = kernels
        g = ks.grid
        assert g.nx == g.ny, "square tiles"
        N = g.nx
        self.N = N
        dev = torch.device(device)
        sup = np.asarray(ks.support).reshape(-1, 2)
        kx = ((sup[:, 0] % N) + N) % N
        ky = ((sup[:, 1] % N) + N) % N
        kx = np.where(kx > N // 2, kx - N, kx)
        ky = np.where(ky > N // 2, ky - N, ky)
        lo, hi = int(min(kx.min(), ky.min())), int(max(kx.max(), ky.max()))
        B = hi - lo + 1
        P = B - 1  # intensity band |p| <= P
        n = n_sub or _sub_len(2 * P + 1)
        self.n, self.P, self.B, self.lo = n, P, B, lo
        F, K = ks.weights.shape
        self.F, self.K = F, K
        H = np.zeros((F, K, B, B), np.complex128)
        H[:, :, ky - lo, kx - lo] = ks.values
        self.H = torch.tensor(H, dtype=torch.complex64, device=dev)
        self.Hc = self.H.conj()
        self.w = torch.tensor(ks.weights, dtype=torch.float32, device=dev)
        q = np.arange(lo, hi + 1)
        self.qN = torch.tensor(q % N, device=dev)           # band index on the N grid
        self.qn = torch.tensor(q % n, device=dev)           # ... on the n grid
        p = np.arange(-P, P + 1)
        self.pN = torch.tensor(p % N, device=dev)
        self.pn = torch.tensor(p % n, device=dev)
        self.px = torch.arange(0, P + 1, device=dev)         # half-spectrum columns
        gh = _gauss_hat(N, params.resist_sigma_nm / g.pitch_nm)
        self.gy = torch.tensor(gh[p % N], dtype=torch.float32, device=dev)          # [2P+1]
        self.gx = torch.tensor(gh[np.arange(P + 1)], dtype=torch.float32, device=dev)  # [P+1]
        fw = params.focus_weights if params.focus_weights is not None else [1.0 / F] * F
        self.cf = torch.tensor(fw, dtype=torch.float32, device=dev).view(1, F, 1, 1)
        self.a = float(params.mask_steepness)
        self.beta = float(params.resist_beta)
        self.thr = float(params.threshold)
        self.dose = float(params.dose)
        self.step = float(params.step)
        self.dev = dev

    def iteration(self, theta, target):
        """theta [T,N,N] f32 (updated in place), target [T,N,N] f32 -> cost [T] f32."""
        N, n, P, F, K = self.N, self.n, self.P, self.F, self.K
        T = theta.shape[0]
        M = torch.sigmoid(self.a * theta)
        Mh = torch.fft.fft2(M) / (N * N)                                   # [T,N,N]
        Mb = Mh.index_select(1, self.qN).index_select(2, self.qN)           # [T,B,B]
        Zb = Mb[:, None, None] * self.H[None]                               # [T,F,K,B,B]
        Zn = torch.zeros((T, F, K, n, n), dtype=torch.complex64, device=self.dev)
        Zn[:, :, :, self.qn[:, None], self.qn[None, :]] = Zb
        E = torch.fft.ifft2(Zn) * (n * n)                                   # coherent fields, n grid
        I = self.dose * (self.w[None, :, :, None, None] * (E.real ** 2 + E.imag ** 2)).sum(2)  # [T,F,n,n]
        Ih = torch.fft.fft2(I) / (n * n)
        Rb = Ih[:, :, self.pn][:, :, :, self.px] * (self.gy[:, None] * self.gx[None, :])  # [T,F,2P+1,P+1]
        Rh = torch.zeros((T, F, N, N // 2 + 1), dtype=torch.complex64, device=self.dev)
        Rh[:, :, self.pN[:, None], self.px[None, :]] = Rb
        R = torch.fft.irfft2(Rh, s=(N, N)) * (N * N)                        # resist image, full res
        Z = torch.sigmoid(self.beta * (R - self.thr))
        e = Z - target[:, None]
        cost = (self.cf * e * e).sum((1, 2, 3))
        D = 2 * self.cf * e * self.beta * Z * (1 - Z)
        Dh = torch.fft.rfft2(D) / (N * N)
        Wb = Dh[:, :, self.pN][:, :, :, self.px] * (self.gy[:, None] * self.gx[None, :])
        Wh = torch.zeros((T, F, n, n // 2 + 1), dtype=torch.complex64, device=self.dev)
        Wh[:, :, self.pn[:, None], self.px[None, :]] = Wb
        Wn = torch.fft.irfft2(Wh, s=(n, n)) * (n * n)                       # band-limited W on the n grid
        U = torch.fft.fft2(Wn[:, :, None] * E) / (n * n)                    # [T,F,K,n,n]
        Ub = U[:, :, :, self.qn][:, :, :, :, self.qn]                       # [T,F,K,B,B]
        G = (2 * self.dose * self.w[None, :, :, None, None] * Ub * self.Hc[None]).sum((1, 2))  # [T,B,B]
        Gh = torch.zeros((T, N, N), dtype=torch.complex64, device=self.dev)
        Gh[:, self.qN[:, None], self.qN[None, :]] = G
        gM = torch.fft.ifft2(Gh).real * (N * N)
        theta -= self.step * gM * self.a * M * (1 - M)
        return cost


def _sub_len(m):
    """smallest 2^a 3^b >= m (cuFFT-friendly decimated grid, like the hand-written path)."""
    best = 1 << 30
    a = 1
    while a < 4 * m:
        b = a
        while b < 4 * m:
            if b >= m:
                best = min(best, b)
            b *= 3
        a *= 2
    return best


def timed(ilt, theta, target, iters, steps=3, warmup=1):
    """Graph-captured `iters` iterations per step; returns (ms per step, cost)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):  # warm plans / allocator before capture
            ilt.iteration(theta.clone(), target)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    th = theta.clone()
    with torch.cuda.graph(g):
        costs = [ilt.iteration(th, target) for _ in range(iters)]
    for _ in range(warmup):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, torch.stack(costs).cpu().numpy()
