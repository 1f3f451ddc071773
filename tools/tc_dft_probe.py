#!/usr/bin/env python
"""Evidence for the tensor-core question: the decimated-grid
row transforms of fk_socs_rows (C5 launch: 36 kernel slots x 384 rows x 32
tiles = 442 368 rows of length n = 384, band B = 179 nonzero inputs) written
as DFT-as-GEMM on the tensor cores (cuBLAS, the tensor-core peak proxy), in
bf16, tf32 and 3xTF32 (hi/lo split, fp32-class accuracy), against the same
transforms on cuFFT in fp32.  Reports time and the rel L-inf error against an
fp64 reference on a sample.

  python tools/tc_dft_probe.py [--rows 442368] [--out gpurun_out/tc_dft_probe.json]
"""
import argparse
import json
import os

import numpy as np
import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=442368)
    ap.add_argument("--n", type=int, default=384)
    ap.add_argument("--band", type=int, default=179)
    ap.add_argument("--out", default="gpurun_out/tc_dft_probe.json")
    a = ap.parse_args()
    n, B, R = a.n, a.band, a.rows
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    # band-limited rows: B nonzero inputs at q in [-(B-1)/2, (B-1)/2] (mod n)
    q = torch.arange(-(B // 2), B // 2 + 1, device=dev) % n
    xb = torch.randn((R, B), generator=g, device=dev, dtype=torch.float32) + \
        1j * torch.randn((R, B), generator=g, device=dev, dtype=torch.float32)
    xb = xb.to(torch.complex64)
    # inverse DFT rows restricted to the band: Y = Xb @ Wb, Wb[j, x] = exp(+2 pi i q_j x / n)
    xs = torch.arange(n, device=dev, dtype=torch.float64)
    Wb = torch.exp(2j * np.pi * q.double()[:, None] * xs[None, :] / n)  # [B, n] complex128
    # real block form: [Xr Xi] @ [[Wr, Wi], [-Wi, Wr]]  ->  [Yr Yi]
    Wr, Wi = Wb.real, Wb.imag
    Wreal = torch.cat([torch.cat([Wr, Wi], 1), torch.cat([-Wi, Wr], 1)], 0)  # [2B, 2n]
    Xreal = torch.cat([xb.real, xb.imag], 1)  # [R, 2B] fp32
    # fp64 reference on a sample
    S = 2048
    ref = (xb[:S].to(torch.complex128) @ Wb)
    ref_real = torch.cat([ref.real, ref.imag], 1)

    def timeit(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            out = fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps, out

    def err(y):
        y = y[:S].double()
        return float((y - ref_real).abs().max() / ref_real.abs().max())

    res = {"rows": R, "n": n, "band": B, "note": "DFT-as-GEMM on cuBLAS (tensor cores) vs cuFFT, same transforms"}
    # cuFFT fp32: scatter band into n-point rows, ifft (unnormalised)
    def cufft():
        z = torch.zeros((R, n), dtype=torch.complex64, device=dev)
        z[:, q] = xb
        return torch.fft.ifft(z) * n
    ms, y = timeit(cufft)
    yr = torch.cat([y.real, y.imag], 1)
    res["cufft_fp32"] = {"ms": ms, "rel_linf": err(yr), "gflop_fft": R * 5 * n * np.log2(n) / 1e9}
    gemm_flop = 2.0 * R * (2 * B) * (2 * n)
    # bf16
    Xb16, Wb16 = Xreal.bfloat16(), Wreal.float().bfloat16()
    ms, y = timeit(lambda: Xb16 @ Wb16)
    res["gemm_bf16"] = {"ms": ms, "rel_linf": err(y.float()), "tflops": gemm_flop / ms / 1e9}
    # tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    Wf = Wreal.float()
    ms, y = timeit(lambda: Xreal @ Wf)
    res["gemm_tf32"] = {"ms": ms, "rel_linf": err(y), "tflops": gemm_flop / ms / 1e9}
    # 3xTF32: (Xh + Xl)(Wh + Wl) ~ Xh Wh + Xh Wl + Xl Wh
    def split(t):
        h = t.view(torch.int32).bitwise_and(-8192).view(torch.float32)  # keep 10 mantissa bits (tf32)
        return h, t - h
    Xh, Xl = split(Xreal.contiguous())
    Wh, Wl = split(Wf.contiguous())
    ms, y = timeit(lambda: Xh @ Wh + (Xh @ Wl + Xl @ Wh))
    res["gemm_3xtf32"] = {"ms": ms, "rel_linf": err(y), "tflops": 3 * gemm_flop / ms / 1e9}
    torch.backends.cuda.matmul.allow_tf32 = False
    ms, y = timeit(lambda: Xreal @ Wf)
    res["gemm_fp32_simt"] = {"ms": ms, "rel_linf": err(y), "tflops": gemm_flop / ms / 1e9}
    print(json.dumps(res, indent=1))
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
