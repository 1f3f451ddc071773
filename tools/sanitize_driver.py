#!/usr/bin/env python
"""Small end-to-end workload for compute-sanitizer (racecheck / synccheck /
memcheck): fp32 fast-path imaging + resist + weighted adjoint, a few ILT
iterations (eager launches, and a replayed CUDA graph), the generic-path
(odd grid) image, rasterization, marching squares and EPE gauges.

  compute-sanitizer --tool racecheck python tools/sanitize_driver.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2602_15036_b200 as L
    from paper_2602_15036_b200 import layouts as LY
    n = int(os.environ.get("SAN_N", "512"))
    model = L.OpticalModel(source=L.make_annular_source(0.4, 0.8, 21))
    grid = L.Grid(n, n, 1.0)
    ks = L.build_socs_kernels(model, grid, [-40.0, 0.0, 40.0], k_fixed=8)
    ctx = L.default_context(0)
    dk = L.DeviceKernels(ks, "f32", ctx)
    mask = L.rasterize_layer(LY.line_space_contacts(n, n, seed=1), grid, 1.0, ctx)
    out = dk.image(mask, sigma_nm=2.0, threshold=0.25, want=("intensity", "resist", "print"))
    W = np.random.default_rng(0).standard_normal((n, n))
    dk.gradient(mask, 1.0, weight=W, focus=2)
    prm = L.IltParams(focus_weights=[0.25, 0.5, 0.25])
    s = L.IltSolver(dk, prm, 2, "f32", ctx)
    s.set_tiles(np.stack([mask, mask[::-1]]))
    s.run(2)
    s.gradient()
    # graph path: a context on a non-default stream captures on the 2nd call
    st = torch.cuda.Stream()
    c2 = L.Context(0, st.cuda_stream)
    s2 = L.IltSolver(L.DeviceKernels(ks, "f32", c2), prm, 1, "f32", c2)
    s2.set_tiles(mask[None])
    for _ in range(3):
        s2.run(2)
    # generic runtime-length path (odd grid) and fp64
    g3 = L.Grid(74, 49, 4.0)
    k3 = L.build_socs_kernels(model, g3, [0.0], k_fixed=4)
    m3 = np.random.default_rng(1).random((49, 74))
    L.DeviceKernels(k3, "f64", ctx).image(m3, sigma_nm=2.0, want=("intensity", "resist"))
    # contours + EPE on the resist image
    r = np.asarray(out["resist"], np.float64)
    r[:2] = 0
    r[-2:] = 0
    r[:, :2] = 0
    r[:, -2:] = 0
    cs = L.marching_squares(r, grid, 0.25, ctx)
    rng = np.random.default_rng(3)
    ga = np.column_stack([rng.uniform(0, n, 256), rng.uniform(0, n, 256), np.ones(256), np.zeros(256)])
    L.measure_epe(cs, ga, 10.0)
    ctx.synchronize()
    print("sanitize driver ok", len(cs.loop_start) - 1)


if __name__ == "__main__":
    main()
