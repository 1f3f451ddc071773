#!/usr/bin/env python
"""Hand-written ILT vs the cuFFT library implementation of the same
algorithm (tools/cufft_ilt.py): agreement of one iteration (cost and theta
update, rel L-inf) and device time per tile-iteration at C2 and C5.

  python tools/cufft_check.py [--out gpurun_out/cufft_check.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import bench as B  # noqa: E402
import paper_2602_15036_b200 as L  # noqa: E402
from cufft_ilt import CufftIlt, timed  # noqa: E402
from paper_2602_15036_b200._lib import F32  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def case(name, tiles, iters, ctx):
    grid, polys, ks, _, _ = B.make_problem(name, 0, kernels="gpu", ctx=ctx)
    N = grid.nx
    tgt = L.rasterize_layer(polys, grid, 1.0, ctx)
    tgt = np.ascontiguousarray(np.broadcast_to(tgt, (tiles, N, N)), np.float32)
    rng = np.random.default_rng(7)
    th0 = (2.0 * tgt - 1.0 + 0.05 * rng.standard_normal(tgt.shape)).astype(np.float32)
    prm = L.IltParams(**B.ILT, focus_weights=[1.0 / len(ks.focus_nm)] * len(ks.focus_nm))
    # ours: one iteration
    sol = L.IltSolver(ks, prm, tiles, "f32", ctx)
    sol.set_tiles(tgt, th0)
    c_ours = sol.run(1)[0]
    th_ours = sol.get_tiles(dtype=F32)[0]
    # cuFFT library path: one iteration
    lib = CufftIlt(ks, prm)
    th = torch.tensor(th0, device="cuda")
    tg = torch.tensor(tgt, device="cuda")
    c_lib = lib.iteration(th, tg).double().cpu().numpy()
    th_lib = th.cpu().numpy()
    d_ours = th_ours.astype(np.float64) - th0
    d_lib = th_lib.astype(np.float64) - th0
    out = {"config": name, "tiles": tiles, "N": N, "n_sub": lib.n, "K": ks.weights.shape[1],
           "F": ks.weights.shape[0],
           "cost_rel": rel(c_ours, c_lib), "update_rel_linf": rel(d_ours, d_lib)}
    # timing: `iters` graph-replayed iterations per step, both device-resident
    ms_lib, _ = timed(lib, th, tg, iters, steps=3, warmup=1)
    st = torch.cuda.Stream()
    ctx.set_stream(st.cuda_stream)
    with torch.cuda.stream(st):
        for _ in range(2):
            sol.run_device(iters)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(3):
            sol.run_device(iters)
        e1.record(st)
    torch.cuda.synchronize()
    ctx.set_stream(0)
    ms_ours = e0.elapsed_time(e1) / 3
    out.update({"iters_per_step": iters,
                "ours_tile_iter_s": tiles * iters / (ms_ours / 1e3),
                "cufft_tile_iter_s": tiles * iters / (ms_lib / 1e3),
                "speedup": ms_lib / ms_ours})
    sol.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/cufft_check.json")
    a = ap.parse_args()
    ctx = L.default_context(0)
    res = [case("c2", 1, 20, ctx), case("c5", 32, 5, ctx)]
    for r in res:
        print(json.dumps(r))
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
