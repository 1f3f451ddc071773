#!/usr/bin/env python
"""Profiling driver for ncu: one eager (non-graph) ILT iteration of a batch of
tiles at a bench config, bracketed by cudaProfilerStart/Stop so that
`ncu --profile-from-start off` sees only that iteration's launches.

  python tools/prof_c5.py [--config c5] [--tiles 32] [--iters 1]

Typical:
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
      --log-file gpurun_out/launches.csv python tools/prof_c5.py
  ncu --set full --import-source on --clock-control none --profile-from-start off \
      -k regex:fk_resist_rows -c 1 -o gpurun_out/resist python tools/prof_c5.py
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--tiles", type=int, default=32)
    ap.add_argument("--iters", type=int, default=1)
    a = ap.parse_args()
    import torch

    import bench
    import paper_2602_15036_b200 as L
    from paper_2602_15036_b200 import layouts as LY
    torch.cuda.set_device(0)
    ctx = L.Context(0)  # legacy stream: eager launches, no graph
    grid, polys, ks, iters, desc = bench.make_problem(a.config, 0, "gpu", ctx)
    dk = L.DeviceKernels(ks, "f32", ctx)
    xy, st = LY.polygon_arrays(polys)
    N = grid.nx
    tgt = torch.empty((N, N), dtype=torch.float64, device="cuda")
    bench._raster_to(ctx, grid, xy, st, tgt)
    t32 = tgt.float().expand(a.tiles, -1, -1).contiguous()
    F = ks.weights.shape[0]
    s = L.IltSolver(dk, L.IltParams(focus_weights=[1.0 / F] * F, **bench.ILT), a.tiles, "f32", ctx)
    cost = torch.zeros((a.iters, a.tiles), dtype=torch.float64, device="cuda")
    for _ in range(2):
        s.set_tiles(t32)
        s.run_device(a.iters, cost)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    s.run_device(a.iters, cost)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print(desc, dk.info(), float(cost[-1].sum()))


if __name__ == "__main__":
    main()
