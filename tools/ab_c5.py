#!/usr/bin/env python
"""A/B timing of library variants on the C5 batch (32 tiles, graph-replayed
ILT iterations), in-graph, best of `reps`; each variant in a fresh process
(LITHOGPU_LIB).  Also checks the variant's per-iteration costs against the
first (baseline) variant.

  python tools/ab_c5.py [--iters 10] [--reps 5] [--tiles 32] name=path[,VAR=VAL...] ...
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys, torch
sys.path.insert(0, ".")
import bench
import paper_2602_15036_b200 as L
from paper_2602_15036_b200 import layouts as LY
cfg, iters, reps, tiles = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
torch.cuda.set_device(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
ctx = L.Context(0); ctx.set_stream(st.cuda_stream)
grid, polys, ks, _, _ = bench.make_problem(cfg, 0, "gpu", ctx)
dk = L.DeviceKernels(ks, "f32", ctx)
xy, starts = LY.polygon_arrays(polys)
N = grid.nx
tgt = torch.empty((N, N), dtype=torch.float64, device="cuda")
bench._raster_to(ctx, grid, xy, starts, tgt)
t32 = tgt.float().expand(tiles, -1, -1).contiguous()
F = ks.weights.shape[0]
prm = L.IltParams(focus_weights=[1.0 / F] * F, **bench.ILT)
sol = L.IltSolver(dk, prm, tiles, "f32", ctx)
cost = torch.zeros((iters, tiles), dtype=torch.float64, device="cuda")
for _ in range(3):
    sol.set_tiles(t32); sol.run_device(iters, cost)
torch.cuda.synchronize()
best = 1e30
for _ in range(reps):
    sol.set_tiles(t32)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st); sol.run_device(iters, cost); e1.record(st); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / iters)
print(json.dumps({"ms_per_iter": best, "tile_iter_s": tiles / (best * 1e-3), "cost": cost[:, 0].tolist()}))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--tiles", type=int, default=32)
    ap.add_argument("--config", default="c5")
    ap.add_argument("variants", nargs="+")
    a = ap.parse_args()
    out = {}
    base = None
    for v in a.variants:
        name, path = v.split("=", 1)
        env = dict(os.environ)
        # name=path[,VAR=VAL...]: extra environment for the variant
        path, *kv = path.split(",")
        for x in kv:
            k, val = x.split("=", 1)
            env[k] = val
        if path != "default":
            env["LITHOGPU_LIB"] = os.path.abspath(path)
        r = subprocess.run([sys.executable, "-c", CHILD, a.config, str(a.iters), str(a.reps), str(a.tiles)],
                           env=env, cwd=ROOT, capture_output=True, text=True)
        if r.returncode != 0:
            out[name] = {"error": r.stderr[-1500:]}
            continue
        d = json.loads(r.stdout.strip().splitlines()[-1])
        if base is None:
            base = d["cost"]
        d["cost_rel_diff_vs_first"] = max(abs(x - y) / abs(y) for x, y in zip(d["cost"], base))
        del d["cost"]
        out[name] = d
        print(name, json.dumps(d), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
