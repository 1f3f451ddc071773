#!/usr/bin/env python
"""In-graph marginal cost of each ILT kernel (timing ablation).

For every kernel name of the fast ILT loop, re-run the C2 step with that
launch removed from the graph (LITHOGPU_ABLATE, read once per process, so
each variant runs in a fresh subprocess) and report the drop in ms per
iteration.  The data flow is broken in the ablated runs; only the timing is
meaningful (FFT timing does not depend on the values).

  python tools/ablate.py [--iters 50] [--reps 5]
"""
import json
import os
import subprocess
import sys

NAMES = ["mask_cols", "socs_cols", "socs_rows", "isub_cols", "resist_rows", "wlp_cols",
         "wlp_rows", "adj_rows", "adj_cols", "grad_cols", "grad_rows"]

CHILD = r'''
import json, sys, torch
sys.path.insert(0, ".")
import bench
import paper_2602_15036_b200 as L
iters, reps = int(sys.argv[1]), int(sys.argv[2])
torch.cuda.set_device(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
ctx = L.Context(0); ctx.set_stream(st.cuda_stream)
grid, polys, ks, _, _ = bench.make_problem("c2", 0)
dk = L.DeviceKernels(ks, "f32", ctx)
from paper_2602_15036_b200 import layouts as LY
xy, starts = LY.polygon_arrays(polys)
N = grid.nx
tgt = torch.empty((1, N, N), dtype=torch.float64, device="cuda")
bench._raster_to(ctx, grid, xy, starts, tgt)
t32 = tgt.float()
th = ((2 * t32 - 1) * 0.5).contiguous()
prm = L.IltParams(focus_weights=[1.0], **bench.ILT)
sol = L.IltSolver(dk, prm, 1, "f32", ctx)
cost = torch.zeros((iters, 1), dtype=torch.float64, device="cuda")
for _ in range(3):
    sol.set_tiles(t32, th); sol.run_device(iters, cost)
torch.cuda.synchronize()
best = 1e30
for _ in range(reps):
    sol.set_tiles(t32, th)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st); sol.run_device(iters, cost); e1.record(st); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / iters)
print(json.dumps({"ms_per_iter": best}))
'''


def run(ablate, iters, reps):
    env = dict(os.environ)
    if ablate:
        env["LITHOGPU_ABLATE"] = ablate
    r = subprocess.run([sys.executable, "-c", CHILD, str(iters), str(reps)], env=env, capture_output=True,
                       text=True, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    if r.returncode != 0:
        raise RuntimeError(r.stderr[-2000:])
    return json.loads(r.stdout.strip().splitlines()[-1])["ms_per_iter"]


def main():
    iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 50
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 5
    base = run(None, iters, reps)
    if "--base" in sys.argv:
        print(json.dumps({"ms_per_iter": base}))
        return
    out = {"ms_per_iter": base, "marginal_us": {}}
    for n in NAMES:
        out["marginal_us"][n] = round((base - run(n, iters, reps)) * 1e3, 2)
    out["all_but_sum_us"] = round(base * 1e3 - sum(out["marginal_us"].values()), 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
