#!/usr/bin/env python
"""Launch timeline of the graph-replayed C2 ILT loop (LITHOGPU_TRACE).

Each fast kernel records its first-CTA start and last-warp end
(%globaltimer) per launch; this prints, for the last replay of `iters`
iterations, every launch's duration and the gap before it.

  python tools/trace.py [--iters 4] [--config c2|c5 ...] [--tiles T]
"""
import json
import os
import subprocess
import sys
import tempfile

CHILD = r'''
import sys, torch
sys.path.insert(0, ".")
import bench
import paper_2602_15036_b200 as L
from paper_2602_15036_b200 import layouts as LY
iters = int(sys.argv[1])
tiles = int(sys.argv[3]) if len(sys.argv) > 3 else 1
torch.cuda.set_device(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
ctx = L.Context(0); ctx.set_stream(st.cuda_stream)
grid, polys, ks, _, _ = bench.make_problem(sys.argv[2], 0)
dk = L.DeviceKernels(ks, "f32", ctx)
xy, starts = LY.polygon_arrays(polys)
N = grid.nx
tgt = torch.empty((1, N, N), dtype=torch.float64, device="cuda")
bench._raster_to(ctx, grid, xy, starts, tgt)
t32 = tgt.float().expand(tiles, -1, -1).contiguous()
th = ((2 * t32 - 1) * 0.5).contiguous()
F = ks.weights.shape[0]
prm = L.IltParams(focus_weights=[1.0 / F] * F, **bench.ILT)
sol = L.IltSolver(dk, prm, tiles, "f32", ctx)
cost = torch.zeros((iters, tiles), dtype=torch.float64, device="cuda")
for _ in range(4):
    sol.set_tiles(t32, th); sol.run_device(iters, cost)
torch.cuda.synchronize()
'''


def main():
    iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 4
    cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "c2"
    tiles = sys.argv[sys.argv.index("--tiles") + 1] if "--tiles" in sys.argv else "1"
    fd, path = tempfile.mkstemp(suffix=".jsonl")
    os.close(fd)
    env = dict(os.environ, LITHOGPU_TRACE=path)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", CHILD, str(iters), cfg, tiles], env=env, cwd=root, capture_output=True,
                       text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stderr[-3000:])
        sys.exit(1)
    recs = [json.loads(x) for x in open(path)]
    os.unlink(path)
    last = []  # the final call's records: slots restart at 0 per call
    for rec in recs:
        if rec["slot"] == 0:
            last = []
        last.append(rec)
    t0 = last[0]["start_ns"]
    prev_end = None
    rows = []
    for rec in last:
        gap = (rec["start_ns"] - prev_end) / 1e3 if prev_end is not None else 0.0
        dur = (rec["end_ns"] - rec["start_ns"]) / 1e3
        rows.append({"name": rec["name"], "start_us": round((rec["start_ns"] - t0) / 1e3, 2),
                     "dur_us": round(dur, 2), "gap_us": round(gap, 2), "ctas": rec["ctas"]})
        prev_end = rec["end_ns"]
    total = (last[-1]["end_ns"] - t0) / 1e3
    per = {}
    for x in rows[len(rows) // iters:]:  # skip the first iteration
        d = per.setdefault(x["name"], [0.0, 0.0, 0])
        d[0] += x["dur_us"]
        d[1] += x["gap_us"]
        d[2] += 1
    summary = {k: {"dur_us": round(v[0] / v[2], 2), "gap_before_us": round(v[1] / v[2], 2)} for k, v in per.items()}
    print(json.dumps({"iters": iters, "span_us": round(total, 2), "per_iter_us": round(total / iters, 2),
                      "per_kernel": summary, "timeline": rows}))


if __name__ == "__main__":
    main()
