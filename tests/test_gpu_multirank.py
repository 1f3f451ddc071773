"""The N>1 path executed on one GPU: two ranks (gloo, one process each,
both on cuda:0) run the real chip.ChipIlt over their contiguous shards of a
seeded chip.  The all-reduced per-iteration global cost
equals the sum of single-process one-tile runs; the max |dL/dtheta| is the
max over tiles; the relative-tolerance stop fires on the same segment on
both ranks.  Plus `torchrun --nproc-per-node 2 bench.py` on one GPU (gloo)
to shake out the bench's N>1 launch path.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import paper_2602_15036_b200 as L
from paper_2602_15036_b200 import chip, layouts as LY

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ITERS = 6


def _problem():
    tl = LY.chip_tiling(256, 3, 1, 64)
    polys = LY.chip_layout(tl, seed=31)
    model = L.OpticalModel(source=L.make_annular_source(0.4, 0.8, 21))
    ks = L.build_socs_kernels(model, L.Grid(tl.n, tl.n, 1.0), [-40.0, 0.0, 40.0], k_fixed=8)
    prm = L.IltParams(step=0.5, focus_weights=[0.25, 0.5, 0.25])
    return tl, polys, ks, prm


def _worker(rank, world, port, q, tol):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    ctx = L.Context(0)
    ctx.set_stream(st.cuda_stream)
    tl, polys, ks, prm = _problem()
    ci = chip.ChipIlt(tl, polys, ks, prm, ctx, rank=rank, world=world)
    res = ci.run(ITERS, sync_every=2)
    ci2 = chip.ChipIlt(tl, polys, ks, prm, ctx, rank=rank, world=world)
    res_tol = ci2.run(ITERS, sync_every=2, tol=tol)
    q.put((rank, list(res.tiles), res.cost.tolist(), res.gmax.tolist(), len(res_tol.cost)))
    dist.destroy_process_group()


def test_two_ranks_real_chip_ilt_gloo(ctx):
    import torch.multiprocessing as mp
    tl, polys, ks, prm = _problem()
    # single-process reference: every tile on its own
    costs, gmaxs = [], []
    for t in range(len(tl)):
        g = tl.tile_grid(t)
        raster = L.rasterize_layer(tl.tile_polygons(polys, t), g, 1.0, ctx)
        s = L.IltSolver(ks, prm, 1, "f32", ctx)
        s.set_tiles(raster[None].astype(np.float32))
        c, gm = s.run(ITERS, with_gmax=True)
        costs.append(c[:, 0])
        gmaxs.append(gm[:, 0])
        s.close()
    want_cost = np.sum(costs, axis=0)
    want_gmax = np.max(gmaxs, axis=0)
    rel_change = np.abs(np.diff(want_cost)) / np.abs(want_cost[:-1])
    tol = float(rel_change[2]) * 1.0001  # checked after the 2nd segment: fires at iteration 2 or 4
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    procs = [mctx.Process(target=_worker, args=(r, 2, port, q, tol)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    assert res[0][1] + res[1][1] == list(range(len(tl)))  # contiguous shards cover the chip
    for r in res:
        assert np.abs(np.array(r[2]) - want_cost).max() <= 1e-9 * np.abs(want_cost).max()
        assert np.array_equal(np.array(r[3]), want_gmax)
    # the stop fires after the first segment (of 2 iterations) whose last relative change <= tol
    done = None
    for k in range(2, ITERS + 1, 2):
        if rel_change[k - 2] <= tol:
            done = k
            break
    assert done is not None and done < ITERS
    assert res[0][4] == res[1][4] == done


def test_torchrun_bench_two_ranks_one_gpu():
    """bench.py's N>1 path (sharding, per-step all-reduce, max-over-ranks
    timing, rank-0 JSON line) with two ranks on one GPU over gloo."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--steps", "1",
           "--warmup", "1", "--dist-backend", "gloo", "--no-cpu-baseline", "--no-secondary"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["tiles_per_rank"] == 128 and d["value"] > 0
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
