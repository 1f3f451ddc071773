#!/usr/bin/env python
"""Benchmark of the B200-native SOCS imaging / ILT hot path.

Headline workload (BASELINE.json configs[4], "C5", the configuration the
metric's "ILT iter/s per tile (1/2/4/8 B200)" is quoted on): ONE seeded
synthetic chip layout cut by `layouts.chip_tiling` into 16 x 16 = 256
halo-padded 2048^2 tiles (core 1792 + 2 x 128 px halo, the optical ambit +
resist-blur guard of `layouts.optical_halo_px`), K = 24 SOCS kernels,
3 focus planes, 50 ILT iterations.  Tiles are sharded over ranks
(`chip.shard`, contiguous blocks) and run in launch batches of 64 tiles
(blockIdx.z = tile, one CUDA graph per batch); the only collective is the
all-reduce of the per-iteration global ILT cost.  One step = all 256 tiles x
50 iterations.  Metric: ILT tile-iterations/s, whole job.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c5|c1|c2|c3|c4]
  torchrun --nproc-per-node N bench.py --gpus N ...

`value` is device-timed (CUDA events on the launch stream, inputs resident
in HBM, working set >> L2, max over ranks).  `e2e` is the same job through
the C ABI from host memory: per tile the polygon arrays (pinned host) ->
GPU rasterization -> ILT -> the tile's core written straight into the
stitched chip mask in pinned host memory (lithogpu_ilt_get_window).
`--impl reference` times the reference's own CPU implementation
(oracle/_ref: the unmodified reference sources, all host threads) on one
tile-iteration of the same chip per step; it never loads liblithogpu.so
(kernels from oracle/kernels_np.py, raster from the reference rasterizer).
Secondary lines (world 1): C2 single tile (value + e2e) and C1 forward
Mpixel/s with its CPU reference.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import re
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (tile N, K, foci, iterations per step, description)
    "c1": (1024, 8, [0.0], 0, "C1: single 1024x1024 tile forward aerial image + threshold resist, K=8, F=1"),
    "c2": (2048, 16, [0.0], 50, "C2: 2048x2048 tile ILT, K=16, F=1, 50 iterations, Gaussian-blur resist"),
    "c3": (2048, 16, [-40.0, -20.0, 0.0, 20.0, 40.0], 50, "C3: through-focus ILT 2048x2048, K=16, F=5"),
    "c4": (4096, 32, [-40.0, 0.0, 40.0], 50, "C4: curvilinear ILT 4096x4096, K=32, F=3"),
    "c5": (2048, 24, [-40.0, 0.0, 40.0], 50,
           "C5: chip-scale 256 halo-padded 2048x2048 tiles (one seeded chip, 16x16 tiles of 1792 core + "
           "2x128 halo), K=24, F=3, 50 ILT iterations, sharded over ranks"),
}
C5_TX = C5_TY = 16
C5_BATCH = 64
C5_SEED = 2602
ILT = dict(mask_steepness=4.0, resist_beta=30.0, threshold=0.25, resist_sigma_nm=2.0, dose=1.0, step=0.5)
OPTICS = dict(wavelength_nm=13.5, na=0.33, sigma_in=0.4, sigma_out=0.8, grid_n=21)
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: exercise the N>1 launch path on one GPU (tests)")
    return ap.parse_args()


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def c5_tiling():
    """The C5 chip: 16 x 16 tiles of 2048 px = 1792 core + 2 x halo (128 px)."""
    from paper_2602_15036_b200 import layouts as LY
    halo = LY.optical_halo_px(OPTICS["wavelength_nm"], OPTICS["na"], 1.0, ILT["resist_sigma_nm"])
    return LY.chip_tiling(CONFIGS["c5"][0], C5_TX, C5_TY, halo)


def make_problem(cfg_name, rank, kernels="host", ctx=None):
    """(grid, polygons, kernel stacks, iterations, description) of a one-tile
    config.  kernels: "host" / "gpu" (the product generators) or "oracle"
    (oracle/kernels_np.py: the reference arm never loads liblithogpu.so)."""
    from paper_2602_15036_b200 import layouts as LY
    from paper_2602_15036_b200.api import Grid, SocsKernelSet
    N, K, foci, iters, desc = CONFIGS[cfg_name]
    grid = Grid(N, N, 1.0, 0.0, 0.0)
    gen = LY.curvilinear if cfg_name == "c4" else LY.line_space_contacts
    polys = gen(N, N, seed=1000 + rank)
    return grid, polys, kernel_stacks(grid, foci, K, kernels, ctx), iters, desc


def kernel_stacks(grid, foci, K, kernels="host", ctx=None):
    from paper_2602_15036_b200.api import SocsKernelSet
    if kernels == "oracle":
        from oracle import kernels_np as KN
        W, sup, V = KN.socs_kernel_stacks(grid.nx, grid.pitch_nm, foci, K, OPTICS["sigma_in"], OPTICS["sigma_out"],
                                          OPTICS["grid_n"], OPTICS["wavelength_nm"], OPTICS["na"])
        return SocsKernelSet(grid, list(foci), W, sup, V)
    import paper_2602_15036_b200 as L
    model = L.OpticalModel(wavelength_nm=OPTICS["wavelength_nm"], na=OPTICS["na"],
                           source=L.make_annular_source(OPTICS["sigma_in"], OPTICS["sigma_out"], OPTICS["grid_n"]))
    return L.build_socs_kernels(model, grid, foci, k_fixed=K, backend=kernels, ctx=ctx)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7:
                rows.append(f)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = max(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        load = [v for v in sm if v > 0.5 * mx] or sm
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# algorithmic model (implemented decimated-band algorithm)
# ---------------------------------------------------------------------------
def fft_flops(L):
    return 5.0 * L * math.log2(L)


def store_e(geo, F, K, tiles=1):
    """Mirror of Plan::reserve: the ILT keeps E_fk for the adjoint rows while
    F*K*n^2 complex64 per launch stays <= 8 GiB (LITHOGPU_STORE_E overrides)."""
    env = os.environ.get("LITHOGPU_STORE_E")
    if env is not None:
        return env.startswith("1")
    return 8 * F * K * geo["n"] ** 2 * tiles <= (8 << 30)


def kernel_model(geo, F, K, tiles=1):
    """Per-TILE FFT flops (5 L log2 L per length-L complex transform) and
    algorithmic bytes of each kernel of one ILT iteration, for the
    implemented decimated-band algorithm.  A launch over a
    batch of T tiles does T times this."""
    N, n, B = geo["N"], geo["n"], geo["B"]
    P, Pm = B - 1, (B - 1) // 2
    c = 8  # complex64 bytes
    fN, fn = fft_flops(N), fft_flops(n)
    se = store_e(geo, F, K, tiles)
    m = {
        "mask_cols": ((Pm + 1) * fN, (Pm + 1) * N * c + B * B * c),
        "socs_cols": (F * K * B * fn, F * K * (B * B * c + n * B * c)),
        "socs_rows": (F * (K + 1) * n * fn, F * K * (n * B * c + (n * n * c if se else 0)) + F * (P + 1) * n * c),
        "isub_cols": (F * (P + 1) * (fn + fN), F * ((P + 1) * n * c + N * (P + 1) * c)),
        "resist_rows": (F * (N // 2) * 2 * fN, F * (2 * N * (P + 1) * c + N * N * 4)),
        "wlp_cols": (F * (P + 1) * (fN + fn), F * ((P + 1) * N * c + n * (P + 1) * c)),
        "wlp_rows": (F * (n // 2) * fn, F * (n * (P + 1) * c + n * n * 4)),
        "adj_rows": (F * K * n * (1 if se else 2) * fn,
                     F * K * ((n * n * c) if se else (n * B * c)) + F * K * B * n * c + F * n * n * 4),
        "adj_cols": (F * K * B * fn, F * K * (B * n * c + 2 * B * B * c)),
        "grad_cols": ((Pm + 1) * fN, F * K * B * B * c + N * (Pm + 1) * c),
        "grad_rows": ((N // 2) * 2 * fN, N * (Pm + 1) * c + 2 * N * N * 4 + (Pm + 1) * N * c),
    }
    return m


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
class Dist:
    """torch.distributed plumbing (NCCL on GPUs; gloo for the one-GPU N>1 test)."""

    def __init__(self, world, local, backend):
        import torch
        self.world = world
        self.local = local
        self.backend = backend
        self.dev = torch.device("cuda", local)
        if world > 1:
            import torch.distributed as dist
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group("gloo")

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            if self.backend == "nccl":
                dist.barrier(device_ids=[self.local])
            else:
                dist.barrier()

    def allreduce(self, t, op="sum"):
        if self.world == 1:
            return t
        import torch.distributed as dist
        o = dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX
        if self.backend == "nccl":
            dist.all_reduce(t, op=o)
            return t
        h = t.cpu()
        dist.all_reduce(h, op=o)
        t.copy_(h)
        return t

    def max_scalar(self, v):
        import torch
        t = torch.tensor([v], dtype=torch.float64, device=self.dev)
        return float(self.allreduce(t, "max").item())

    def close(self):
        if self.world > 1:
            import torch.distributed as dist
            self.barrier()
            dist.destroy_process_group()


def timed_steps(step, steps, stream, D, flush=None):
    """CUDA-event time of each of `steps` calls of step(), barrier + sync on
    both sides; returns (per-step ms list, summed ms max over ranks)."""
    import torch
    times = []
    for _ in range(steps):
        if flush is not None:
            flush.fill_(1.0)  # L2 flush between steps (not timed)
        D.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    return times, D.max_scalar(float(np.sum(times)))


def run_chip(args, world, rank, local):
    """C5 headline (see module docstring)."""
    import torch
    import paper_2602_15036_b200 as L
    from paper_2602_15036_b200 import chip, layouts as LY
    local = local % max(1, torch.cuda.device_count())  # several ranks may share one GPU (gloo test path)
    torch.cuda.set_device(local)
    D = Dist(world, local, args.dist_backend)
    dev = D.dev
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx = L.Context(local)
    ctx.set_stream(stream.cuda_stream)

    N, K, foci, iters, desc = CONFIGS["c5"]
    F = len(foci)
    tl = c5_tiling()
    T = len(tl)
    t_setup = time.perf_counter()
    polys = LY.chip_layout(tl, seed=C5_SEED)
    bb = LY.polygon_bboxes(polys)
    grid = L.Grid(N, N, 1.0)
    ks = kernel_stacks(grid, foci, K, "gpu", ctx)
    dk = L.DeviceKernels(ks, "f32", ctx)
    info = dk.info()
    mine = list(chip.shard(T, world, rank))
    tile_polys = [LY.polygon_arrays(tl.tile_polygons(polys, t, bboxes=bb)) for t in mine]
    # device-resident inputs for `value`: the tiles' target rasters (GPU rasterizer)
    targets = torch.empty((len(mine), N, N), dtype=torch.float32, device=dev)
    tmp = torch.empty((N, N), dtype=torch.float64, device=dev)
    for j, t in enumerate(mine):
        xy, st = tile_polys[j]
        _raster_to(ctx, tl.tile_grid(t), xy, st, tmp)
        targets[j].copy_(tmp)
    del tmp
    prm = L.IltParams(focus_weights=[1.0 / F] * F, **ILT)
    batches = [(b0, min(b0 + C5_BATCH, len(mine))) for b0 in range(0, len(mine), C5_BATCH)]
    solvers, costs = {}, {}
    for b0, b1 in batches:
        nt = b1 - b0
        if nt not in solvers:
            solvers[nt] = L.IltSolver(dk, prm, nt, "f32", ctx)
            costs[nt] = torch.zeros((iters, nt), dtype=torch.float64, device=dev)
    gcost = torch.zeros(iters, dtype=torch.float64, device=dev)
    setup_s = time.perf_counter() - t_setup

    def step():
        gcost.zero_()
        for b0, b1 in batches:
            s = solvers[b1 - b0]
            s.set_tiles(targets[b0:b1])        # theta0 = (2 target - 1) 2/a on the device
            s.run_device(iters, costs[b1 - b0])  # one CUDA graph: all iterations of the batch
            gcost.add_(costs[b1 - b0].sum(dim=1))
        D.allreduce(gcost)  # global cost per iteration: the only cross-GPU traffic

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    l0 = ctx.launch_count()
    times, total_ms = timed_steps(step, args.steps, stream, D)
    launches = ctx.launch_count() - l0
    clk = clocks.stop()
    ms = total_ms / args.steps
    value = T * iters / (ms / 1e3)
    final_cost = gcost.cpu().numpy()

    # ---- per-kernel CUDA-event profile of one full batch (separate, eager) ----
    roof = None
    prof = None
    if rank == 0:
        b0, b1 = batches[0]
        s = solvers[b1 - b0]
        ctx.set_profiling(True)
        ctx.profile_report(reset=True)
        s.set_tiles(targets[b0:b1])
        s.run_device(iters, costs[b1 - b0])
        torch.cuda.synchronize()
        prof = ctx.profile_report(reset=True)
        ctx.set_profiling(False)
        roof = _roofline(ctx, info, N, F, K, b1 - b0, prof, iters, "c5")

    # ---- end to end through the C ABI from host memory ----
    e2e = None
    if not args.no_e2e:
        e2e = _chip_e2e(args, ctx, tl, mine, tile_polys, batches, solvers, costs, iters, D, stream, dev, ks, prm,
                        local)

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = _cpu_baseline("c5")
        secondary = None
        if not args.no_secondary and world == 1:
            secondary = {"c2": run_tile(args, 1, 0, local, "c2", ctx=ctx, stream=stream, D=D, quiet=True,
                                        steps=min(args.steps, 10)),
                         "c1": _c1_forward(ctx, stream, cpu=not args.no_cpu_baseline),
                         "library_cufft": _library_cufft(ks, prm, targets[:C5_BATCH], value)}
        res = {
            "metric": f"ILT tile-iterations/s ({desc})",
            "value": value,
            "unit": "tile-iter/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic: one seeded line/space+contact chip layout (layouts.chip_layout, seed "
                    f"{C5_SEED}, {len(polys)} polygons), GPU-rasterized per tile; GPU Abbe-SVD SOCS kernels",
            "config": {"workload": desc, "tiles_total": T, "tiles_per_rank": len(mine), "tiles_per_launch": C5_BATCH,
                       "tile": N, "core": tl.core, "halo": tl.halo, "chip_px": [tl.chip.nx, tl.chip.ny],
                       "K": K, "F": F, "iterations_per_step": iters,
                       "decimated_grid": info["nx_sub"], "kernel_band": info["band_x"],
                       "computed_focus_stacks": info.get("fast_stacks"),
                       "kernel_transforms_per_stack": info.get("fast_order"), "ilt": ILT,
                       "l2": f"inputs and per-batch working set ({C5_BATCH} tiles, GBs) far above the 126 MB L2",
                       "parallelism": f"{T} tiles sharded over {world} rank(s) (contiguous blocks); one all-reduce "
                                      "of the per-iteration global cost per step; no tile data crosses GPUs",
                       "scaling_note": "total work fixed (256 tiles): every rank runs the same batched "
                                       "launches on its shard",
                       "setup_s": round(setup_s, 2)},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
            "final_cost": [float(final_cost[0]), float(final_cost[-1])],
            "secondary": secondary,
        }
        if world == 1 and roof is not None:
            res["in_graph"] = _in_graph_timeline("c5", roof["kernel"], roof["flops_per_launch"], roof["peak"],
                                                 tiles=roof["tiles_per_launch"])
        print(json.dumps(res), flush=True)
    D.close()


def _library_cufft(ks, prm, targets, ours_value, iters=3):
    """The same decimated band-limited ILT iteration on cuFFT (tools/cufft_ilt.py:
    torch.fft, batched plans over the launch batch, fields in HBM, CUDA graph),
    on the C5 launch batch: what the hand-written kernels buy over a library
    implementation of the same algorithm.  Agreement with liblithogpu is
    checked in tools/cufft_check.py (profiles/r2_cufft_baseline.json)."""
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from cufft_ilt import CufftIlt, timed
    try:
        lib = CufftIlt(ks, prm)
        a = prm.mask_steepness
        theta = ((2 * targets - 1) * (2.0 / a)).contiguous()
        ms, _ = timed(lib, theta, targets.contiguous(), iters, steps=2, warmup=1)
        v = targets.shape[0] * iters / (ms / 1e3)
        del lib
        torch.cuda.empty_cache()
        return {"impl": "cuFFT (torch.fft) batched, device-resident, graph-captured; same decimated algorithm, "
                        "no kernel pairs / mirror-stack merge",
                "tiles": int(targets.shape[0]), "value": v, "unit": "tile-iter/s",
                "ours_over_library": ours_value / v}
    except Exception as e:  # diagnostics only: never fails the headline
        return {"error": repr(e)[:300]}


def _chip_e2e(args, ctx, tl, mine, tile_polys, batches, solvers, costs, iters, D, stream, dev, ks, prm, local):
    """Same job through the C ABI from host memory: pinned polygon arrays ->
    lithogpu_rasterize (device raster) -> lithogpu_ilt_set_tiles /
    lithogpu_ilt_run -> lithogpu_ilt_get_window_async writing each tile's core
    straight into the stitched chip mask (pinned host, f32).  Two contexts
    (streams) alternate over the launch batches, so batch b's 3.3 GB/step of
    D2H runs on the copy engine under batch b+1's iterations."""
    import ctypes as C

    import torch
    import paper_2602_15036_b200 as L
    from paper_2602_15036_b200._lib import F64, check, lib
    N = tl.n
    c, h = tl.core, tl.halo
    pinned = [(torch.from_numpy(xy).pin_memory(), torch.from_numpy(st).pin_memory()) for xy, st in tile_polys]
    chip_mask = torch.zeros((tl.ty * c, tl.tx * c), dtype=torch.float32).pin_memory()
    nb = max(b1 - b0 for b0, b1 in batches)
    # second context / stream with its own kernel upload and solvers
    stream2 = torch.cuda.Stream(device=dev)
    ctx2 = L.Context(local)
    ctx2.set_stream(stream2.cuda_stream)
    dk2 = L.DeviceKernels(ks, "f32", ctx2)
    solvers2 = {nt: L.IltSolver(dk2, prm, nt, "f32", ctx2) for nt in solvers}
    costs2 = {nt: torch.zeros_like(costs[nt]) for nt in costs}
    lanes = [(ctx, stream, solvers, costs), (ctx2, stream2, solvers2, costs2)]
    rasters = [torch.empty((nb, N, N), dtype=torch.float64, device=dev) for _ in lanes]
    cost_host = torch.zeros((len(batches), iters), dtype=torch.float64).pin_memory()

    def e2e_step():
        for bi, (b0, b1) in enumerate(batches):
            cx, st, sv, cs = lanes[bi % 2]
            s = sv[b1 - b0]
            raster = rasters[bi % 2]
            for j in range(b0, b1):
                xy, stt = pinned[j]
                g = tl.tile_grid(mine[j]).c()
                check(lib().lithogpu_rasterize(cx.handle, C.byref(g), xy.data_ptr(), stt.data_ptr(), stt.numel() - 1,
                                               1.0, raster[j - b0].data_ptr()))
            check(lib().lithogpu_ilt_set_tiles(s._h, raster.data_ptr(), None, F64))
            check(lib().lithogpu_ilt_run(s._h, iters, cs[b1 - b0].data_ptr(), None))
            with torch.cuda.stream(st):
                cost_host[bi].copy_(cs[b1 - b0].sum(dim=1), non_blocking=True)
            for j in range(b0, b1):
                i, jj = tl.tile_ij(mine[j])
                s.get_window(j - b0, h, h, c, c, out=chip_mask[jj * c:(jj + 1) * c, i * c:(i + 1) * c], async_=True)

    for _ in range(max(1, min(args.warmup, 2))):
        e2e_step()
    torch.cuda.synchronize()
    et = []
    for _ in range(args.steps):
        D.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()
        torch.cuda.synchronize()  # every stream: the last batch's D2H has landed in the chip mask
        et.append((time.perf_counter() - t0) * 1e3)
    e_ms = D.max_scalar(float(np.sum(et))) / args.steps
    h2d = int(sum(xy.nbytes + st.nbytes for xy, st in tile_polys))
    d2h = int(len(mine) * c * c * 4 + cost_host.numel() * 8)
    for sv in solvers2.values():
        sv.close()
    return {"value": len(tl) * iters / (e_ms / 1e3), "unit": "tile-iter/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": e_ms,
            "path": "C ABI: pinned polygons -> lithogpu_rasterize -> lithogpu_ilt_set_tiles/run -> "
                    "lithogpu_ilt_get_window_async (tile cores into the stitched chip mask, pinned host f32); "
                    "two contexts alternate over the batches so each batch's D2H overlaps the next batch",
            "timer": "host perf_counter with device sync on both sides, max over ranks"}


def _roofline(ctx, info, N, F, K, tiles, prof, iters, cfg):
    """Dominant kernel of the profiled launch sequence against the measured
    FP32 (FFMA) peak: algorithmic FFT flops per launch (kernel_model x tiles)
    / CUDA-event launch duration."""
    peak_fp32 = ctx.fp32_peak_tflops()
    geo = {"N": N, "n": info["nx_sub"], "B": info["band_x"]}
    Kt = info.get("fast_order") or K
    Ft = info.get("fast_stacks") or F
    model = kernel_model(geo, Ft, Kt, tiles)
    kernel_ms = {k: v[1] / v[0] for k, v in prof.items()}
    top = max(prof, key=lambda k: prof[k][1])
    f1, b1 = model.get(top, (0.0, 0.0))
    flops, byts = f1 * tiles, b1 * tiles
    top_ms = kernel_ms[top]
    achieved = flops / (top_ms * 1e-3) / 1e12
    tot = sum(x[1] for x in prof.values())
    shares = {k: round(v[1] / tot, 4) for k, v in prof.items()}
    pk = _peaks()
    hbm_peak = pk.get("hbm_gbs") or pk.get("hbm_copy_gbs")
    traffic, tsrc = _ncu_traffic(top, cfg, tiles)
    whole_flops = sum(model[k][0] for k in model) * tiles
    return {"bound": "fp32", "kernel": top, "achieved": achieved, "peak": peak_fp32, "unit": "TFLOP/s",
            "frac": achieved / peak_fp32 if peak_fp32 else None, "traffic": traffic, "traffic_source": tsrc,
            "peak_source": "measured on-box FFMA microbenchmark (lithogpu_fp32_peak); MEASURED_PEAKS.json has "
                           "no FP32 entry",
            "tiles_per_launch": tiles, "flops_per_launch": flops, "algorithmic_bytes_per_launch": byts,
            "kernel_ms": top_ms, "hbm_gbs_algorithmic": byts / (top_ms * 1e-3) / 1e9, "hbm_peak_gbs": hbm_peak,
            "frac_hbm": (byts / (top_ms * 1e-3) / 1e9 / hbm_peak) if hbm_peak else None,
            "bound_note": "FP32-pipe / issue bound (FFT butterflies): the band-limited algorithm moves ~30x fewer "
                          "bytes than a full-grid design; HBM view in hbm_* / frac_hbm",
            "whole_iteration_tflops": whole_flops / (tot / iters * 1e-3) / 1e12 if tot else None,
            "kernel_share": shares, "kernel_ms_avg": kernel_ms,
            "instrumented_iter_ms": tot / iters}


def run_tile(args, world, rank, local, cfg, ctx=None, stream=None, D=None, quiet=False, steps=None):
    """One tile per GPU (C2 / C3 / C4): the old headline, now a secondary line."""
    import torch
    import paper_2602_15036_b200 as L
    from paper_2602_15036_b200 import layouts as LY

    own = D is None
    if own:
        local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        D = Dist(world, local, args.dist_backend)
        stream = torch.cuda.Stream(device=D.dev)  # non-default stream: ILT loop is graph-captured
        torch.cuda.set_stream(stream)
        ctx = L.Context(local)
        ctx.set_stream(stream.cuda_stream)
    dev = D.dev
    steps = steps or args.steps
    grid, polys, ks, iters, desc = make_problem(cfg, rank, "gpu", ctx)
    N = grid.nx
    F, K = ks.weights.shape
    dk = L.DeviceKernels(ks, "f32", ctx)
    info = dk.info()
    xy, starts = LY.polygon_arrays(polys)
    target = torch.empty((1, N, N), dtype=torch.float64, device=dev)
    _raster_to(ctx, grid, xy, starts, target)
    target32 = target.float()
    prm = L.IltParams(focus_weights=[1.0 / F] * F, **ILT)
    solver = L.IltSolver(dk, prm, 1, "f32", ctx)
    cost_dev = torch.zeros((iters, 1), dtype=torch.float64, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def step():
        solver.set_tiles(target32)
        solver.run_device(iters, cost_dev)  # one CUDA graph: all iterations
        D.allreduce(cost_dev)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local) if not quiet else None
    if clocks:
        clocks.start()
    l0 = ctx.launch_count()
    times, total_ms = timed_steps(step, steps, stream, D, flush)
    launches = ctx.launch_count() - l0
    clk = clocks.stop() if clocks else None
    ms = total_ms / steps
    value = world * iters / (ms / 1e3)
    final_cost = cost_dev[:, 0].cpu().numpy()

    roof = None
    if rank == 0:
        ctx.set_profiling(True)
        ctx.profile_report(reset=True)
        step()
        torch.cuda.synchronize()
        prof = ctx.profile_report(reset=True)
        ctx.set_profiling(False)
        roof = _roofline(ctx, info, N, F, K, 1, prof, iters, cfg)

    e2e = None
    if not args.no_e2e:
        mask_host = torch.empty((1, N, N), dtype=torch.float32).pin_memory()
        cost_host = torch.empty((iters, 1), dtype=torch.float64).pin_memory()
        xy_pin = torch.from_numpy(xy).pin_memory()
        st_pin = torch.from_numpy(starts).pin_memory()
        tgt_dev = torch.empty((1, N, N), dtype=torch.float64, device=dev)

        def e2e_step():
            _raster_to(ctx, grid, xy_pin.numpy(), st_pin.numpy(), tgt_dev)  # H2D polygons + GPU raster
            solver.set_tiles(tgt_dev)                                         # theta0 from target
            solver.run_device(iters, cost_dev)
            D.allreduce(cost_dev)
            cost_host.copy_(cost_dev, non_blocking=True)
            _get_mask(solver, mask_host)                                      # D2H final mask
        for _ in range(max(1, min(args.warmup, 2))):
            e2e_step()
        torch.cuda.synchronize()
        et = []
        for _ in range(steps):
            flush.fill_(1.0)
            D.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_step()
            torch.cuda.synchronize()
            et.append((time.perf_counter() - t0) * 1e3)
        e_ms = D.max_scalar(float(np.sum(et))) / steps
        e2e = {"value": world * iters / (e_ms / 1e3), "unit": "tile-iter/s",
               "h2d_bytes_per_step": int(xy.nbytes + starts.nbytes),
               "d2h_bytes_per_step": int(mask_host.numel() * 4 + cost_host.numel() * 8),
               "ms_per_step": e_ms, "timer": "host perf_counter with device sync on both sides"}
    solver.close()
    res = None
    if rank == 0:
        res = {
            "metric": f"ILT tile-iterations/s ({desc})", "value": value, "unit": "tile-iter/s", "n_gpus": world,
            "steps": steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded layout, GPU-rasterized; Abbe-SVD SOCS kernels)",
            "config": {"workload": desc, "tile": N, "K": K, "F": F, "iterations_per_step": iters, "tiles_per_gpu": 1,
                       "decimated_grid": info["nx_sub"], "kernel_band": info["band_x"],
                       "kernel_transforms_per_stack": info.get("fast_order"),
                       "computed_focus_stacks": info.get("fast_stacks"), "ilt": ILT,
                       "l2": "flushed between steps (256 MiB write, untimed)",
                       "parallelism": f"one tile per rank, {world} rank(s); per-step all-reduce of the cost vector"},
            "roofline": roof, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk,
            "final_cost": [float(final_cost[0]), float(final_cost[-1])] if len(final_cost) else None,
        }
        if not quiet:
            if not args.no_cpu_baseline and world == 1:
                res["cpu_baseline"] = _cpu_baseline(cfg)
            if world == 1 and roof:
                res["in_graph"] = _in_graph_timeline(cfg, roof["kernel"], roof["flops_per_launch"], roof["peak"])
            print(json.dumps(res), flush=True)
    if own:
        D.close()
    return res


def _raster_to(ctx, grid, xy, starts, out_dev):
    import ctypes as C
    from paper_2602_15036_b200._lib import check, lib
    g = grid.c()
    check(lib().lithogpu_rasterize(ctx.handle, C.byref(g), xy.ctypes.data, starts.ctypes.data,
                                   len(starts) - 1, 1.0, out_dev.data_ptr()))


def _get_mask(solver, mask_host):
    from paper_2602_15036_b200._lib import F32, check, lib
    check(lib().lithogpu_ilt_get_tiles(solver._h, None, mask_host.data_ptr(), F32))


def _c1_forward(ctx, stream, cpu=True):
    """C1 (configs[0]): 1024^2 tile, K=8, forward aerial + blur + threshold;
    device-resident, CUDA-event timed, Mpixel/s; and the reference
    (oracle/_ref image_socs -> resist_filter -> threshold, imaging.cpp:218-241,
    316-323, ai.cpp:85-94) on the same tile on 1 and on all host cores."""
    import torch
    import paper_2602_15036_b200 as L
    from paper_2602_15036_b200 import layouts as LY
    grid, polys, ks, _, desc = make_problem("c1", 0, "host")
    dk = L.DeviceKernels(ks, "f32", ctx)
    xy, starts = LY.polygon_arrays(polys)
    dev = torch.device("cuda", ctx.device)
    mask = torch.empty((grid.ny, grid.nx), dtype=torch.float64, device=dev)
    _raster_to(ctx, grid, xy, starts, mask)
    m32 = mask.float()
    for _ in range(3):
        dk.image(m32, sigma_nm=2.0, threshold=0.25, want=("intensity", "resist", "print"))
    torch.cuda.synchronize()
    reps = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        dk.image(m32, sigma_nm=2.0, threshold=0.25, want=("intensity", "resist", "print"))
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out = {"workload": desc, "ms_per_image": ms, "mpix_s": grid.nx * grid.ny / (ms * 1e-3) / 1e6,
           "outputs": "aerial f32 + resist f32 + print u8", "l2": "warm (repeated image)"}
    # end to end from host memory: host mask in, host aerial/resist/print out
    mh = m32.cpu().numpy()
    dk.image(mh, sigma_nm=2.0, threshold=0.25, want=("intensity", "resist", "print"))
    t0 = time.perf_counter()
    for _ in range(10):
        dk.image(mh, sigma_nm=2.0, threshold=0.25, want=("intensity", "resist", "print"))
    e_ms = (time.perf_counter() - t0) / 10 * 1e3
    out["e2e"] = {"value": grid.nx * grid.ny / (e_ms * 1e-3) / 1e6, "unit": "Mpixel/s", "ms_per_image": e_ms,
                  "h2d_bytes_per_image": int(mh.nbytes), "d2h_bytes_per_image": int(grid.nx * grid.ny * 9),
                  "timer": "host perf_counter around the synchronous host-buffer API call"}
    if cpu:
        out["cpu_baseline"] = _cpu_c1(grid, polys, ks)
    out["contours"] = _contours_c1(ctx, stream, dk, m32, grid)
    return out


def _cpu_c1(grid, polys, ks):
    """Reference C1 on the host: image_socs + resist_filter + threshold of the
    same 1024^2 tile (fp64), 1 thread and all threads."""
    from oracle import refpy as R
    if not R.available():
        return {"unavailable": "oracle/_ref not built"}
    mask = R.rasterize(polys, grid.nx, grid.ny, grid.pitch_nm, grid.origin_x_nm, grid.origin_y_nm, 1.0)
    out = {"unit": "Mpixel/s", "kind": "reference",
           "sample": "1 image of the C1 tile per thread setting: reference image_socs -> gaussian_blur -> "
                     "threshold (fp64, FFT stand-in)"}
    cores = os.cpu_count() or 1
    for th in (1, cores):
        R.set_threads(th)
        t0 = time.perf_counter()
        I = R.image_socs(mask, ks.weights[0], ks.support, ks.values[0])
        rr = R.gaussian_blur(I, 2.0, 1.0)
        _ = (rr >= 0.25)
        dt = time.perf_counter() - t0
        out["value_1core" if th == 1 else "value"] = grid.nx * grid.ny / dt / 1e6
        out["s_1core" if th == 1 else "s_all"] = dt
    out["cores"] = cores
    return out


def _contours_c1(ctx, stream, dk, m32, grid, n_gauges=4096, radius=20.0):
    """SURVEY §8f rank 1 stage on the C1 resist image: GPU marching squares +
    EPE gauges against the reference contour.cpp on one host core."""
    import torch
    import paper_2602_15036_b200 as L
    res = dk.image(m32, sigma_nm=2.0, want=("resist",))["resist"].to(torch.float64)
    res[:2, :] = 0.0  # clear the tile frame (halo): contours must close inside the tile
    res[-2:, :] = 0.0
    res[:, :2] = 0.0
    res[:, -2:] = 0.0
    rng = np.random.default_rng(7)
    ang = rng.uniform(0, 2 * np.pi, n_gauges)
    gauges = np.column_stack([rng.uniform(0, grid.nx, n_gauges), rng.uniform(0, grid.ny, n_gauges),
                              np.cos(ang), np.sin(ang)])
    for _ in range(2):
        cs = L.marching_squares(res, grid, ILT["threshold"], ctx)
        L.measure_epe(cs, gauges, radius)
    torch.cuda.synchronize()
    reps = 10
    t0 = time.perf_counter()
    for _ in range(reps):
        cs = L.marching_squares(res, grid, ILT["threshold"], ctx)
    t1 = time.perf_counter()
    for _ in range(reps):
        epe, op = L.measure_epe(cs, gauges, radius)
    t2 = time.perf_counter()
    out = {"stage": "marching_squares + measure_epe (contour.cpp:58-201) on the C1 resist image",
           "loops": len(cs.loop_start) - 1, "points": int(len(cs.xs)), "gauges": n_gauges,
           "gpu_ms_contours": (t1 - t0) / reps * 1e3, "gpu_ms_epe": (t2 - t1) / reps * 1e3,
           "timer": "host perf_counter around the synchronous API call (device field, host result)"}
    try:
        from oracle import refpy as R
        if R.available():
            R.set_threads(1)
            f = res.cpu().numpy()
            t0 = time.perf_counter()
            R.marching_squares(f, ILT["threshold"], grid.pitch_nm, grid.origin_x_nm, grid.origin_y_nm)
            t1 = time.perf_counter()
            R.measure_epe(gauges, radius)
            t2 = time.perf_counter()
            out.update({"ref_cpu_ms_contours": (t1 - t0) * 1e3, "ref_cpu_ms_epe": (t2 - t1) * 1e3,
                        "ref_cores": 1})
    except Exception as e:  # the reference arm is optional here
        out["ref_error"] = str(e)[:200]
    return out


def _ncu_traffic(kernel, cfg="c5", tiles=None):
    """dram__bytes_read.sum + dram__bytes_write.sum of `kernel` (per launch) from
    the newest committed `ncu --set full` capture summary of this config
    (profiles/r<round>_<cfg>_*_ncu.json, tools/ncu_summarize.py; newest =
    highest round, then highest version number).  ncu flushes caches before
    each replay, so this is an upper bound on a warm step's HBM traffic."""
    import glob

    def key(p):
        nums = [int(x) for x in re.findall(r"\d+", os.path.basename(p))]
        return nums
    cands = glob.glob(os.path.join(ROOT, "profiles", f"*_{cfg}_*ncu.json"))
    if not cands and cfg == "c2":
        cands = glob.glob(os.path.join(ROOT, "profiles", "r1_s2_v*_ncu.json"))
    best = None
    for p in sorted(cands, key=key):
        try:
            caps = json.load(open(p)).get("full_captures", {})
        except Exception:
            continue
        c = caps.get("fk_" + kernel) or caps.get(kernel)
        if c and c.get("dram_bytes") is not None:
            best = (c["dram_bytes"], f"{os.path.basename(p)} ({c.get('kernel')}, grid {c.get('grid')})",
                    c.get("grid"))
    if not best:
        return None, None
    b, src, grid = best
    if tiles and grid:  # per launch of `tiles` tiles: scale by the capture's blockIdx.z tile count
        try:
            z = int(str(grid).strip("()").split(",")[2])
            if z > 0 and z != tiles:
                return b * tiles / z, src + f", scaled x{tiles}/{z} tiles"
        except Exception:
            pass
    return b, src


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def _in_graph_timeline(cfg_name, top, top_flops, peak, tiles=1):
    """Per-kernel durations inside the replayed CUDA graph (tools/trace.py:
    first-CTA start to last-warp end from %globaltimer stamps, no per-launch
    events breaking the graph), and the dominant kernel's roofline fraction on
    that duration beside the event-timed one."""
    try:
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "trace.py"), "--config", cfg_name,
                            "--tiles", str(tiles)], cwd=ROOT, capture_output=True, text=True, timeout=600)
        d = json.loads(r.stdout.strip().splitlines()[-1])
        per = d["per_kernel"]
        us = per.get(top, {}).get("dur_us")
        out = {"tiles_per_launch": tiles, "per_iter_us": d["per_iter_us"],
               "kernel_us": {k: v["dur_us"] for k, v in per.items()},
               "gap_us": {k: v["gap_before_us"] for k, v in per.items()}}
        if us:
            out.update({"top_kernel": top, "achieved_tflops": top_flops / (us * 1e-6) / 1e12,
                        "frac": top_flops / (us * 1e-6) / 1e12 / peak if peak else None})
        return out
    except Exception as e:
        return {"unavailable": str(e)[:200]}


# ---------------------------------------------------------------------------
# reference arm (CPU): oracle/_ref, never liblithogpu.so
# ---------------------------------------------------------------------------
def _ref_problem(cfg_name):
    """(grid, kernels, target raster, iterations, description) for the
    reference arm and cpu_baseline: C5 uses tile 0 of the same chip; kernels
    from oracle/kernels_np.py, raster from the reference rasterize_layer."""
    from oracle import refpy as R
    if cfg_name == "c5":
        from paper_2602_15036_b200 import layouts as LY
        from paper_2602_15036_b200.api import Grid
        N, K, foci, iters, desc = CONFIGS["c5"]
        tl = c5_tiling()
        polys = LY.chip_layout(tl, seed=C5_SEED)
        g = tl.tile_grid(0)
        target = R.rasterize(tl.tile_polygons(polys, 0), g.nx, g.ny, g.pitch_nm, g.origin_x_nm, g.origin_y_nm, 1.0)
        ks = kernel_stacks(Grid(N, N, 1.0), foci, K, "oracle")
        return g, ks, target, iters, desc
    grid, polys, ks, iters, desc = make_problem(cfg_name, 0, "oracle")
    target = R.rasterize(polys, grid.nx, grid.ny, grid.pitch_nm, grid.origin_x_nm, grid.origin_y_nm, 1.0)
    return grid, ks, target, iters, desc


def _fft_speed(n=2048):
    """The reference's fft2 stand-in (oracle/fft64.c, the FFTW3 role) on one
    n^2 complex128 transform: 1 thread, all threads, and numpy.fft.fft2
    (pocketfft, single-threaded) on the same data as a tuned-FFT yardstick."""
    import ctypes as C
    from oracle import refpy as R
    a = np.random.default_rng(0).standard_normal((n, n)) + 1j * np.random.default_rng(1).standard_normal((n, n))
    out = {"n": n}
    cores = os.cpu_count() or 1
    for th in (1, cores):
        R.set_threads(th)
        b = a.copy()
        R.lib().oracle_fft2(b.ctypes.data_as(C.c_void_p), n, n, -1)
        t0 = time.perf_counter()
        R.lib().oracle_fft2(b.ctypes.data_as(C.c_void_p), n, n, -1)
        out["standin_ms_1thread" if th == 1 else "standin_ms_all"] = (time.perf_counter() - t0) * 1e3
    np.fft.fft2(a)
    t0 = time.perf_counter()
    np.fft.fft2(a)
    out["pocketfft_ms_1thread"] = (time.perf_counter() - t0) * 1e3
    out["standin_parallel_speedup"] = out["standin_ms_1thread"] / out["standin_ms_all"]
    out["threads"] = cores
    return out


def _ilt_prm():
    return [ILT["mask_steepness"], ILT["resist_beta"], ILT["threshold"], ILT["resist_sigma_nm"], ILT["dose"],
            ILT["step"]]


def _cpu_baseline(cfg_name, n_iter=1):
    """Reference CPU implementation (oracle/_ref) on a bounded sample: n_iter
    ILT iterations of one tile on all host threads; per-core figure from the
    FFT stand-in's measured parallel speed-up (the FFTs are ~all of the time)."""
    from oracle import refpy as R
    if not R.available():
        return {"value": None, "unit": "tile-iter/s", "cores": 0, "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    grid, ks, target, iters, desc = _ref_problem(cfg_name)
    cores = os.cpu_count() or 1
    R.set_threads(cores)
    theta = ((2 * target - 1) * (2.0 / ILT["mask_steepness"])).copy()
    F = ks.weights.shape[0]
    t0 = time.perf_counter()
    for _ in range(n_iter):
        R.ilt_iteration(theta, target, ks.weights, ks.support, ks.values, [1.0 / F] * F, _ilt_prm(), grid.pitch_nm)
    dt = time.perf_counter() - t0
    fs = _fft_speed()
    value = n_iter / dt
    return {"value": value, "unit": "tile-iter/s", "cores": cores, "kind": "reference",
            "per_core_value": value / fs["standin_parallel_speedup"],
            "per_core_note": "all-core value / the FFT stand-in's measured 2048^2 parallel speed-up",
            "fft2": fs,
            "sample": f"{n_iter} ILT iteration(s) of one {grid.nx}x{grid.ny} tile (K={ks.weights.shape[1]}, F={F}) "
                      f"through the unmodified reference image_socs/gaussian_blur/fft2 (fp64, FFT stand-in, "
                      f"{cores} OpenMP threads), {dt:.1f} s; the whole {CONFIGS[cfg_name][3]}-iteration job "
                      f"extrapolates linearly (tiles x iterations)"}


def run_reference(args, world, rank):
    if rank != 0:
        return None
    from oracle import refpy as R
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libref_litho.so not built"}))
        return None
    grid, ks, target, iters, desc = _ref_problem(args.config)
    cores = os.cpu_count() or 1
    R.set_threads(cores)
    F = ks.weights.shape[0]
    theta = ((2 * target - 1) * (2.0 / ILT["mask_steepness"])).copy()

    def step():  # bounded sample: one ILT iteration of one tile per step
        R.ilt_iteration(theta, target, ks.weights, ks.support, ks.values, [1.0 / F] * F, _ilt_prm(), grid.pitch_nm)

    warm = min(args.warmup, 1)  # host code: one warm-up (page faults, plans) is enough
    for _ in range(warm):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    ms = dt / args.steps * 1e3
    value = 1.0 / (ms / 1e3)
    res = {"impl": "reference", "metric": f"ILT tile-iterations/s ({desc})", "value": value,
           "unit": "tile-iter/s", "n_gpus": world, "steps": args.steps, "warmup": warm,
           "ms_per_step": ms, "higher_is_better": True, "scaling": "strong" if args.config == "c5" else "weak",
           "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (same seeded layout as the GPU arm; kernels from oracle/kernels_np.py, the same "
                   "Abbe-SVD route as the product generator; raster by the reference rasterize_layer)",
           "config": {"workload": desc, "tile": grid.nx, "K": int(ks.weights.shape[1]), "F": F,
                      "iterations_per_step": 1,
                      "note": "one ILT iteration of one tile per step (bounded CPU sample); warm-up capped at 1"},
           "cpu_baseline": {"value": value, "unit": "tile-iter/s", "cores": cores, "kind": "reference",
                            "sample": "1 ILT iteration of one tile per step, unmodified reference sources "
                                      "(oracle/_ref), FFT stand-in on all host threads"},
           "e2e": {"value": value, "unit": "tile-iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)
    return res


def main():
    args = parse()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    if args.config == "c5":
        run_chip(args, world, rank, local)
    elif args.config == "c1":
        import torch
        import paper_2602_15036_b200 as L
        torch.cuda.set_device(local)
        st = torch.cuda.Stream()
        torch.cuda.set_stream(st)
        ctx = L.Context(local)
        ctx.set_stream(st.cuda_stream)
        if rank == 0:
            print(json.dumps(_c1_forward(ctx, st, cpu=not args.no_cpu_baseline)), flush=True)
    else:
        run_tile(args, world, rank, local, args.config)


if __name__ == "__main__":
    main()
