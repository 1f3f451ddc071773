#!/usr/bin/env python
"""Benchmark of the B200-native SOCS imaging / ILT hot path.

Headline workload (BASELINE.json configs[1], "C2"): one 2048x2048 tile per
GPU, K = 16 SOCS kernels, 1 focus plane, Gaussian-blur (sigma 2 nm) sigmoid
resist, 50 ILT gradient iterations = one step.  Metric: ILT
tile-iterations/s, whole job (weak scaling: one tile per rank, the global
cost all-reduced over NCCL every iteration when N > 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

`value` is device-timed (CUDA events, inputs resident in HBM, L2 flushed
between steps, max over ranks); `e2e` runs the same job through the public
API from host buffers: polygon layout H2D -> GPU rasterization -> ILT -> mask
D2H.  `--impl reference` times the reference's own CPU implementation
(oracle/_ref: the unmodified reference sources, all host threads) on the
same config.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import threading
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
           "C5: chip-scale 256 halo-padded 2048x2048 tiles, K=24, F=3, 50 ILT iterations, sharded over ranks"),
}
C5_TILES, C5_BATCH = 256, 32
ILT = dict(mask_steepness=4.0, resist_beta=30.0, threshold=0.25, resist_sigma_nm=2.0, dose=1.0, step=0.5)
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_problem(cfg_name, rank):
    import paper_2602_15036_b200 as L
    from paper_2602_15036_b200 import layouts as LY
    N, K, foci, iters, desc = CONFIGS[cfg_name]
    grid = L.Grid(N, N, 1.0, 0.0, 0.0)
    gen = LY.curvilinear if cfg_name == "c4" else LY.line_space_contacts
    polys = gen(N, N, seed=1000 + rank)
    model = L.OpticalModel(source=L.make_annular_source(0.4, 0.8, 21))
    ks = L.build_socs_kernels(model, grid, foci, k_fixed=K)
    return grid, polys, ks, iters, desc


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
    """Per-launch FFT flops (5 L log2 L per length-L complex transform) and
    algorithmic bytes of each kernel of one ILT iteration on one tile, for the
    implemented decimated-band algorithm."""
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


def run_c5(args, world, rank, local):
    """C5 (configs[4]): 256 independent halo-padded 2048^2 tiles (seeded
    synthetic layouts, one per tile), sharded over ranks (chip.shard); each
    rank runs its tiles in launch batches of C5_BATCH (blockIdx.z = tile),
    50 ILT iterations per batch, and the per-iteration global cost is
    all-reduced once per step.  Weak scaling in the number of GPUs with a
    fixed total of 256 tiles -> reported as "strong" (total work fixed)."""
    import torch
    import paper_2602_15036_b200 as L
    from paper_2602_15036_b200 import chip, layouts as LY
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx = L.Context(local)
    ctx.set_stream(stream.cuda_stream)
    N, K, foci, iters, desc = CONFIGS["c5"]
    grid = L.Grid(N, N, 1.0)
    model = L.OpticalModel(source=L.make_annular_source(0.4, 0.8, 21))
    ks = L.build_socs_kernels(model, grid, foci, k_fixed=K, backend="gpu", ctx=ctx)
    dk = L.DeviceKernels(ks, "f32", ctx)
    info = dk.info()
    mine = list(chip.shard(C5_TILES, world, rank))
    targets = torch.empty((len(mine), N, N), dtype=torch.float32, device=dev)
    tmp = torch.empty((N, N), dtype=torch.float64, device=dev)
    for j, t in enumerate(mine):
        xy, starts = LY.polygon_arrays(LY.line_space_contacts(N, N, seed=5000 + t))
        _raster_to(ctx, grid, xy, starts, tmp)
        targets[j].copy_(tmp)
    theta0 = (2 * targets - 1) * (2.0 / ILT["mask_steepness"])
    F = len(foci)
    prm = L.IltParams(focus_weights=[1.0 / F] * F, **ILT)
    nb = min(C5_BATCH, max(1, len(mine)))
    solver = L.IltSolver(dk, prm, nb, "f32", ctx)
    cost = torch.zeros((iters, nb), dtype=torch.float64, device=dev)
    gcost = torch.zeros(iters, dtype=torch.float64, device=dev)

    def step():
        gcost.zero_()
        for b0 in range(0, len(mine), nb):
            b1 = min(b0 + nb, len(mine))
            tg, th = targets[b0:b1], theta0[b0:b1]
            if b1 - b0 < nb:  # ragged last batch: pad with copies of the first tile (cost not counted)
                tg = torch.cat([tg, targets[:nb - (b1 - b0)]])
                th = torch.cat([th, theta0[:nb - (b1 - b0)]])
            solver.set_tiles(tg.contiguous(), th.contiguous())
            solver.run_device(iters, cost)
            gcost.add_(cost[:, :b1 - b0].sum(dim=1))
        if world > 1:
            import torch.distributed as dist
            dist.all_reduce(gcost)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    times = []
    l0 = ctx.launch_count()
    for _ in range(args.steps):
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    launches = ctx.launch_count() - l0
    clk = clocks.stop()
    total_ms = float(np.sum(times))
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / args.steps
    if rank == 0:
        print(json.dumps({
            "metric": f"ILT tile-iterations/s ({desc})", "value": C5_TILES * iters / (ms / 1e3),
            "unit": "tile-iter/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (one seeded line/space+contact layout per tile, GPU-rasterized; "
                                    "GPU Abbe-SVD kernels)",
            "config": {"workload": desc, "tiles_total": C5_TILES, "tiles_per_rank": len(mine),
                       "tiles_per_launch": nb, "tile": N, "K": K, "F": F, "iterations_per_step": iters,
                       "computed_focus_stacks": info.get("fast_stacks"),
                       "kernel_transforms_per_stack": info.get("fast_order"), "ilt": ILT,
                       "l2": "working set (tiles x ~100 MB) far above L2",
                       "parallelism": f"256 tiles sharded over {world} rank(s); NCCL all-reduce of the "
                                      f"per-iteration global cost once per step"},
            "e2e": None, "gpu_launches": int(launches), "clocks": clk,
            "final_cost": [float(gcost[0]), float(gcost[-1])]}), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


def run_ours(args, world, rank, local):
    import torch
    import paper_2602_15036_b200 as L
    from paper_2602_15036_b200 import layouts as LY

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.Stream(device=dev)  # non-default stream: ILT loop is graph-captured
    torch.cuda.set_stream(stream)
    ctx = L.Context(local)
    ctx.set_stream(stream.cuda_stream)

    grid, polys, ks, iters, desc = make_problem(args.config, rank)
    N = grid.nx
    F, K = ks.weights.shape
    dk = L.DeviceKernels(ks, "f32", ctx)
    info = dk.info()
    xy, starts = LY.polygon_arrays(polys)

    # device-resident inputs: target raster (GPU rasterizer) and theta0
    target = torch.empty((1, N, N), dtype=torch.float64, device=dev)
    _raster_to(ctx, grid, xy, starts, target)
    target32 = target.float()
    theta0 = ((2 * target32 - 1) * (2.0 / ILT["mask_steepness"])).contiguous()
    prm = L.IltParams(focus_weights=[1.0 / F] * F, **ILT)
    solver = L.IltSolver(dk, prm, 1, "f32", ctx)
    cost_dev = torch.zeros((iters, 1), dtype=torch.float64, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def step():
        solver.set_tiles(target32, theta0)
        solver.run_device(iters, cost_dev)  # one CUDA graph: all iterations
        if world > 1:
            import torch.distributed as dist
            dist.all_reduce(cost_dev)  # global ILT cost of every iteration (sum over tiles / ranks)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    times = []
    l0 = ctx.launch_count()
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flush between steps (not timed)
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    launches = ctx.launch_count() - l0
    clk = clocks.stop()
    total_ms = float(np.sum(times))
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * iters / (ms_per_step / 1e3)  # tile-iterations/s, whole job
    final_cost = cost_dev[:, 0].cpu().numpy()

    # ---- per-kernel CUDA-event profile (separate instrumented steps) ----
    ctx.set_profiling(True)
    ctx.profile_report(reset=True)
    nprof = 2
    for _ in range(nprof):
        step()
    torch.cuda.synchronize()
    prof = ctx.profile_report(reset=True)
    ctx.set_profiling(False)
    peak_fp32 = ctx.fp32_peak_tflops()
    geo = {"N": N, "n": info["nx_sub"], "B": info["band_x"]}
    Kt = info.get("fast_order") or K  # transforms per stack (kernel pairs: ceil(K/2))
    Ft = info.get("fast_stacks") or F  # computed focus stacks (mirror stacks merged)
    model = kernel_model(geo, Ft, Kt)
    kernel_ms = {k: v[1] / v[0] for k, v in prof.items()}
    top = max(prof, key=lambda k: prof[k][1])
    top_flops, top_bytes = model.get(top, (0.0, 0.0))
    top_ms = kernel_ms[top]
    achieved = top_flops / (top_ms * 1e-3) / 1e12
    iter_ms_prof = sum(v[1] for v in prof.values()) / (nprof * iters)
    shares = {k: round(v[1] / sum(x[1] for x in prof.values()), 4) for k, v in prof.items()}

    # ---- end to end through the public API from host buffers ----
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
            if world > 1:
                import torch.distributed as dist
                dist.all_reduce(cost_dev)
            cost_host.copy_(cost_dev, non_blocking=True)
            _get_mask(solver, mask_host)                                      # D2H final mask
        for _ in range(max(1, args.warmup)):
            e2e_step()
        torch.cuda.synchronize()
        et = []
        for _ in range(args.steps):
            flush.fill_(1.0)
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_step()
            torch.cuda.synchronize()
            et.append((time.perf_counter() - t0) * 1e3)
        e_ms = float(np.sum(et))
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e_ms /= args.steps
        e2e = {"value": world * iters / (e_ms / 1e3), "unit": "tile-iter/s",
               "h2d_bytes_per_step": int(xy.nbytes + starts.nbytes),
               "d2h_bytes_per_step": int(mask_host.numel() * 4 + cost_host.numel() * 8),
               "ms_per_step": e_ms, "timer": "host perf_counter with device sync on both sides"}

    # ---- secondary: C1 forward aerial-image throughput (Mpixel/s) ----
    aerial = None
    batched = None
    if rank == 0:
        aerial = _c1_forward(ctx, stream)
        batched = _batched_ilt(ctx, stream, dk, target32, theta0, prm, iters)

    result = None
    if rank == 0:
        cpu = None
        cufftw = None
        if not args.no_cpu_baseline and world == 1:
            cpu = _cpu_baseline(args.config)
            cufftw = _cufftw_baseline(args.config)
        result = {
            "metric": f"ILT tile-iterations/s ({desc})",
            "value": value,
            "unit": "tile-iter/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (seeded line/space+contact layout, GPU-rasterized; Abbe-SVD SOCS kernels)",
            "config": {"workload": desc, "tile": N, "K": K, "F": F, "iterations_per_step": iters,
                       "tiles_per_gpu": 1, "decimated_grid": info["nx_sub"], "kernel_band": info["band_x"],
                       "kernel_transforms_per_stack": Kt, "computed_focus_stacks": Ft,
                       "ilt": ILT, "l2": "flushed between steps (256 MiB write, untimed)",
                       "parallelism": f"tiles sharded over {world} rank(s); NCCL all-reduce of the per-iteration "
                                      f"global cost vector once per step (no tile data crosses GPUs)"},
            "roofline": {"bound": "fp32", "kernel": top, "achieved": achieved, "peak": peak_fp32,
                         "unit": "TFLOP/s", "frac": achieved / peak_fp32 if peak_fp32 else None,
                         "traffic": _ncu_traffic(top)[0],
                         "traffic_source": _ncu_traffic(top)[1],
                         "peak_source": "measured on-box FFMA microbenchmark (lithogpu_fp32_peak)",
                         "flops_per_launch": top_flops, "algorithmic_bytes_per_launch": top_bytes,
                         "kernel_ms": top_ms,
                         "hbm_gbs_algorithmic": top_bytes / (top_ms * 1e-3) / 1e9,
                         "hbm_peak_gbs": _peaks().get("hbm_gbs"),
                         "frac_hbm": (top_bytes / (top_ms * 1e-3) / 1e9 / _peaks()["hbm_gbs"])
                         if _peaks().get("hbm_gbs") else None,
                         "bound_note": "FP32-pipe / issue bound (FFT butterflies): the band-limited algorithm moves "
                                       "~30x fewer bytes than a full-grid design; HBM view in hbm_* / frac_hbm",
                         "kernel_share": shares, "kernel_ms_avg": kernel_ms,
                         "instrumented_iter_ms": iter_ms_prof},
            "cpu_baseline": cpu,
            "reference_cufftw": cufftw,
            "in_graph": _in_graph_timeline(args.config, top, top_flops, peak_fp32) if world == 1 else None,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
            "final_cost": [float(final_cost[0]), float(final_cost[-1])] if len(final_cost) else None,
            "aerial_c1": aerial,
            "batched_tiles": batched,
        }
        print(json.dumps(result), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    return result


def _raster_to(ctx, grid, xy, starts, out_dev):
    import ctypes as C
    from paper_2602_15036_b200._lib import check, lib
    g = grid.c()
    check(lib().lithogpu_rasterize(ctx.handle, C.byref(g), xy.ctypes.data, starts.ctypes.data,
                                   len(starts) - 1, 1.0, out_dev.data_ptr()))


def _get_mask(solver, mask_host):
    from paper_2602_15036_b200._lib import F32, check, lib
    check(lib().lithogpu_ilt_get_tiles(solver._h, None, mask_host.data_ptr(), F32))


def _c1_forward(ctx, stream):
    """C1 (configs[0]): 1024^2 tile, K=8, forward aerial + blur + threshold;
    device-resident, CUDA-event timed.  Mpixel/s."""
    import torch
    import paper_2602_15036_b200 as L
    from paper_2602_15036_b200 import layouts as LY
    grid, polys, ks, _, desc = make_problem("c1", 0)
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
    contours = _contours_c1(ctx, stream, dk, m32, grid)
    return {"workload": desc, "ms_per_image": ms, "mpix_s": grid.nx * grid.ny / (ms * 1e-3) / 1e6,
            "contours": contours,
            "outputs": "aerial f32 + resist f32 + print u8", "l2": "warm (repeated image)"}


def _contours_c1(ctx, stream, dk, m32, grid, n_gauges=4096, radius=20.0):
    """SURVEY §8f rank 1 stage on the C1 resist image: GPU marching squares +
    EPE gauges (device-resident field, host-synchronised result sizes, as the
    API returns them) against the reference contour.cpp on one host core."""
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
    # evaluate_epe (opc.cpp:140-151) over a batch of 8 MEEF-style probe masks, fused on the device
    m64 = m32.double()
    probes = torch.stack([torch.roll(m64, shifts=k % 3, dims=k % 2) for k in range(8)])
    probes[:, :16, :] = 0.0
    probes[:, -16:, :] = 0.0
    probes[:, :, :16] = 0.0
    probes[:, :, -16:] = 0.0
    ph = probes.cpu().numpy()
    L.evaluate_epe(ph, dk, gauges, 1.0, 2.0, ILT["threshold"], radius)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L.evaluate_epe(ph, dk, gauges, 1.0, 2.0, ILT["threshold"], radius)
    out["gpu_ms_evaluate_epe_per_mask"] = (time.perf_counter() - t0) / len(ph) * 1e3
    out["evaluate_epe_batch"] = len(ph)
    try:
        from oracle import refpy as R
        if R.available():
            # the reference pipeline on one probe (image_socs -> gaussian_blur -> contours -> EPE)
            ks = dk.kernels if hasattr(dk, "kernels") else None
            R.set_threads(1)
            if ks is not None:
                t0 = time.perf_counter()
                I = R.image_socs(ph[0], ks.weights[0], ks.support, ks.values[0])
                rr = R.gaussian_blur(I, 2.0, 1.0)
                R.marching_squares(rr, ILT["threshold"])
                R.measure_epe(gauges, radius)
                out["ref_cpu_ms_evaluate_epe_per_mask"] = (time.perf_counter() - t0) * 1e3
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


def _batched_ilt(ctx, stream, dk, target32, theta0, prm, iters, tiles=8):
    """Same C2 tile replicated `tiles` times in one launch sequence
    (blockIdx.z = tile): the chip-scale regime (C5 puts 32 tiles on each GPU)
    where the imaging kernels fill all SMs.  Tile-iterations/s on one GPU."""
    import torch
    import paper_2602_15036_b200 as L
    solver = L.IltSolver(dk, prm, tiles, "f32", ctx)
    tg = target32.expand(tiles, -1, -1).contiguous()
    th = theta0.expand(tiles, -1, -1).contiguous()
    cost = torch.zeros((iters, tiles), dtype=torch.float64, device=target32.device)
    for _ in range(3):
        solver.set_tiles(tg, th)
        solver.run_device(iters, cost)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record(stream)
    for _ in range(reps):
        solver.set_tiles(tg, th)
        solver.run_device(iters, cost)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    solver.close()
    return {"tiles_per_gpu": tiles, "ms_per_step": ms, "tile_iter_s": tiles * iters / (ms * 1e-3),
            "note": f"{tiles} C2 tiles batched per launch, {iters} iterations per step"}


def _ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum of `kernel` (per launch) from
    the newest committed `ncu --set full` capture summary (profiles/*_ncu.json,
    tools/ncu_summarize.py).  ncu flushes caches before each replay, so this
    counts the L2-resident intermediates a warm step never takes to HBM."""
    import glob
    best = None
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu.json"))):
        try:
            caps = json.load(open(p)).get("full_captures", {})
        except Exception:
            continue
        c = caps.get("fk_" + kernel) or caps.get(kernel)
        if c and c.get("dram_bytes") is not None:
            best = (c["dram_bytes"], f"{os.path.basename(p)} ({c.get('kernel')}, grid {c.get('grid')})")
    return best if best else (None, None)


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def _ref_problem(cfg_name):
    import paper_2602_15036_b200 as L
    grid, polys, ks, iters, desc = make_problem(cfg_name, 0)
    from oracle import refpy as R
    target = R.rasterize(polys, grid.nx, grid.ny, grid.pitch_nm, grid.origin_x_nm, grid.origin_y_nm, 1.0)
    return grid, ks, target, iters, desc


def _cpu_baseline(cfg_name, n_iter=2):
    """Reference CPU implementation (oracle/_ref) on a bounded sample."""
    from oracle import refpy as R
    if not R.available():
        return {"value": None, "unit": "tile-iter/s", "cores": 0, "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    grid, ks, target, iters, desc = _ref_problem(cfg_name)
    cores = os.cpu_count() or 1
    R.set_threads(cores)
    theta = ((2 * target - 1) * (2.0 / ILT["mask_steepness"])).copy()
    F = ks.weights.shape[0]
    prm = [ILT["mask_steepness"], ILT["resist_beta"], ILT["threshold"], ILT["resist_sigma_nm"], ILT["dose"],
           ILT["step"]]
    t0 = time.perf_counter()
    for _ in range(n_iter):
        R.ilt_iteration(theta, target, ks.weights, ks.support, ks.values, [1.0 / F] * F, prm, grid.pitch_nm)
    dt = time.perf_counter() - t0
    return {"value": n_iter / dt, "unit": "tile-iter/s", "cores": cores, "kind": "reference",
            "sample": f"{n_iter} ILT iterations of the {grid.nx}x{grid.ny} tile (K={ks.weights.shape[1]}, F={F}) "
                      f"through the unmodified reference image_socs/gaussian_blur/fft2 (fp64, FFT shim, "
                      f"{cores} OpenMP threads), {dt:.1f} s"}


def _in_graph_timeline(cfg_name, top, top_flops, peak):
    """Per-kernel durations inside the replayed CUDA graph (tools/trace.py:
    first-CTA start to last-warp end from %globaltimer stamps, no per-launch
    events breaking the graph), and the dominant kernel's roofline fraction on
    that duration beside the event-timed one."""
    try:
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "trace.py"), "--config", cfg_name],
                           cwd=ROOT, capture_output=True, text=True, timeout=300)
        d = json.loads(r.stdout.strip().splitlines()[-1])
        per = d["per_kernel"]
        us = per.get(top, {}).get("dur_us")
        out = {"per_iter_us": d["per_iter_us"], "kernel_us": {k: v["dur_us"] for k, v in per.items()},
               "gap_us": {k: v["gap_before_us"] for k, v in per.items()}}
        if us:
            out.update({"top_kernel": top, "achieved_tflops": top_flops / (us * 1e-6) / 1e12,
                        "frac": top_flops / (us * 1e-6) / 1e12 / peak if peak else None})
        return out
    except Exception as e:
        return {"unavailable": str(e)[:200]}


def _cufftw_baseline(cfg_name, n_iter=2):
    """The unmodified reference with its FFTW calls on NVIDIA cuFFTW (library
    GPU FFTs; the reference algorithm, host memory, a plan per fft2 call):
    the naive GPU port the hand-written path is measured against.  Run in a
    subprocess so the two reference builds never share one process."""
    code = (
        "import json, sys, time, numpy as np; sys.path.insert(0, '.');"
        "import bench; from oracle import refpy as R; R.use_variant('cufftw');"
        "assert R.available();"
        f"g, ks, t, it, d = bench._ref_problem('{cfg_name}');"
        "th = ((2 * t - 1) * (2.0 / bench.ILT['mask_steepness'])).copy(); F = ks.weights.shape[0];"
        "prm = [bench.ILT[k] for k in ('mask_steepness', 'resist_beta', 'threshold', 'resist_sigma_nm', 'dose', 'step')];"
        "R.ilt_iteration(th, t, ks.weights, ks.support, ks.values, [1.0 / F] * F, prm, g.pitch_nm);"
        "t0 = time.perf_counter();"
        f"[R.ilt_iteration(th, t, ks.weights, ks.support, ks.values, [1.0 / F] * F, prm, g.pitch_nm) for _ in range({n_iter})];"
        f"dt = (time.perf_counter() - t0) / {n_iter};"
        "print(json.dumps({'value': 1.0 / dt, 'unit': 'tile-iter/s', 'ms_per_iteration': dt * 1e3}))")
    try:
        r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
        out = json.loads(r.stdout.strip().splitlines()[-1])
        out["sample"] = (f"{n_iter} ILT iterations (after 1 warm-up) of the same tile through the unmodified "
                         "reference with FFTW resolved by cuFFTW (GPU FFTs on host buffers, fp64)")
        return out
    except Exception as e:  # optional data point
        return {"unavailable": str(e)[:200]}


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
    prm = [ILT["mask_steepness"], ILT["resist_beta"], ILT["threshold"], ILT["resist_sigma_nm"], ILT["dose"],
           ILT["step"]]
    theta = ((2 * target - 1) * (2.0 / ILT["mask_steepness"])).copy()

    def step():  # bounded sample: one ILT iteration of the tile per step
        R.ilt_iteration(theta, target, ks.weights, ks.support, ks.values, [1.0 / F] * F, prm, grid.pitch_nm)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    ms = dt / args.steps * 1e3
    value = 1.0 / (ms / 1e3)
    res = {"impl": "reference", "metric": f"ILT tile-iterations/s ({desc})", "value": value,
           "unit": "tile-iter/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic (same seeded layout and kernels as the GPU arm)",
           "config": {"workload": desc, "tile": grid.nx, "K": int(ks.weights.shape[1]), "F": F,
                      "iterations_per_step": 1, "note": "one ILT iteration per step (bounded CPU sample)"},
           "cpu_baseline": {"value": value, "unit": "tile-iter/s", "cores": cores, "kind": "reference",
                            "sample": "1 ILT iteration per step of the same tile, unmodified reference "
                                      "sources (oracle/_ref), OpenMP FFT shim"},
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
        run_c5(args, world, rank, local)
        return
    run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
