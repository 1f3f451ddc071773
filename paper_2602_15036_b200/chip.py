"""Chip-scale ILT over halo-padded tiles, sharded across ranks (one process
per GPU).  SURVEY.md §8e: tiles are independent (cyclic convolution inside
each halo-padded window), so the only data-path exchange is the all-reduce of
the global ILT cost and convergence scalars (per iteration, batched into one
call per graph-replayed segment of iterations).

Torch is plumbing here: torch.distributed (NCCL on GPUs, gloo in CPU tests)
for the scalar all-reduce; all imaging / adjoint work runs in liblithogpu.so.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np


def shard(n_tiles: int, world: int, rank: int) -> range:
    """Contiguous block of tiles for `rank` (sizes differ by at most one)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("shard: bad world/rank")
    base, extra = divmod(n_tiles, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def allreduce_scalars(cost, gmax, group=None):
    """Global ILT cost (sum over tiles / ranks) and convergence scalar (max
    |dL/dtheta|) — the only cross-GPU traffic of the tiled ILT."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        host = cost.is_cuda and dist.get_backend(group) == "gloo"  # gloo: reduce host copies

        def red(t, op):
            if host:
                h = t.cpu()
                dist.all_reduce(h, op=op, group=group)
                t.copy_(h)
            else:
                dist.all_reduce(t, op=op, group=group)
        red(cost, dist.ReduceOp.SUM)
        if gmax is not None:
            red(gmax, dist.ReduceOp.MAX)
    return cost, gmax


@dataclass
class ChipResult:
    cost: np.ndarray           # [iters] global cost per iteration
    gmax: np.ndarray           # [iters] global max |dL/dtheta|
    tiles: range               # this rank's tiles
    mask: Optional[np.ndarray] = None  # [n_mine, n, n] final masks (if requested)


class ChipIlt:
    """ILT of this rank's shard of a tiled chip layout, tiles batched into one
    device launch sequence (blockIdx.z = tile)."""

    def __init__(self, tiling, polys: Sequence[np.ndarray], kernels, params, ctx, rank: int = 0,
                 world: int = 1, dbu_per_nm: float = 1.0):
        import torch

        from . import api
        from .layouts import polygon_arrays, polygon_bboxes
        self.tiling = tiling
        self.rank, self.world = rank, world
        self.mine = shard(len(tiling), world, rank)
        self.ctx = ctx
        n = tiling.n
        dev = torch.device("cuda", ctx.device)
        self.target = torch.empty((len(self.mine), n, n), dtype=torch.float64, device=dev)
        bb = polygon_bboxes(polys)
        for j, t in enumerate(self.mine):
            g = tiling.tile_grid(t)
            tp = tiling.tile_polygons(polys, t, dbu_per_nm, bboxes=bb)
            xy, st = polygon_arrays(tp)
            _raster(ctx, g, xy, st, self.target[j], dbu_per_nm)
        # a rank with an empty shard (world > tiles) runs no solver and
        # contributes zero cost / gmax to the all-reduce
        self.solver = api.IltSolver(kernels, params, len(self.mine), "f32", ctx) if len(self.mine) else None
        self.target32 = self.target.float().contiguous()
        if self.solver is not None:
            self.solver.set_tiles(self.target32)

    def run(self, iters: int, want_mask: bool = False, sync_every: Optional[int] = None,
            tol: Optional[float] = None) -> ChipResult:
        """`iters` ILT iterations of this rank's tiles (see segmented_ilt)."""
        if self.solver is None:
            def run_segment(k, cost, gmax):  # empty shard: zero partials
                cost.zero_()
                gmax.zero_()
            n_tiles = 1
        else:
            run_segment, n_tiles = self.solver.run_device, self.solver.n_tiles
        gl_cost, gl_gmax = segmented_ilt(run_segment, iters, n_tiles, sync_every, tol, self.target.device)
        res = ChipResult(gl_cost, gl_gmax, self.mine)
        if want_mask:
            n = self.tiling.n
            res.mask = self.solver.get_tiles()[1] if self.solver is not None else np.zeros((0, n, n))
        return res


def segmented_ilt(run_segment, iters: int, n_tiles: int, sync_every: Optional[int] = None,
                  tol: Optional[float] = None, device="cpu"):
    """Drive `iters` ILT iterations as graph-replayed segments of `sync_every`
    (default: all of them).  run_segment(k, cost[k, n_tiles], gmax[k, n_tiles])
    enqueues k iterations of this rank's tiles.  After each segment the
    per-iteration global cost (sum over tiles and ranks) and max |dL/dtheta|
    (max over tiles and ranks) of the whole segment are all-reduced in one
    call each: no blocking collective per iteration on the critical path.
    With `tol`, stop after the first segment whose last global relative cost
    change is <= tol.  Returns (global cost [done], global gmax [done])."""
    import torch
    seg = max(1, min(iters, sync_every or iters))
    cost = torch.zeros((iters, n_tiles), dtype=torch.float64, device=device)
    gmax = torch.zeros((iters, n_tiles), dtype=torch.float64, device=device)
    gl_cost = torch.zeros(iters, dtype=torch.float64, device=device)
    gl_gmax = torch.zeros(iters, dtype=torch.float64, device=device)
    done = 0
    while done < iters:
        k = min(seg, iters - done)
        run_segment(k, cost[done:done + k], gmax[done:done + k])
        gl_cost[done:done + k] = cost[done:done + k].sum(dim=1)
        gl_gmax[done:done + k] = gmax[done:done + k].amax(dim=1)
        c, g = allreduce_scalars(gl_cost[done:done + k].clone(), gl_gmax[done:done + k].clone())
        gl_cost[done:done + k] = c
        gl_gmax[done:done + k] = g
        done += k
        if tol is not None and done >= 2:
            c2 = gl_cost[done - 2:done].cpu().numpy()
            if abs(c2[1] - c2[0]) <= tol * abs(c2[0]):
                break
    return gl_cost[:done].cpu().numpy(), gl_gmax[:done].cpu().numpy()


def _raster(ctx, grid, xy, starts, out_dev, dbu):
    import ctypes as C

    from ._lib import check, lib
    g = grid.c()
    check(lib().lithogpu_rasterize(ctx.handle, C.byref(g), xy.ctypes.data, starts.ctypes.data,
                                   len(starts) - 1, dbu, out_dev.data_ptr()))
