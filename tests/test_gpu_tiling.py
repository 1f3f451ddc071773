"""Halo-padded chip tiling on the GPU.

- Tile rasters: every GPU tile raster is bitwise the matching sub-block of
  the REFERENCE rasterize_layer (oracle/_ref, raster.cpp:53-95) of the
  halo-extended chip window.
- Tile images: each tile is a closed cyclic window imaged exactly as the
  reference images a make_window window (opc.cpp:97-112 -> image_socs,
  imaging.cpp:218-241): GPU aerial / resist of the tile == oracle image of
  the same window at 1e-4.  The core-vs-larger-window difference (the halo
  truncation of the hard-pupil tail) is the same number for the GPU and the
  oracle, and is recorded here.
- ChipIlt over a seeded chip: stitched cores of the sharded batched run are
  bitwise the stitched cores of independent one-tile runs.
"""
import os

import numpy as np
import pytest

import paper_2602_15036_b200 as L
from paper_2602_15036_b200 import chip, layouts as LY
from oracle import oracle as O
from oracle import refpy as R

pytestmark = pytest.mark.gpu


def rel_linf(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    s = np.abs(b).max()
    return float(np.abs(a - b).max() / (s if s > 0 else 1.0))


def euv():
    return L.OpticalModel(source=L.make_annular_source(0.4, 0.8, 21))


@pytest.mark.parametrize("curvy", [False, True])
def test_gpu_tile_rasters_bitwise_vs_reference_window(ctx, curvy):
    tl = LY.chip_tiling(256, 3, 2, 64, origin_nm=(-37.0, 18.0))
    polys = LY.chip_layout(tl, seed=9, curvilinear_layout=curvy)
    ext = tl.extended_grid()
    full = R.rasterize(polys, ext.nx, ext.ny, ext.pitch_nm, ext.origin_x_nm, ext.origin_y_nm, 1.0)
    bb = LY.polygon_bboxes(polys)
    tiles = []
    for t in range(len(tl)):
        g = tl.tile_grid(t)
        got = L.rasterize_layer(tl.tile_polygons(polys, t, bboxes=bb), g, 1.0, ctx)
        i, j = tl.tile_ij(t)
        sub = full[j * tl.core:j * tl.core + tl.n, i * tl.core:i * tl.core + tl.n]
        # bitwise the reference rasterizer on the same tile grid
        want = R.rasterize(polys, g.nx, g.ny, g.pitch_nm, g.origin_x_nm, g.origin_y_nm, 1.0)
        assert np.array_equal(got, want), t
        if curvy:
            # all-angle clip intersections round differently for another
            # window origin: the reference itself is shift-invariant only to
            # fp64 rounding (x = (p.x/dbu - origin)/pitch, raster.cpp:68-69)
            assert np.abs(got - sub).max() <= 1e-10, t
        else:
            assert np.array_equal(got, sub), t  # Manhattan: every intersection exact
        tiles.append(got)
    h = tl.halo
    st = tl.stitch(np.stack(tiles))
    if curvy:
        assert np.abs(st - full[h:h + tl.chip.ny, h:h + tl.chip.nx]).max() <= 1e-10
    else:
        assert np.array_equal(st, full[h:h + tl.chip.ny, h:h + tl.chip.nx])


def test_tile_images_vs_oracle_and_halo_truncation(ctx):
    """GPU tile image == oracle image of the same cyclic window (1e-4); the
    core of the tile vs the same region of a 4x larger window: the GPU's
    difference equals the oracle's (the truncation is the window semantics,
    not an error of the GPU path)."""
    O.set_threads(os.cpu_count() or 1)
    core, W = 256, 1024
    model = euv()
    big_g = L.Grid(W, W, 1.0)
    polys = LY.line_space_contacts(W, W, seed=3)
    big = O.rasterize(polys, W, W)
    ks_big = L.build_socs_kernels(model, big_g, [0.0], k_fixed=8)
    I_big = O.image_socs(big, ks_big.weights[0], ks_big.support, ks_big.values[0])
    R_big = O.gaussian_blur(I_big, 2.0, 1.0)
    c0 = (W - core) // 2
    halo = LY.optical_halo_px(model.wavelength_nm, model.na, 1.0, 2.0)
    assert halo == 128
    rows = []
    for h in (64, halo):
        n = core + 2 * h
        x0 = c0 - h
        tile = np.ascontiguousarray(big[x0:x0 + n, x0:x0 + n])
        # the GPU rasterizes the tile window itself (origin x0): bitwise the sub-block
        g = L.Grid(n, n, 1.0, float(x0), float(x0))
        assert np.array_equal(L.rasterize_layer(polys, g, 1.0, ctx), tile)
        ks = L.build_socs_kernels(model, L.Grid(n, n, 1.0), [0.0], k_fixed=8)
        dk = L.DeviceKernels(ks, "f32", ctx)
        out = dk.image(tile, sigma_nm=2.0, want=("intensity", "resist"))
        I_t = O.image_socs(tile, ks.weights[0], ks.support, ks.values[0])
        R_t = O.gaussian_blur(I_t, 2.0, 1.0)
        assert rel_linf(out["intensity"], I_t) <= 1e-4
        assert rel_linf(out["resist"], R_t) <= 1e-4
        cs = np.s_[h:h + core, h:h + core]
        bs = np.s_[c0:c0 + core, c0:c0 + core]
        e_gpu = rel_linf(out["resist"][cs], R_big[bs])
        e_orc = rel_linf(R_t[cs], R_big[bs])
        assert abs(e_gpu - e_orc) <= 1e-4, (h, e_gpu, e_orc)
        rows.append((h, e_orc))
    # recorded bound of the hard-pupil truncation
    for h, e in rows:
        assert e < 0.06, rows
    print("halo truncation (halo px, core-vs-window rel Linf):", rows)


def test_chip_ilt_stitched_cores(ctx):
    """ChipIlt over one seeded chip (2x2 tiles of 256 = 128 core + 2x64 halo),
    tiles batched in one launch sequence: stitched final-mask cores and the
    per-iteration global cost equal independent one-tile runs."""
    tl = LY.chip_tiling(256, 2, 2, 64)
    polys = LY.chip_layout(tl, seed=4)
    ks = L.build_socs_kernels(euv(), L.Grid(tl.n, tl.n, 1.0), [-40.0, 0.0, 40.0], k_fixed=8)
    prm = L.IltParams(step=0.5, focus_weights=[0.25, 0.5, 0.25])
    ci = chip.ChipIlt(tl, polys, ks, prm, ctx)
    res = ci.run(3, want_mask=True)
    masks = []
    tot = np.zeros(3)
    for t in range(len(tl)):
        g = tl.tile_grid(t)
        raster = L.rasterize_layer(tl.tile_polygons(polys, t), g, 1.0, ctx)
        s = L.IltSolver(ks, prm, 1, "f32", ctx)
        s.set_tiles(raster[None].astype(np.float32))
        tot += s.run(3)[:, 0]
        masks.append(s.get_tiles()[1][0])
        s.close()
    assert np.array_equal(tl.stitch(res.mask), tl.stitch(np.stack(masks)))
    assert np.abs(res.cost - tot).max() <= 1e-9 * np.abs(tot).max()


def test_ilt_get_window_stitches_chip_mask(ctx):
    """lithogpu_ilt_get_window writes each tile's core straight into the
    stitched chip mask (host and device destinations) == stitch(get_tiles)."""
    import torch
    tl = LY.chip_tiling(192, 2, 2, 32)
    polys = LY.chip_layout(tl, seed=6)
    ks = L.build_socs_kernels(euv(), L.Grid(tl.n, tl.n, 1.0), [0.0], k_fixed=6)
    ci = chip.ChipIlt(tl, polys, ks, L.IltParams(step=0.5, focus_weights=[1.0]), ctx)
    ci.run(2)
    want = tl.stitch(ci.solver.get_tiles(dtype=0)[1])
    host = np.zeros((tl.chip.ny, tl.chip.nx), np.float32)
    dev = torch.zeros((tl.chip.ny, tl.chip.nx), dtype=torch.float32, device="cuda")
    c, h = tl.core, tl.halo
    for t in range(len(tl)):
        i, j = tl.tile_ij(t)
        ci.solver.get_window(t, h, h, c, c, out=host[j * c:(j + 1) * c, i * c:(i + 1) * c])
        ci.solver.get_window(t, h, h, c, c, out=dev[j * c:(j + 1) * c, i * c:(i + 1) * c])
    ctx.synchronize()
    assert np.array_equal(host, want)
    assert np.array_equal(dev.cpu().numpy(), want)
    # stream-ordered variant into page-locked host memory; pageable memory is a usage error
    pinned = torch.zeros((tl.chip.ny, tl.chip.nx), dtype=torch.float32).pin_memory()
    for t in range(len(tl)):
        i, j = tl.tile_ij(t)
        ci.solver.get_window(t, h, h, c, c, out=pinned[j * c:(j + 1) * c, i * c:(i + 1) * c], async_=True)
    ctx.synchronize()
    assert np.array_equal(pinned.numpy(), want)
    with pytest.raises(L.api.LithoUsageError):
        ci.solver.get_window(0, h, h, c, c, out=host[:c, :c], async_=True)
