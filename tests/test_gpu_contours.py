"""GPU marching squares + EPE gauges against the
reference itself (oracle/_ref: marching_squares contour.cpp:58-168,
measure_epe contour.cpp:181-201 over bvh.cpp:241-273).  Bar: bitwise equal
loops (order, start point, every fp64 coordinate) and EPE records."""
import numpy as np
import pytest

import paper_2602_15036_b200 as L
from oracle import refpy as R

pytestmark = pytest.mark.gpu


def gauss_field(nx, ny, seed, n=12, border=4):
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:ny, 0:nx].astype(np.float64)
    f = np.zeros((ny, nx))
    for _ in range(n):
        cx, cy = rng.uniform(border + 3, nx - border - 3), rng.uniform(border + 3, ny - border - 3)
        s = rng.uniform(2.0, 0.08 * min(nx, ny) + 3)
        f += rng.uniform(0.3, 1.0) * np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / (2 * s * s))
    f[:border, :] = f[-border:, :] = 0.0
    f[:, :border] = f[:, -border:] = 0.0
    return f


def same_contours(got, field, thr, grid):
    st, xs, ys = R.marching_squares(field, thr, grid.pitch_nm, grid.origin_x_nm, grid.origin_y_nm)
    assert np.array_equal(got.loop_start, st)
    assert np.array_equal(got.xs, xs) and np.array_equal(got.ys, ys)
    return st


@pytest.mark.parametrize("nx,ny,pitch,ox,oy,thr,seed", [
    (64, 48, 1.0, 0.0, 0.0, 0.3, 1),
    (200, 160, 0.5, -12.25, 7.5, 0.25, 2),
    (512, 512, 1.0, 3.0, -5.0, 0.45, 3),
    (333, 257, 2.0, 0.0, 0.0, 0.6, 4),
])
def test_marching_squares_bit_exact(ctx, nx, ny, pitch, ox, oy, thr, seed):
    f = gauss_field(nx, ny, seed)
    g = L.Grid(nx, ny, pitch, ox, oy)
    got = L.marching_squares(f, g, thr, ctx)
    st = same_contours(got, f, thr, g)
    assert len(st) > 1


def test_marching_squares_saddles_and_exact_threshold(ctx):
    """checkerboard saddles (both center cases) and node values equal to the
    threshold (the reference's +eps perturbation)."""
    rng = np.random.default_rng(9)
    f = np.zeros((40, 40))
    f[4:36, 4:36] = rng.integers(0, 3, (32, 32)).astype(np.float64) * 0.5  # values 0, .5, 1
    g = L.Grid(40, 40, 1.0)
    for thr in (0.5, 0.25, 0.75):
        same_contours(L.marching_squares(f, g, thr, ctx), f, thr, g)


def test_marching_squares_resist_image(ctx):
    """contours of a GPU resist image (C1-like tile) at the resist threshold."""
    from paper_2602_15036_b200 import layouts as LY
    n = 256
    grid = L.Grid(n, n, 1.0)
    polys = LY.line_space_contacts(n, n, seed=5)
    mask = L.rasterize_layer(polys, grid, 1.0, ctx)
    model = L.OpticalModel(source=L.make_annular_source(0.4, 0.8, 21))
    ks = L.build_socs_kernels(model, grid, [0.0], k_fixed=8)
    dk = L.DeviceKernels(ks, "f64", ctx)
    res = dk.image(mask, sigma_nm=2.0, want=("resist",))["resist"]
    res = np.asarray(res, np.float64).copy()
    res[:2, :] = res[-2:, :] = 0.0  # closed contours (open chains throw in the reference)
    res[:, :2] = res[:, -2:] = 0.0
    got = L.marching_squares(res, grid, 0.25, ctx)
    same_contours(got, res, 0.25, grid)
    # EPE gauges on the target edges of the first few lines
    rng = np.random.default_rng(3)
    gauges = np.column_stack([rng.uniform(8, n - 8, 300), rng.uniform(8, n - 8, 300),
                              np.zeros(300), np.zeros(300)])
    ang = rng.uniform(0, 2 * np.pi, 300)
    gauges[:, 2], gauges[:, 3] = np.cos(ang), np.sin(ang)
    gauges[:100, 2], gauges[:100, 3] = 1.0, 0.0  # axis-aligned normals (Manhattan targets)
    for radius in (5.0, 20.0):
        epe, op = L.measure_epe(got, gauges, radius)
        R.marching_squares(res, 0.25, 1.0, 0.0, 0.0)
        re, ro = R.measure_epe(gauges, radius)
        assert np.array_equal(op, ro)
        assert np.array_equal(epe, re)


def test_epe_random_gauges(ctx):
    f = gauss_field(300, 220, 11)
    g = L.Grid(300, 220, 1.0, -4.0, 9.0)
    got = L.marching_squares(f, g, 0.35, ctx)
    same_contours(got, f, 0.35, g)
    rng = np.random.default_rng(12)
    k = 2000
    ang = rng.uniform(0, 2 * np.pi, k)
    gauges = np.column_stack([rng.uniform(-10, 310, k), rng.uniform(0, 240, k), np.cos(ang), np.sin(ang)])
    for radius in (0.0, 3.0, 15.0, 60.0):
        epe, op = L.measure_epe(got, gauges, radius)
        re, ro = R.measure_epe(gauges, radius)
        assert np.array_equal(op, ro), radius
        assert np.array_equal(epe, re), radius


def test_contour_edge_cases(ctx):
    g = L.Grid(30, 30, 1.0)
    empty = L.marching_squares(np.zeros((30, 30)), g, 0.5, ctx)
    assert len(empty.loops) == 0 and len(empty.xs) == 0
    epe, op = L.measure_epe(empty, np.array([[10.0, 10.0, 1.0, 0.0]]), 5.0)
    assert op.tolist() == [True] and epe.tolist() == [0.0]
    one = L.marching_squares(np.ones((1, 30)), L.Grid(30, 1, 1.0), 0.5, ctx)
    assert len(one.loops) == 0
    bad = np.zeros((30, 30))
    bad[5, 5] = np.nan
    with pytest.raises(ValueError):
        L.marching_squares(bad, g, 0.5, ctx)
    openf = np.zeros((30, 30))
    openf[10:20, 0:15] = 1.0  # touches the border: open chain
    with pytest.raises(RuntimeError):
        L.marching_squares(openf, g, 0.5, ctx)
    with pytest.raises(RuntimeError):
        R.marching_squares(openf, 0.5)


def test_evaluate_epe_fused_batch(ctx):
    """evaluate_epe (opc.cpp:140-151) on the device for a batch of masks (MEEF
    probe style): bit-identical to the unfused GPU steps, and equal to the
    reference pipeline (image_socs -> gaussian_blur -> marching_squares ->
    measure_epe, oracle/_ref) to fp64 FFT rounding."""
    from paper_2602_15036_b200 import layouts as LY
    n = 192
    grid = L.Grid(n, n, 1.0)
    base = L.rasterize_layer(LY.line_space_contacts(n, n, seed=8), grid, 1.0, ctx)
    base[:16, :] = base[-16:, :] = 0.0
    base[:, :16] = base[:, -16:] = 0.0
    masks = np.stack([base, np.roll(base, 1, axis=1), np.roll(base, -2, axis=0)])
    model = L.OpticalModel(source=L.make_annular_source(0.4, 0.8, 21))
    ks = L.build_socs_kernels(model, grid, [-40.0, 0.0, 40.0], k_fixed=6)
    rng = np.random.default_rng(21)
    k = 400
    ang = rng.choice([0.0, np.pi / 2, np.pi, 1.5 * np.pi], k)
    gauges = np.column_stack([rng.uniform(20, n - 20, k), rng.uniform(20, n - 20, k), np.cos(ang), np.sin(ang)])
    dk = L.DeviceKernels(ks, "f64", ctx)
    epe, op, res = L.evaluate_epe(masks, dk, gauges, 1.0, 2.0, 0.25, 12.0, focus=1, want_resist=True)
    assert epe.shape == (3, k) and res.shape == (3, n, n)
    for t in range(3):
        r1 = np.asarray(dk.image(masks[t], focus=1, sigma_nm=2.0, want=("resist",))["resist"])
        assert np.array_equal(res[t], r1)
        cs = L.marching_squares(r1, grid, 0.25, ctx)
        e1, o1 = L.measure_epe(cs, gauges, 12.0)
        assert np.array_equal(epe[t], e1) and np.array_equal(op[t], o1)
        # reference pipeline
        I = R.image_socs(masks[t], ks.weights[1], ks.support, ks.values[1])
        rr = R.gaussian_blur(I, 2.0, 1.0)
        assert np.abs(rr - r1).max() <= 1e-10 * np.abs(rr).max()
        R.marching_squares(rr, 0.25)
        re, ro = R.measure_epe(gauges, 12.0)
        assert np.array_equal(ro, op[t])
        assert np.abs(re - epe[t]).max() < 1e-6
    assert op.sum() < op.size  # most gauges see an edge
    # device-resident masks (torch CUDA tensor) give the same records
    import torch
    e_d, o_d = L.evaluate_epe(torch.from_numpy(masks).cuda(), dk, gauges, 1.0, 2.0, 0.25, 12.0, focus=1)
    assert np.array_equal(e_d, epe) and np.array_equal(o_d, op)
    bad = masks.copy()
    bad[0, 5, 5] = np.nan
    with pytest.raises(ValueError):
        L.evaluate_epe(bad, dk, gauges, 1.0, 2.0, 0.25, 12.0, focus=1)
