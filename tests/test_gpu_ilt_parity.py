"""GPU parity of the ILT gradient at the north-star tolerance (rel L-inf
<= 1e-4, fp32) on the shapes bench.py measures, through the C ABI
(lithogpu_ilt_gradient: cost and dcost/dtheta at the current theta, theta
unchanged) against the fp64 CPU oracle (oracle/litho_oracle.c
orc_ilt_iteration, whose W = 1 reduction is the reference
intensity_gradient, ai.cpp:11-42, and whose new parts are pinned by central
differences in tests/test_oracle.py).

Also: the CUDA-graph path (context on a non-default stream: capture on the
second identical call, replay afterwards) against the oracle trajectory,
with a second solver of another resist sigma and an image() call interleaved
between replays (shared Gaussian tables, mask spectra and graph keys).
"""
import os

import numpy as np
import pytest

import paper_2602_15036_b200 as L
from paper_2602_15036_b200 import layouts as LY
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-4
ILT = dict(mask_steepness=4.0, resist_beta=30.0, threshold=0.25, resist_sigma_nm=2.0, dose=1.0, step=0.5)
PRM = [ILT[k] for k in ("mask_steepness", "resist_beta", "threshold", "resist_sigma_nm", "dose", "step")]


def rel_linf(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    s = np.abs(b).max()
    return float(np.abs(a - b).max() / (s if s > 0 else 1.0))


@pytest.fixture(scope="module", autouse=True)
def oracle_threads():
    O.set_threads(os.cpu_count() or 1)


def euv():
    return L.OpticalModel(source=L.make_annular_source(0.4, 0.8, 21))


def bench_tile(n, seed, curvilinear=False):
    """The bench's inputs: a seeded layout raster as target, theta0 from it."""
    gen = LY.curvilinear if curvilinear else LY.line_space_contacts
    target = O.rasterize(gen(n, n, seed=seed), n, n)
    theta0 = (2 * target - 1) * (2.0 / ILT["mask_steepness"])
    return target, theta0


def oracle_grad(theta, target, ks, fw):
    th = np.ascontiguousarray(theta, np.float64).copy()
    return O.ilt_iteration(th, target, ks.weights, ks.support, ks.values, fw, PRM, ks.grid.pitch_nm)


# (N, K, foci, name): C2, C3, and smaller shapes of the same plans
SHAPES = [
    (256, 16, (0.0,), "256/K16/F1"),
    (512, 16, (-40.0, 0.0, 40.0), "512/K16/F3"),
    (256, 8, (-40.0, -20.0, 0.0, 20.0, 40.0), "256/K8/F5"),
    (2048, 16, (0.0,), "C2 2048/K16/F1"),
    (2048, 16, (-40.0, -20.0, 0.0, 20.0, 40.0), "C3 2048/K16/F5"),
]


@pytest.mark.parametrize("n,K,foci,name", SHAPES, ids=[s[3] for s in SHAPES])
def test_ilt_gradient_vs_oracle(ctx, n, K, foci, name):
    F = len(foci)
    ks = L.build_socs_kernels(euv(), L.Grid(n, n, 1.0), list(foci), k_fixed=K)
    fw = [1.0 / F] * F
    target, theta0 = bench_tile(n, seed=1000 + n + F)
    # a perturbed theta0 so the mask is not saturated at two levels only
    theta0 = theta0 + np.random.default_rng(n + F).standard_normal(theta0.shape) * 0.25
    solver = L.IltSolver(ks, L.IltParams(focus_weights=fw, **ILT), 1, "f32", ctx)
    solver.set_tiles(target[None], theta0[None])
    cost, grad = solver.gradient()
    c_ref, g_ref = oracle_grad(theta0, target, ks, fw)
    assert abs(cost[0] - c_ref) <= TOL * abs(c_ref), (cost[0], c_ref)
    err = rel_linf(grad[0], g_ref)
    assert err <= TOL, err
    # theta is unchanged by the gradient evaluation
    th, _ = solver.get_tiles()
    assert np.array_equal(th[0], theta0.astype(np.float32).astype(np.float64))


def test_ilt_gradient_c5_batched(ctx):
    """C5 shape (2048^2, K=24, F=3) through the 32-tile batched launch the
    chip bench uses: first, middle and last tile of the batch against the
    oracle; the others bitwise equal to their own one-tile evaluation."""
    n, K, foci, T = 2048, 24, (-40.0, 0.0, 40.0), 32
    F = len(foci)
    fw = [1.0 / F] * F
    ks = L.build_socs_kernels(euv(), L.Grid(n, n, 1.0), list(foci), k_fixed=K, backend="gpu", ctx=ctx)
    dk = L.DeviceKernels(ks, "f32", ctx)
    rng = np.random.default_rng(5)
    tg = np.empty((T, n, n), np.float32)
    th = np.empty((T, n, n), np.float32)
    for t in range(T):
        a, b = bench_tile(n, seed=5000 + t)
        tg[t] = a
        th[t] = b + rng.standard_normal(b.shape) * 0.25
    solver = L.IltSolver(dk, L.IltParams(focus_weights=fw, **ILT), T, "f32", ctx)
    solver.set_tiles(tg, th)
    cost, grad = solver.gradient()
    for t in (0, T // 2, T - 1):
        c_ref, g_ref = oracle_grad(th[t], tg[t], ks, fw)
        assert abs(cost[t] - c_ref) <= TOL * abs(c_ref), (t, cost[t], c_ref)
        err = rel_linf(grad[t], g_ref)
        assert err <= TOL, (t, err)
    one = L.IltSolver(dk, L.IltParams(focus_weights=fw, **ILT), 1, "f32", ctx)
    for t in (1, 7, T - 2):
        one.set_tiles(tg[t:t + 1], th[t:t + 1])
        c1, g1 = one.gradient()
        assert c1[0] == cost[t]
        assert np.array_equal(g1[0], grad[t])


@pytest.mark.slow
def test_ilt_gradient_c4(ctx):
    """C4 shape (curvilinear 4096^2, K=32, F=3; N = 4096 and n = 768 plans)."""
    n, K, foci = 4096, 32, (-40.0, 0.0, 40.0)
    F = len(foci)
    fw = [1.0 / F] * F
    ks = L.build_socs_kernels(euv(), L.Grid(n, n, 1.0), list(foci), k_fixed=K, backend="gpu", ctx=ctx)
    target, theta0 = bench_tile(n, seed=77, curvilinear=True)
    theta0 = theta0 + np.random.default_rng(3).standard_normal(theta0.shape) * 0.25
    solver = L.IltSolver(ks, L.IltParams(focus_weights=fw, **ILT), 1, "f32", ctx)
    solver.set_tiles(target[None], theta0[None])
    cost, grad = solver.gradient()
    c_ref, g_ref = oracle_grad(theta0, target, ks, fw)
    assert abs(cost[0] - c_ref) <= TOL * abs(c_ref), (cost[0], c_ref)
    assert rel_linf(grad[0], g_ref) <= TOL


@pytest.mark.timeout(300)
def test_c4_graph_replays_complete(sctx):
    """Regression: many graph-replayed C4 iterations on a stream (two-warp row
    groups of the n = 768 plan, empty slots of the paired in-focus stack) run
    to completion with a deterministic cost trajectory (a TMA double-buffer
    phase race once hung here)."""
    import torch
    n, K, foci = 4096, 32, (-40.0, 0.0, 40.0)
    ks = L.build_socs_kernels(euv(), L.Grid(n, n, 1.0), list(foci), k_fixed=K, backend="gpu", ctx=sctx)
    target, theta0 = bench_tile(n, seed=5)
    solver = L.IltSolver(ks, L.IltParams(focus_weights=[1.0 / 3] * 3, **ILT), 1, "f32", sctx)
    cost = torch.zeros((50, 1), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    first = None
    for _ in range(12):
        solver.set_tiles(target[None].astype(np.float32), theta0[None].astype(np.float32))
        solver.run_device(50, cost)
        sctx.synchronize()
        c = cost[:, 0].cpu().numpy().copy()
        if first is None:
            first = c
        assert np.array_equal(c, first)
    assert first[-1] < first[0]


def test_ilt_gradient_f64_path(ctx):
    """fp64 (reference-tolerance) path: gradient at 1e-9."""
    n, foci = 64, (-40.0, 0.0, 40.0)
    ks = L.build_socs_kernels(euv(), L.Grid(n, n, 1.0), list(foci), k_fixed=8)
    fw = [0.2, 0.5, 0.3]
    rng = np.random.default_rng(2)
    target = (rng.random((n, n)) > 0.5).astype(np.float64)
    theta0 = rng.standard_normal((n, n)) * 0.5
    solver = L.IltSolver(ks, L.IltParams(focus_weights=fw, **ILT), 1, "f64", ctx)
    solver.set_tiles(target[None], theta0[None])
    cost, grad = solver.gradient()
    c_ref, g_ref = oracle_grad(theta0, target, ks, fw)
    assert abs(cost[0] - c_ref) <= 1e-9 * abs(c_ref)
    assert rel_linf(grad[0], g_ref) <= 1e-9


@pytest.fixture()
def sctx():
    """A context on a non-default stream: the ILT graph capture / replay path
    (ilt_run_impl captures only when ctx->stream != nullptr)."""
    import torch
    c = L.Context(0)
    st = torch.cuda.Stream()
    c.set_stream(st.cuda_stream)
    yield c
    c.synchronize()
    c.close()


def test_ilt_graph_replay_vs_oracle(sctx):
    """eager (1st call), capture (2nd), replay (3rd, 4th): the per-iteration
    cost of every call and the gradient at the final theta against the
    oracle trajectory; a second solver with another resist sigma and an
    intensity-only image() (sigma 0) run between the replays on the same
    kernel stacks."""
    n, foci = 512, (-40.0, 0.0, 40.0)
    F = len(foci)
    fw = [0.25, 0.5, 0.25]
    ks = L.build_socs_kernels(euv(), L.Grid(n, n, 1.0), list(foci), k_fixed=16)
    dk = L.DeviceKernels(ks, "f32", sctx)
    target, theta0 = bench_tile(n, seed=21)
    prm_a = L.IltParams(focus_weights=fw, **dict(ILT, step=0.05))
    prm_b = L.IltParams(focus_weights=fw, **dict(ILT, step=0.05, resist_sigma_nm=3.0))
    sa = L.IltSolver(dk, prm_a, 1, "f32", sctx)
    sb = L.IltSolver(dk, prm_b, 1, "f32", sctx)
    sa.set_tiles(target[None], theta0[None])
    sb.set_tiles(target[None], theta0[None])
    pa = [PRM[0], PRM[1], PRM[2], 2.0, 1.0, 0.05]
    pb = [PRM[0], PRM[1], PRM[2], 3.0, 1.0, 0.05]
    tha = theta0.copy()
    thb = theta0.copy()
    mask = (np.random.default_rng(1).random((n, n)) > 0.5).astype(np.float32)
    want_img = O.image_socs(mask, ks.weights[0], ks.support, ks.values[0])
    for call in range(4):
        ca = sa.run(2)[:, 0]
        img = dk.image(mask, focus=0)["intensity"]  # sigma 0 between the two solvers' graphs
        cb = sb.run(2)[:, 0]
        assert rel_linf(img, want_img) <= TOL
        for j in range(2):
            c_ref, _ = O.ilt_iteration(tha, target, ks.weights, ks.support, ks.values, fw, pa, 1.0)
            assert abs(ca[j] - c_ref) <= TOL * abs(c_ref), ("a", call, j, ca[j], c_ref)
            c_ref, _ = O.ilt_iteration(thb, target, ks.weights, ks.support, ks.values, fw, pb, 1.0)
            assert abs(cb[j] - c_ref) <= TOL * abs(c_ref), ("b", call, j, cb[j], c_ref)
    # gradient at the end of the trajectory, both solvers
    for s, th, p in ((sa, tha, pa), (sb, thb, pb)):
        cost, g = s.gradient()
        t2 = th.copy()
        c_ref, g_ref = O.ilt_iteration(t2, target, ks.weights, ks.support, ks.values, fw, p, 1.0)
        assert abs(cost[0] - c_ref) <= TOL * abs(c_ref)
        assert rel_linf(g[0], g_ref) <= TOL
        # the fp32 theta trajectory stays on the fp64 one
        assert rel_linf(s.get_tiles()[0][0], th) <= TOL


def test_ilt_gradient_device_buffers(sctx):
    """device-resident gradient (torch CUDA tensor) equals the host one."""
    import torch
    n = 256
    ks = L.build_socs_kernels(euv(), L.Grid(n, n, 1.0), [0.0], k_fixed=8)
    target, theta0 = bench_tile(n, seed=3)
    s = L.IltSolver(ks, L.IltParams(focus_weights=[1.0], **ILT), 1, "f32", sctx)
    s.set_tiles(target[None], theta0[None])
    c_h, g_h = s.gradient()
    like = torch.empty(1, device="cuda")
    c_d, g_d = s.gradient(like=like)
    sctx.synchronize()
    assert c_h[0] == c_d[0]
    assert np.array_equal(g_d.cpu().numpy(), g_h)
