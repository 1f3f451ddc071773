"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle
(oracle/, itself pinned to the reference) and the committed golden vectors.

Tolerances: fp32 path rel L-inf <= 1e-4 (north star); fp64 path at the
reference's own test tolerances (test_imaging.cpp: 1e-6 .. 1e-10).
Rasterization: bitwise.
"""
import numpy as np
import pytest

import paper_2602_15036_b200 as L
from oracle import oracle as O
from oracle import refpy as R

pytestmark = pytest.mark.gpu


def rel_linf(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    s = np.abs(b).max()
    return np.abs(a - b).max() / (s if s > 0 else 1.0)


def euv(grid_n=7):
    return L.OpticalModel(source=L.make_annular_source(0.4, 0.8, grid_n))


def kernels_for(n, pitch, focus=(0.0,), k=0, floor=0.995, grid_n=7, ny=None):
    g = L.Grid(n, ny or n, pitch)
    return L.build_socs_kernels(euv(grid_n), g, list(focus), k_fixed=k, energy_floor=floor)


# (nx, ny, pitch, K, grid_n): small generic-DFT grids, decimated pow2 grids, C1 scale
IMG_CASES = [
    (16, 16, 4.0, 0, 7),
    (24, 24, 4.0, 0, 7),
    (16, 12, 4.0, 0, 7),
    (64, 64, 1.0, 8, 21),
    (256, 256, 1.0, 8, 21),
    (128, 256, 1.0, 12, 21),
    (1024, 1024, 1.0, 8, 21),
    (2048, 2048, 1.0, 16, 21),
]


@pytest.mark.parametrize("nx,ny,pitch,K,gn", IMG_CASES)
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_image_socs_vs_oracle(ctx, nx, ny, pitch, K, gn, prec):
    rng = np.random.default_rng(nx * 7 + ny)
    ks = kernels_for(nx, pitch, (30.0,), k=K, grid_n=gn, ny=ny)
    mask = rng.random((ny, nx))
    want = O.image_socs(mask, ks.weights[0], ks.support, ks.values[0], dose=1.3)
    dk = L.DeviceKernels(ks, prec, ctx)
    got = dk.image(mask, dose=1.3)["intensity"]
    tol = 1e-4 if prec == "f32" else 1e-10
    assert rel_linf(got, want) < tol, dk.info()


@pytest.mark.parametrize("prec,tol", [("f32", 1e-4), ("f64", 1e-10)])
def test_resist_image_vs_oracle(ctx, prec, tol):
    rng = np.random.default_rng(3)
    ks = kernels_for(256, 1.0, (0.0,), k=8, grid_n=21)
    mask = (rng.random((256, 256)) > 0.6).astype(np.float64)
    I = O.image_socs(mask, ks.weights[0], ks.support, ks.values[0])
    Rr = O.gaussian_blur(I, 2.0, 1.0)
    dk = L.DeviceKernels(ks, prec, ctx)
    out = dk.image(mask, sigma_nm=2.0, threshold=0.25, want=("intensity", "resist", "print"))
    assert rel_linf(out["intensity"], I) < tol
    assert rel_linf(out["resist"], Rr) < tol
    ref_print = O.threshold(Rr, 0.25)
    guard = np.abs(Rr - 0.25) > 1e-4 * np.abs(Rr).max()
    assert np.array_equal(out["print"][guard], ref_print[guard])


def test_full_rank_equals_reference_hopkins(ctx):
    """reference test_imaging.cpp:157-171 run through the drop-in (fp64)."""
    rng = np.random.default_rng(41)
    for n in (12, 16, 24):
        for focus in (0.0, 30.0):
            rk = R.RefKernels(n, n, 4.0, focus=focus, energy_floor=1.0, full_rank=True)
            ks = L.SocsKernelSet(L.Grid(n, n, 4.0), [focus], rk.weights[None], rk.support, rk.values[None])
            mask = rng.random((n, n))
            got = L.image_socs(mask, ks, 1.0, precision="f64", ctx=ctx)
            assert rel_linf(got, rk.hopkins(mask)) < 1e-6


def test_clear_field_flat(ctx):
    """reference test_imaging.cpp:186-195."""
    rk = R.RefKernels(24, 24, 4.0, energy_floor=1.0, full_rank=True)
    ks = L.SocsKernelSet(L.Grid(24, 24, 4.0), [0.0], rk.weights[None], rk.support, rk.values[None])
    got = L.image_socs(np.ones((24, 24)), ks, 1.3, precision="f64", ctx=ctx)
    assert np.abs(got - 1.3).max() < 1e-6


@pytest.mark.parametrize("shape,pitch,sigma", [((12, 16), 2.0, 2.5), ((256, 256), 1.0, 2.0),
                                               ((64, 128), 1.0, 3.0)])
def test_gaussian_blur_vs_oracle(ctx, shape, pitch, sigma):
    rng = np.random.default_rng(59)
    v = rng.random(shape)
    g = L.Grid(shape[1], shape[0], pitch)
    got = L.gaussian_blur(g, v, sigma, ctx)
    assert rel_linf(got, O.gaussian_blur(v, sigma, pitch)) < 1e-10
    assert np.array_equal(L.gaussian_blur(g, v, 0.0, ctx), v)


@pytest.mark.parametrize("n,pitch,K,gn", [(16, 4.0, 0, 5), (64, 1.0, 8, 21), (256, 1.0, 16, 21),
                                          (512, 1.0, 16, 21)])
@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("weighted", [False, True])
def test_gradient_vs_oracle(ctx, n, pitch, K, gn, prec, weighted):
    rng = np.random.default_rng(89 + n)
    ks = kernels_for(n, pitch, (0.0,), k=K, grid_n=gn, floor=1.0 if K == 0 else 0.995)
    mask = rng.random((n, n))
    W = rng.standard_normal((n, n)) if weighted else None
    want = O.weighted_gradient(mask, ks.weights[0], ks.support, ks.values[0], W, dose=1.3)
    got = L.intensity_gradient(mask, ks, 1.3, weight=W, precision=prec, ctx=ctx)
    tol = 1e-4 if prec == "f32" else 1e-9
    assert rel_linf(got, want) < tol


@pytest.mark.parametrize("n,F,K,prec,tol", [(64, 1, 8, "f64", 1e-9), (64, 3, 8, "f64", 1e-9),
                                            (256, 1, 16, "f32", 1e-4), (256, 5, 8, "f32", 1e-4),
                                            (24, 3, 0, "f64", 1e-9), (2048, 1, 16, "f32", 1e-4),
                                            (512, 3, 16, "f32", 1e-4)])
def test_ilt_step_vs_oracle(ctx, n, F, K, prec, tol):
    rng = np.random.default_rng(7 * n + F)
    pitch = 4.0 if n == 24 else 1.0
    foci = [-40.0, -20.0, 0.0, 20.0, 40.0][:F] if F == 5 else ([-40.0, 0.0, 40.0][:F] if F == 3 else [0.0])
    ks = kernels_for(n, pitch, foci, k=K, grid_n=7 if n == 24 else 21)
    target = (rng.random((n, n)) > 0.5).astype(np.float64)
    theta0 = rng.standard_normal((n, n)) * 0.5
    prm = L.IltParams(mask_steepness=4.0, resist_beta=30.0, threshold=0.25, resist_sigma_nm=2.0,
                      dose=1.0, step=0.05, focus_weights=[1.0 / F] * F)
    solver = L.IltSolver(ks, prm, 1, prec, ctx)
    solver.set_tiles(target[None], theta0[None])
    cost = solver.run(1)
    theta_gpu, _ = solver.get_tiles()
    th = theta0.copy()
    c_ref, g_ref = O.ilt_iteration(th, target, ks.weights, ks.support, ks.values, [1.0 / F] * F,
                                   [4.0, 30.0, 0.25, 2.0, 1.0, 0.05], pitch)
    assert abs(cost[0, 0] - c_ref) <= tol * abs(c_ref) * 10
    # theta update = -step * grad: compare the gradients (rel L-inf on the step)
    assert rel_linf(theta_gpu[0] - theta0, th - theta0) < tol * 10


def test_rasterize_bit_exact_vs_reference(ctx):
    rng = np.random.default_rng(5)
    # random all-angle 8-vertex polygons (reference test_geometry.cpp:90-104), healed by the reference
    for trial in range(6):
        poly = [tuple(int(v) for v in rng.integers(5, 121, 2)) for _ in range(8)]
        healed = R.heal([poly])
        for (ox, oy, pitch, dbu) in [(0.0, 0.0, 1.0, 1.0), (-3.25, 1.5, 0.5, 2.0)]:
            nx = ny = 300
            want = R.rasterize([poly], nx, ny, pitch, ox, oy, dbu)
            got = L.rasterize_layer(healed, L.Grid(nx, ny, pitch, ox, oy), dbu, ctx)
            assert np.array_equal(got, want)


def test_rasterize_known_answers(ctx):
    """reference test_geometry.cpp:77-88."""
    g = L.Grid(8, 8, 1.0)
    r = L.rasterize_layer([[(2, 2), (6, 2), (6, 6), (2, 6)]], g, 1.0, ctx)
    assert r[3, 3] == 1.0 and r[0, 0] == 0.0
    r = L.rasterize_layer([[(0, 0), (9, 0), (9, 16), (0, 16)]], g, 2.0, ctx)
    assert abs(r[3, 4] - 0.5) < 1e-12


def test_threshold_semantics(ctx):
    v = np.array([0.1, 0.25, 0.2500001, 0.3, 0.0])
    out = L.threshold(v, 0.25, ctx)
    assert out.tolist() == [0.0, 1.0, 1.0, 1.0, 0.0]


def test_gradient_selects_focus_stack(ctx):
    """intensity_gradient on stack `focus` of a multi-focus set (fp32 fast path
    views the stack as a one-focus plan)."""
    rng = np.random.default_rng(17)
    ks = kernels_for(256, 1.0, (-40.0, 0.0, 40.0), k=8, grid_n=21)
    mask = rng.random((256, 256))
    W = rng.standard_normal((256, 256))
    for f in (0, 2):
        want = O.weighted_gradient(mask, ks.weights[f], ks.support, ks.values[f], W, dose=1.1)
        got = L.intensity_gradient(mask, ks, 1.1, weight=W, focus=f, precision="f32", ctx=ctx)
        assert rel_linf(got, want) < 1e-4


@pytest.mark.parametrize("n,F,K", [(256, 1, 16), (512, 3, 8)])
def test_ilt_multi_iteration_graph_vs_oracle(ctx, n, F, K):
    """several ILT iterations in one call, repeated so the CUDA-graph capture
    and replay paths both run, against the oracle iterated the same way."""
    rng = np.random.default_rng(11 * n + F)
    foci = [-40.0, 0.0, 40.0][:F] if F == 3 else [0.0]
    ks = kernels_for(n, 1.0, foci, k=K, grid_n=21)
    target = (rng.random((n, n)) > 0.5).astype(np.float64)
    theta0 = rng.standard_normal((n, n)) * 0.5
    prm = L.IltParams(mask_steepness=4.0, resist_beta=30.0, threshold=0.25, resist_sigma_nm=2.0,
                      dose=1.0, step=0.05, focus_weights=[1.0 / F] * F)
    solver = L.IltSolver(ks, prm, 1, "f32", ctx)
    solver.set_tiles(target[None], theta0[None])
    costs = [solver.run(2)[:, 0] for _ in range(3)]  # eager, capture, replay
    theta_gpu, _ = solver.get_tiles()
    th = theta0.copy()
    c_ref = []
    for _ in range(6):
        c, _ = O.ilt_iteration(th, target, ks.weights, ks.support, ks.values, [1.0 / F] * F,
                               [4.0, 30.0, 0.25, 2.0, 1.0, 0.05], 1.0)
        c_ref.append(c)
    got = np.concatenate(costs)
    assert np.abs(got - np.array(c_ref)).max() <= 1e-4 * np.abs(c_ref).max()
    assert rel_linf(theta_gpu[0] - theta0, th - theta0) < 1e-3


def test_ilt_stored_fields_bit_identical(ctx, monkeypatch):
    """keeping E_fk for the adjoint (LITHOGPU_STORE_E=1) and recomputing it
    (=0) run the same arithmetic: results must be bitwise equal."""
    rng = np.random.default_rng(23)
    n = 512
    ks = kernels_for(n, 1.0, (0.0,), k=16, grid_n=21)
    target = (rng.random((n, n)) > 0.5).astype(np.float64)
    prm = L.IltParams(step=0.05, focus_weights=[1.0])
    out = []
    for flag in ("0", "1"):
        monkeypatch.setenv("LITHOGPU_STORE_E", flag)
        dk = L.DeviceKernels(ks, "f32", ctx)
        solver = L.IltSolver(dk, prm, 1, "f32", ctx)
        solver.set_tiles(target[None])
        cost = solver.run(3)
        out.append((cost.copy(), solver.get_tiles()[0].copy()))
        solver.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])


@pytest.mark.parametrize("n,K,foci", [(256, 12, (0.0,)), (256, 0, (-40.0, 0.0, 40.0)), (2048, 16, (0.0, 40.0))])
def test_gpu_kernel_generation_vs_host(ctx, n, K, foci):
    """GPU Abbe-SVD (cuBLAS + cuSOLVER) against the host
    generator: same eigenvalues, eigenvectors of the TCC with the reference
    phase rule, and (full rank) the same image."""
    model = euv(21)
    grid = L.Grid(n, n, 1.0)
    host = L.build_socs_kernels(model, grid, list(foci), k_fixed=K)
    gpu = L.build_socs_kernels(model, grid, list(foci), k_fixed=K, backend="gpu", ctx=ctx)
    assert np.array_equal(host.support, gpu.support)
    assert gpu.weights.shape == host.weights.shape
    assert np.abs(gpu.weights - host.weights).max() <= 1e-10 * host.weights.max()
    S = len(host.support)
    src = np.asarray(model.source)
    fc = model.na / model.wavelength_nm
    fx = host.support[:, 0] / (n * 1.0)
    fy = host.support[:, 1] / (n * 1.0)
    for f, foc in enumerate(foci):
        # Q[i][s] = sqrt(w_s) P(f_i + s fc)
        gx = fx[:, None] + src[None, :, 0] * fc
        gy = fy[:, None] + src[None, :, 1] * fc
        f2 = gx ** 2 + gy ** 2
        Q = np.where(f2 <= fc * fc, np.exp(-1j * np.pi * model.wavelength_nm * foc * f2), 0.0) * np.sqrt(src[:, 2])
        for k in range(min(4, gpu.weights.shape[1])):
            u, lam = gpu.values[f, k], gpu.weights[f, k]
            if lam == 0:
                continue
            r = Q @ (Q.conj().T @ u) - lam * u
            assert np.abs(r).max() <= 1e-9 * lam * np.abs(u).max()
            i = int(np.argmax(np.abs(u)))
            assert abs(u[i].imag) <= 1e-12 * abs(u[i]) and u[i].real > 0
    if n == 256 and K == 0:  # energy-floor truncation: images agree
        rng = np.random.default_rng(4)
        mask = rng.random((n, n))
        for f in range(len(foci)):
            a = O.image_socs(mask, host.weights[f], host.support, host.values[f])
            b = O.image_socs(mask, gpu.weights[f], gpu.support, gpu.values[f])
            assert rel_linf(b, a) < 1e-6


def test_kernel_pairs_engage_and_match(ctx, monkeypatch):
    """in-focus kernels of the symmetric annular source are Hermitian-symmetric:
    the fast path runs them as pairs (half the kernel transforms) with the
    same images / gradients / ILT steps as the per-kernel path and the oracle."""
    n = 512
    ks = kernels_for(n, 1.0, (0.0,), k=16, grid_n=21)
    defocus = kernels_for(n, 1.0, (40.0,), k=16, grid_n=21)
    rng = np.random.default_rng(31)
    mask = (rng.random((n, n)) > 0.5).astype(np.float64)
    W = rng.standard_normal((n, n))
    dk = L.DeviceKernels(ks, "f32", ctx)
    assert dk.info()["fast_order"] == 8
    assert L.DeviceKernels(defocus, "f32", ctx).info()["fast_order"] == 16
    monkeypatch.setenv("LITHOGPU_NO_PAIRS", "1")
    dk1 = L.DeviceKernels(ks, "f32", ctx)
    assert dk1.info()["fast_order"] == 16
    want = O.image_socs(mask, ks.weights[0], ks.support, ks.values[0])
    a = dk.image(mask)["intensity"]
    b = dk1.image(mask)["intensity"]
    assert rel_linf(a, want) < 1e-4 and rel_linf(b, want) < 1e-4
    gw = O.weighted_gradient(mask, ks.weights[0], ks.support, ks.values[0], W, dose=1.0)
    assert rel_linf(dk.gradient(mask, 1.0, weight=W), gw) < 1e-4
    prm = L.IltParams(step=0.05, focus_weights=[1.0])
    th0 = rng.standard_normal((n, n)) * 0.5
    out = []
    for d in (dk, dk1):
        s = L.IltSolver(d, prm, 1, "f32", ctx)
        s.set_tiles(mask[None], th0[None])
        c = s.run(2)
        out.append((c, s.get_tiles()[0]))
    assert np.abs(out[0][0] - out[1][0]).max() <= 1e-4 * np.abs(out[1][0]).max()
    assert rel_linf(out[0][1] - th0, out[1][1] - th0) < 1e-3


def test_mirror_focus_stacks_merge(ctx, monkeypatch):
    """paraxial -F / +F stacks of the symmetric source are conjugate mirrors:
    the fast path computes one of them (fast_stacks), with images, gradients
    and ILT cost equal to the oracle on every stack's own kernels."""
    n = 256
    foci = (-40.0, 0.0, 40.0)
    ks = kernels_for(n, 1.0, foci, k=8, grid_n=21)
    dk = L.DeviceKernels(ks, "f32", ctx)
    assert dk.info()["fast_stacks"] == 2
    rng = np.random.default_rng(37)
    mask = (rng.random((n, n)) > 0.5).astype(np.float64)
    W = rng.standard_normal((n, n))
    for f in range(3):
        want = O.image_socs(mask, ks.weights[f], ks.support, ks.values[f])
        assert rel_linf(dk.image(mask, focus=f)["intensity"], want) < 1e-4
        gw = O.weighted_gradient(mask, ks.weights[f], ks.support, ks.values[f], W, dose=1.0)
        assert rel_linf(dk.gradient(mask, 1.0, weight=W, focus=f), gw) < 1e-4
    prm = L.IltParams(step=0.05, focus_weights=[0.2, 0.5, 0.3])
    th0 = rng.standard_normal((n, n)) * 0.5
    out = []
    for merge in ("", "1"):
        if merge:
            monkeypatch.setenv("LITHOGPU_NO_FOCUS_MERGE", "1")
        d = L.DeviceKernels(ks, "f32", ctx)
        assert d.info()["fast_stacks"] == (3 if merge else 2)
        s = L.IltSolver(d, prm, 1, "f32", ctx)
        s.set_tiles(mask[None], th0[None])
        out.append((s.run(2), s.get_tiles()[0]))
    th = th0.copy()
    c_ref, _ = O.ilt_iteration(th, mask, ks.weights, ks.support, ks.values, [0.2, 0.5, 0.3],
                               [4.0, 30.0, 0.25, 2.0, 1.0, 0.05], 1.0)
    assert abs(out[0][0][0, 0] - c_ref) <= 1e-4 * abs(c_ref)
    assert np.abs(out[0][0] - out[1][0]).max() <= 1e-4 * np.abs(out[1][0]).max()
    assert rel_linf(out[0][1] - th0, out[1][1] - th0) < 1e-3


def test_rasterize_rectangles_bit_exact(ctx):
    """Manhattan layouts (the bench targets): rectangles take the exact
    full-pixel shortcut inside, the clip chain on their edges; bitwise equal
    to the reference at fractional origins / pitches / dbu."""
    from paper_2602_15036_b200 import layouts as LY
    rng = np.random.default_rng(77)
    polys = LY.line_space_contacts(300, 260, seed=3)
    # extra rectangles and an L shape with odd coordinates, healed by the reference
    extra = [[(7, 9), (51, 9), (51, 33), (7, 33)], [(201, 150), (237, 150), (237, 211), (219, 211), (219, 171),
                                                   (201, 171)]]
    healed_extra = R.heal(extra)
    for (ox, oy, pitch, dbu) in [(0.0, 0.0, 1.0, 1.0), (-3.25, 1.5, 0.5, 2.0), (0.3, -0.7, 1.25, 1.0)]:
        nx, ny = int(330 / pitch), int(290 / pitch)
        for layer in (polys, healed_extra):
            want = R.rasterize(layer, nx, ny, pitch, ox, oy, dbu)
            got = L.rasterize_layer(layer, L.Grid(nx, ny, pitch, ox, oy), dbu, ctx)
            assert np.array_equal(got, want), (ox, oy, pitch, dbu)
    assert rng is not None


@pytest.mark.parametrize("K,foci", [(5, (0.0,)), (6, (-30.0, 30.0))])
def test_odd_pairs_and_two_mirror_stacks(ctx, K, foci):
    """odd K (the last kernel pair has one member) and a lone -F/+F pair of
    stacks: images and one ILT step against the oracle."""
    n = 128
    ks = kernels_for(n, 1.0, foci, k=K, grid_n=21)
    dk = L.DeviceKernels(ks, "f32", ctx)
    info = dk.info()
    F = len(foci)
    if F == 1:
        assert info["fast_order"] == (K + 1) // 2
    else:
        assert info["fast_stacks"] == 1
    rng = np.random.default_rng(K)
    mask = rng.random((n, n))
    for f in range(F):
        want = O.image_socs(mask, ks.weights[f], ks.support, ks.values[f])
        assert rel_linf(dk.image(mask, focus=f)["intensity"], want) < 1e-4
    target = (mask > 0.5).astype(np.float64)
    th0 = rng.standard_normal((n, n)) * 0.5
    prm = L.IltParams(step=0.05, focus_weights=[1.0 / F] * F)
    s = L.IltSolver(dk, prm, 1, "f32", ctx)
    s.set_tiles(target[None], th0[None])
    c = s.run(1)
    th = th0.copy()
    c_ref, _ = O.ilt_iteration(th, target, ks.weights, ks.support, ks.values, [1.0 / F] * F,
                               [4.0, 30.0, 0.25, 2.0, 1.0, 0.05], 1.0)
    assert abs(c[0, 0] - c_ref) <= 1e-4 * abs(c_ref)
    assert rel_linf(s.get_tiles()[0][0] - th0, th - th0) < 1e-3


def test_evaluate_epe_f32_kernels(ctx):
    """evaluate_epe on the fp32 fast path (resist widened to f64 on the device)
    against the fp64 path: same open flags, EPE within the fp32 image tolerance."""
    from paper_2602_15036_b200 import layouts as LY
    n = 256
    grid = L.Grid(n, n, 1.0)
    m = L.rasterize_layer(LY.line_space_contacts(n, n, seed=4), grid, 1.0, ctx)
    m[:16, :] = m[-16:, :] = 0.0
    m[:, :16] = m[:, -16:] = 0.0
    ks = kernels_for(n, 1.0, (0.0,), k=8, grid_n=21)
    rng = np.random.default_rng(5)
    k = 300
    ang = rng.choice([0.0, np.pi / 2, np.pi, 1.5 * np.pi], k)
    g = np.column_stack([rng.uniform(20, n - 20, k), rng.uniform(20, n - 20, k), np.cos(ang), np.sin(ang)])
    e32, o32 = L.evaluate_epe(m, L.DeviceKernels(ks, "f32", ctx), g, 1.0, 2.0, 0.25, 10.0)
    e64, o64 = L.evaluate_epe(m, L.DeviceKernels(ks, "f64", ctx), g, 1.0, 2.0, 0.25, 10.0)
    both = ~o32 & ~o64
    assert (o32 != o64).sum() <= 2  # a gauge exactly at the search radius may flip
    assert np.abs(e32[both] - e64[both]).max() < 0.05  # nm; fp32 intensity 1e-4 rel near the threshold


def test_mixed_kernel_pairs_through_focus(ctx, monkeypatch):
    """through-focus set (-40, 0, 40): the in-focus stack runs as kernel pairs
    inside the same launches as the defocused (unpaired, mirror-merged)
    stack; images, gradients and ILT cost against the oracle and against the
    unpaired path."""
    n = 256
    foci = (-40.0, 0.0, 40.0)
    ks = kernels_for(n, 1.0, foci, k=8, grid_n=21)
    dk = L.DeviceKernels(ks, "f32", ctx)
    info = dk.info()
    assert info["fast_stacks"] == 2 and info["fast_order"] == 8
    rng = np.random.default_rng(53)
    mask = (rng.random((n, n)) > 0.5).astype(np.float64)
    W = rng.standard_normal((n, n))
    for f in range(3):
        want = O.image_socs(mask, ks.weights[f], ks.support, ks.values[f])
        assert rel_linf(dk.image(mask, focus=f)["intensity"], want) < 1e-4
        gw = O.weighted_gradient(mask, ks.weights[f], ks.support, ks.values[f], W, dose=1.0)
        assert rel_linf(dk.gradient(mask, 1.0, weight=W, focus=f), gw) < 1e-4
    prm = L.IltParams(step=0.05, focus_weights=[0.25, 0.5, 0.25])
    th0 = rng.standard_normal((n, n)) * 0.5
    out = []
    for nopair in ("", "1"):
        if nopair:
            monkeypatch.setenv("LITHOGPU_NO_PAIRS", "1")
        d = L.DeviceKernels(ks, "f32", ctx)
        s = L.IltSolver(d, prm, 1, "f32", ctx)
        s.set_tiles(mask[None], th0[None])
        out.append((s.run(2), s.get_tiles()[0]))
    th = th0.copy()
    c_ref, _ = O.ilt_iteration(th, mask, ks.weights, ks.support, ks.values, [0.25, 0.5, 0.25],
                               [4.0, 30.0, 0.25, 2.0, 1.0, 0.05], 1.0)
    assert abs(out[0][0][0, 0] - c_ref) <= 1e-4 * abs(c_ref)
    assert np.abs(out[0][0] - out[1][0]).max() <= 1e-4 * np.abs(out[1][0]).max()
    assert rel_linf(out[0][1] - th0, out[1][1] - th0) < 1e-3


def test_batched_tiles_match_single_tile_runs(ctx):
    """tiles batched on blockIdx.z (the chip-scale launches) compute each tile
    exactly as a one-tile run: costs and theta bitwise equal."""
    n, T = 256, 3
    ks = kernels_for(n, 1.0, (-40.0, 0.0, 40.0), k=8, grid_n=21)
    dk = L.DeviceKernels(ks, "f32", ctx)
    rng = np.random.default_rng(61)
    targets = (rng.random((T, n, n)) > 0.5).astype(np.float64)
    th0 = rng.standard_normal((T, n, n)) * 0.5
    prm = L.IltParams(step=0.05, focus_weights=[0.25, 0.5, 0.25])
    sb = L.IltSolver(dk, prm, T, "f32", ctx)
    sb.set_tiles(targets, th0)
    cb = sb.run(3)
    thb = sb.get_tiles()[0]
    for t in range(T):
        s1 = L.IltSolver(dk, prm, 1, "f32", ctx)
        s1.set_tiles(targets[t:t + 1], th0[t:t + 1])
        c1 = s1.run(3)
        assert np.array_equal(c1[:, 0], cb[:, t])
        assert np.array_equal(s1.get_tiles()[0][0], thb[t])
        s1.close()


def test_chip_ilt_tiles_and_costs(ctx):
    """chip.ChipIlt on a 2x2-tile window (world 1): the global per-iteration
    cost is the sum of the per-tile costs of independent one-tile runs."""
    from paper_2602_15036_b200 import chip, layouts as LY
    core, halo = 96, 16
    n = core + 2 * halo
    chipg = L.Grid(2 * core, 2 * core, 1.0, 0.0, 0.0)
    tiling = LY.Tiling(chipg, core, halo)
    polys = LY.line_space_contacts(2 * core, 2 * core, seed=12)
    ks = kernels_for(n, 1.0, (0.0,), k=8, grid_n=21)
    prm = L.IltParams(step=0.05, focus_weights=[1.0])
    ci = chip.ChipIlt(tiling, polys, ks, prm, ctx)
    res = ci.run(4, sync_every=2)
    assert len(res.cost) == 4 and list(res.tiles) == [0, 1, 2, 3]
    tot = np.zeros(4)
    from paper_2602_15036_b200 import layouts
    for t in range(4):
        g = tiling.tile_grid(t)
        raster = L.rasterize_layer(tiling.tile_polygons(polys, t), g, 1.0, ctx)
        s = L.IltSolver(ks, prm, 1, "f32", ctx)
        s.set_tiles(raster[None].astype(np.float32))
        tot += s.run(4)[:, 0]
    assert np.abs(res.cost - tot).max() <= 1e-6 * np.abs(tot).max()
    assert np.all(res.gmax > 0)


def test_c4_scale_image_and_gradient(ctx):
    """4096^2 tiles (C4: N = 4096 plans, decimated n = 768 plans) against the
    oracle: aerial image and weighted gradient, fp32 1e-4."""
    n = 4096
    ks = kernels_for(n, 1.0, (40.0,), k=4, grid_n=21)
    rng = np.random.default_rng(97)
    mask = (rng.random((n, n)) > 0.5).astype(np.float64)
    dk = L.DeviceKernels(ks, "f32", ctx)
    assert dk.info()["nx_sub"] == 768
    want = O.image_socs(mask, ks.weights[0], ks.support, ks.values[0])
    assert rel_linf(dk.image(mask)["intensity"], want) < 1e-4
    W = rng.standard_normal((n, n))
    gw = O.weighted_gradient(mask, ks.weights[0], ks.support, ks.values[0], W, dose=1.0)
    assert rel_linf(dk.gradient(mask, 1.0, weight=W), gw) < 1e-4


@pytest.mark.parametrize("n", [256, 2048])
def test_off_axis_source_asymmetric_kernels(ctx, n):
    """An off-axis (asymmetric) source: kernels without Hermitian symmetry, so
    no kernel pairs and no mirror-stack merge, on the fast path (the TCC support
    itself stays the centered disk |f| <= (1 + sigma_max) f_c, imaging.cpp:
    120-129), against the oracle for the image, the weighted gradient and one
    ILT step."""
    src = np.array([[0.35, 0.2, 0.7], [0.55, -0.1, 0.3]])
    model = L.OpticalModel(source=src)
    ks = L.build_socs_kernels(model, L.Grid(n, n, 1.0), [0.0, 25.0], k_fixed=2)
    rng = np.random.default_rng(n)
    mask = (rng.random((n, n)) > 0.5).astype(np.float64)
    dk = L.DeviceKernels(ks, "f32", ctx)
    for f in range(2):
        want = O.image_socs(mask, ks.weights[f], ks.support, ks.values[f])
        got = dk.image(mask, focus=f)["intensity"]
        assert rel_linf(got, want) < 1e-4
    W = rng.standard_normal((n, n))
    gw = O.weighted_gradient(mask, ks.weights[0], ks.support, ks.values[0], W)
    assert rel_linf(L.intensity_gradient(mask, dk, 1.0, weight=W, precision="f32", ctx=ctx), gw) < 1e-4
    prm = [4.0, 30.0, 0.25, 2.0, 1.0, 0.5]
    theta0 = (2 * mask - 1) * 0.5
    th = theta0.copy()
    c_ref, g_ref = O.ilt_iteration(th, mask, ks.weights, ks.support, ks.values, [0.5, 0.5], prm, 1.0)
    s = L.IltSolver(dk, L.IltParams(*prm, focus_weights=[0.5, 0.5]), 1, "f32", ctx)
    s.set_tiles(mask[None], theta0[None])
    cost, grad = s.gradient()
    assert abs(cost[0] - c_ref) <= 1e-4 * abs(c_ref)
    assert rel_linf(grad[0], g_ref) < 1e-4
