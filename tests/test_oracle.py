"""CPU: pin the oracle (oracle/litho_oracle.c) to the reference.

Against the committed golden vectors (generated from the reference itself by
tests/golden/make_golden.py) and, when oracle/_ref is built, against the
reference live on fresh random inputs.  Plus the reference's own property
tests (test_imaging.cpp / test_opc_ai.cpp) restated on the oracle.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle import refpy as R

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("n", [12, 16, 24])
@pytest.mark.parametrize("focus", [0, 30])
def test_socs_matches_golden_and_hopkins(n, focus):
    p = f"socs_{n}_{focus}_"
    img = O.image_socs(GOLD[p + "mask"], GOLD[p + "weights"], GOLD[p + "support"], GOLD[p + "values"])
    assert rel(img, GOLD[p + "image"]) < 1e-12
    assert rel(img, GOLD[p + "hopkins"]) < 1e-6  # test_imaging.cpp:169


def test_truncated_kernels_and_dose():
    img = O.image_socs(GOLD["trunc_mask"], GOLD["trunc_weights"], GOLD["trunc_support"], GOLD["trunc_values"],
                       dose=1.3)
    assert rel(img, GOLD["trunc_image13"]) < 1e-12
    one = O.image_socs(GOLD["trunc_mask"], GOLD["trunc_weights"], GOLD["trunc_support"], GOLD["trunc_values"])
    assert rel(1.3 * one, img) < 1e-12  # dose linearity, test_imaging.cpp:173-184


def test_clear_field():
    img = O.image_socs(np.ones((24, 24)), GOLD["clear_weights"], GOLD["clear_support"], GOLD["clear_values"],
                       dose=1.3)
    assert rel(img, GOLD["clear_image"]) < 1e-12
    assert np.abs(img - 1.3).max() < 1e-6  # test_imaging.cpp:194


def test_blur_golden_and_direct():
    out = O.gaussian_blur(GOLD["blur_in"], 2.5, 2.0)
    assert rel(out, GOLD["blur_out"]) < 1e-12
    # direct cyclic convolution oracle, test_imaging.cpp:243-266
    v = GOLD["blur_in"]
    ny, nx = v.shape
    sp = 2.5 / 2.0
    rx = min(nx // 2, int(np.ceil(6 * sp)) + 1)
    ry = min(ny // 2, int(np.ceil(6 * sp)) + 1)
    d = [(dx, dy) for dy in range(-ry, ry + 1) for dx in range(-rx, rx + 1)]
    w = np.array([np.exp(-0.5 * (dx * dx + dy * dy) / sp ** 2) for dx, dy in d])
    w /= w.sum()
    want = np.zeros_like(v)
    for (dx, dy), ww in zip(d, w):
        want += ww * np.roll(np.roll(v, dy, 0), dx, 1)
    assert rel(out, want) < 1e-10
    assert abs(out.sum() - v.sum()) < 1e-10 * abs(v.sum())


def test_gradient_golden():
    args = (GOLD["grad_mask"], GOLD["grad_weights"], GOLD["grad_support"], GOLD["grad_values"])
    assert rel(O.weighted_gradient(*args, dose=1.3), GOLD["grad_uniform"]) < 1e-12
    assert rel(O.weighted_gradient(*args, W=GOLD["grad_W"], dose=1.3), GOLD["grad_weighted"]) < 1e-12


def test_gradient_central_differences():
    """test_opc_ai.cpp:266-295: adjoint vs FD (h=1e-5, <= 1e-4 max|grad|)."""
    mask, w, s, v = GOLD["grad_mask"], GOLD["grad_weights"], GOLD["grad_support"], GOLD["grad_values"]
    W = GOLD["grad_W"]
    for weight in (None, W):
        grad = O.weighted_gradient(mask, w, s, v, weight, dose=1.3)

        def total(m):
            I = O.image_socs(m, w, s, v, dose=1.3)
            return float(np.sum(I if weight is None else weight * I))

        scale = np.abs(grad).max()
        for j in range(0, mask.size, 7):
            e = np.zeros(mask.size)
            e[j] = 1e-5
            e = e.reshape(mask.shape)
            fd = (total(mask + e) - total(mask - e)) / 2e-5
            assert abs(fd - grad.flat[j]) <= 1e-4 * scale


def test_threshold_refs():
    mask, w, s, v = GOLD["grad_mask"], GOLD["grad_weights"], GOLD["grad_support"], GOLD["grad_values"]
    zp = O.threshold(O.image_socs(mask, w, s, v), 0.2)
    assert np.array_equal(zp, GOLD["zprint"])
    zr = O.threshold(O.gaussian_blur((mask > 0.5).astype(float), 2.0, 4.0), 0.5)
    assert np.array_equal(zr, GOLD["zround"])
    assert set(np.unique(zp)) <= {0.0, 1.0}


def _healed(t):
    n = GOLD[f"raster_{t}_healed_n"]
    xy = GOLD[f"raster_{t}_healed"]
    out, o = [], 0
    for k in n:
        out.append(xy[o:o + k])
        o += k
    return out


@pytest.mark.parametrize("t", range(8))
def test_raster_bit_exact_golden(t):
    h = _healed(t)
    assert np.array_equal(O.rasterize(h, 140, 140, 1.0, 0.0, 0.0, 1.0), GOLD[f"raster_{t}_out"])
    assert np.array_equal(O.rasterize(h, 300, 300, 0.5, -3.25, 1.5, 2.0), GOLD[f"raster_{t}_out_off"])


def test_raster_known_answers():
    r = O.rasterize([[(2, 2), (6, 2), (6, 6), (2, 6)]], 8, 8)
    assert np.array_equal(r, GOLD["raster_kat_full"]) and r[3, 3] == 1.0 and r[0, 0] == 0.0
    r = O.rasterize([[(0, 0), (9, 0), (9, 16), (0, 16)]], 8, 8, dbu_per_nm=2.0)
    assert np.array_equal(r, GOLD["raster_kat_half"]) and abs(r[3, 4] - 0.5) < 1e-12


def test_raster_area_conservation():
    """test_geometry.cpp:90-104: sum of pixels == healed area."""
    for t in range(8):
        h = _healed(t)
        area2 = sum(int(np.sum(p[:, 0] * np.roll(p[:, 1], -1) - np.roll(p[:, 0], -1) * p[:, 1])) for p in h)
        r = O.rasterize(h, 140, 140)
        assert abs(r.sum() - area2 / 2.0) <= 1e-9 * max(1.0, abs(area2 / 2.0))


def test_ilt_step_golden():
    th = GOLD["ilt_theta0"].copy()
    cost, grad = O.ilt_iteration(th, GOLD["ilt_target"], GOLD["ilt_weights"], GOLD["ilt_support"],
                                 GOLD["ilt_values"], [1 / 3] * 3, GOLD["ilt_params"], pitch=4.0)
    assert abs(cost - float(GOLD["ilt_cost"])) <= 1e-12 * abs(cost)
    assert rel(grad, GOLD["ilt_grad"]) < 1e-12
    assert rel(th, GOLD["ilt_theta1"]) < 1e-12


def test_ilt_gradient_central_differences():
    """The ILT cost gradient (new, not in the reference) pinned by the
    reference's own methodology: central differences, h = 1e-5."""
    base = GOLD["ilt_theta0"]
    args = (GOLD["ilt_target"], GOLD["ilt_weights"], GOLD["ilt_support"], GOLD["ilt_values"], [1 / 3] * 3,
            GOLD["ilt_params"], 4.0)
    _, grad = O.ilt_iteration(base.copy(), *args)
    scale = np.abs(grad).max()

    def cost(th):
        c, _ = O.ilt_iteration(th.copy(), *args)
        return c

    for j in range(0, base.size, 37):
        e = np.zeros(base.size)
        e[j] = 1e-5
        e = e.reshape(base.shape)
        fd = (cost(base + e) - cost(base - e)) / 2e-5
        assert abs(fd - grad.flat[j]) <= 1e-4 * scale


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
def test_oracle_vs_reference_live():
    rng = np.random.default_rng(7)
    for n, pitch, focus in [(20, 4.0, 10.0), (32, 2.0, -25.0)]:
        k = R.RefKernels(n, n, pitch, focus=focus, energy_floor=0.99)
        m = rng.random((n, n))
        a = R.image_socs(m, k.weights, k.support, k.values, pitch=pitch, dose=0.9)
        b = O.image_socs(m, k.weights, k.support, k.values, dose=0.9)
        assert rel(b, a) < 1e-12
        W = rng.standard_normal((n, n))
        a = R.weighted_gradient(m, k.weights, k.support, k.values, W, pitch=pitch)
        b = O.weighted_gradient(m, k.weights, k.support, k.values, W)
        assert rel(b, a) < 1e-12
    polys = [[(3, 4), (50, 9), (41, 60), (12, 37)], [(70, 70), (99, 70), (99, 99), (70, 99)]]
    h = R.heal(polys)
    assert np.array_equal(O.rasterize(h, 128, 128, 0.75, -1.0, 2.5, 1.0),
                          R.rasterize(polys, 128, 128, 0.75, -1.0, 2.5, 1.0))


@pytest.mark.parametrize("n,pitch,focus,grid_n", [(16, 4.0, 0.0, 7), (24, 4.0, 30.0, 7), (32, 2.0, -20.0, 5)])
def test_numpy_kernel_source_vs_reference_decompose_tcc(n, pitch, focus, grid_n):
    """oracle/kernels_np.py (the reference arm's kernel source) against the
    reference build_tcc + decompose_tcc itself (oracle/_ref): same support
    order, eigenvalues, and the same full-rank image."""
    from oracle import kernels_np as KN
    if not R.available():
        pytest.skip("oracle/_ref not built")
    rk = R.RefKernels(n, n, pitch, focus=focus, grid_n=grid_n, energy_floor=1.0)
    src = KN.annular_source(0.4, 0.8, grid_n)
    w, sup, v = KN.socs_kernels(n, n, pitch, src, focus, 0, energy_floor=1.0)
    assert np.array_equal(sup, rk.support)
    k = min(len(w), rk.K)
    assert np.abs(w[:k] - rk.weights[:k]).max() <= 1e-10 * rk.weights[0]
    rng = np.random.default_rng(n)
    mask = rng.random((n, n))
    a = O.image_socs(mask, w, sup, v)
    b = O.image_socs(mask, rk.weights, rk.support, rk.values)
    assert rel(a, b) < 1e-9


def test_numpy_kernel_source_vs_product_generator():
    """the same numbers as the product's host generator at a BASELINE-like
    band (256^2, 1 nm, K = 12, through focus)."""
    import paper_2602_15036_b200 as L
    from oracle import kernels_np as KN
    n = 256
    W, sup, V = KN.socs_kernel_stacks(n, 1.0, [-40.0, 0.0], 12)
    ks = L.build_socs_kernels(L.OpticalModel(source=L.make_annular_source(0.4, 0.8, 21)), L.Grid(n, n, 1.0),
                              [-40.0, 0.0], k_fixed=12)
    assert np.array_equal(sup, ks.support)
    assert np.abs(W - ks.weights).max() <= 1e-10 * ks.weights.max()
    mask = np.random.default_rng(1).random((n, n))
    for f in range(2):
        a = O.image_socs(mask, W[f], sup, V[f])
        b = O.image_socs(mask, ks.weights[f], ks.support, ks.values[f])
        assert rel(a, b) < 1e-8
