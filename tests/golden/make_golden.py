"""Generate tests/golden/golden.npz from the REFERENCE ITSELF (oracle/_ref:
the unmodified reference sources compiled by oracle/build_ref.sh).

Run in the build container (needs /root/reference):  python tests/golden/make_golden.py
Each case mirrors a reference test (file:line cited) or a BASELINE-shaped
input; the committed fixture pins the CPU oracle and the GPU path without
needing /root/reference at test time.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import refpy as R  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def kern(prefix, k, store):
    store[prefix + "weights"] = k.weights
    store[prefix + "support"] = k.support
    store[prefix + "values"] = k.values


def main():
    g = {}
    # --- full-rank SOCS vs Hopkins, test_imaging.cpp:157-171 (seed 41 stand-in) ---
    rng = np.random.default_rng(41)
    for n in (12, 16, 24):
        for focus in (0, 30):
            k = R.RefKernels(n, n, 4.0, focus=float(focus), energy_floor=1.0, full_rank=True)
            mask = rng.random((n, n))
            p = f"socs_{n}_{focus}_"
            kern(p, k, g)
            g[p + "mask"] = mask
            g[p + "image"] = R.image_socs(mask, k.weights, k.support, k.values, pitch=4.0)
            g[p + "hopkins"] = k.hopkins(mask)
    # --- truncated energy-floor kernels + dose 1.3 image (dose linearity input) ---
    k = R.RefKernels(16, 16, 4.0, focus=0.0, energy_floor=0.995)
    mask = np.random.default_rng(43).random((16, 16))
    kern("trunc_", k, g)
    g["trunc_mask"] = mask
    g["trunc_image13"] = R.image_socs(mask, k.weights, k.support, k.values, pitch=4.0, dose=1.3)
    # --- clear field, test_imaging.cpp:186-195 ---
    k = R.RefKernels(24, 24, 4.0, energy_floor=1.0, full_rank=True)
    kern("clear_", k, g)
    g["clear_image"] = R.image_socs(np.ones((24, 24)), k.weights, k.support, k.values, pitch=4.0, dose=1.3)
    # --- gaussian blur, test_imaging.cpp:232-271 ---
    v = np.random.default_rng(59).random((12, 16))
    g["blur_in"] = v
    g["blur_out"] = R.gaussian_blur(v, 2.5, 2.0)
    # --- gradient, test_opc_ai.cpp:266-295 (grid_n 5, dose 1.3) + weighted variant ---
    k = R.RefKernels(16, 16, 4.0, sigma_in=0.4, sigma_out=0.8, grid_n=5, energy_floor=1.0, full_rank=True)
    kern("grad_", k, g)
    rng = np.random.default_rng(89)
    mask = rng.random((16, 16))
    W = rng.standard_normal((16, 16))
    g["grad_mask"] = mask
    g["grad_W"] = W
    g["grad_uniform"] = R.intensity_gradient(mask, k.weights, k.support, k.values, pitch=4.0, dose=1.3)
    g["grad_weighted"] = R.weighted_gradient(mask, k.weights, k.support, k.values, W, pitch=4.0, dose=1.3)
    # --- z_print / z_round, test_opc_ai.cpp:326-352 ---
    g["zprint"] = R.z_print(mask, k.weights, k.support, k.values, 0.2, pitch=4.0)
    g["zround"] = R.z_round((mask > 0.5).astype(float), 2.0, 0.5, pitch=4.0)
    # --- rasterization, test_geometry.cpp:77-105 (random all-angle 8-gons, healed) ---
    rng = np.random.default_rng(5)
    polys = []
    for t in range(8):
        poly = [tuple(int(v) for v in rng.integers(5, 121, 2)) for _ in range(8)]
        healed = R.heal([poly])
        polys.append((poly, healed))
    for t, (poly, healed) in enumerate(polys):
        g[f"raster_{t}_input"] = np.array(poly, np.int64)
        g[f"raster_{t}_healed_n"] = np.array([len(h) for h in healed], np.int64)
        g[f"raster_{t}_healed"] = np.concatenate(healed) if healed else np.zeros((0, 2), np.int64)
        g[f"raster_{t}_out"] = R.rasterize([poly], 140, 140, 1.0, 0.0, 0.0, 1.0)
        g[f"raster_{t}_out_off"] = R.rasterize([poly], 300, 300, 0.5, -3.25, 1.5, 2.0)
    g["raster_kat_full"] = R.rasterize([[(2, 2), (6, 2), (6, 6), (2, 6)]], 8, 8)
    g["raster_kat_half"] = R.rasterize([[(0, 0), (9, 0), (9, 16), (0, 16)]], 8, 8, dbu_per_nm=2.0)
    # --- one through-focus ILT step composed from reference calls (24^2, F=3) ---
    ks = [R.RefKernels(24, 24, 4.0, focus=f, k_fixed=6) for f in (-40.0, 0.0, 40.0)]
    Kmin = min(x.K for x in ks)
    Wt = np.stack([x.weights[:Kmin] for x in ks])
    Vt = np.stack([x.values[:Kmin] for x in ks])
    rng = np.random.default_rng(505)
    target = (rng.random((24, 24)) > 0.5).astype(float)
    theta = rng.standard_normal((24, 24)) * 0.5
    g["ilt_weights"], g["ilt_support"], g["ilt_values"] = Wt, ks[0].support, Vt
    g["ilt_target"], g["ilt_theta0"] = target, theta.copy()
    g["ilt_params"] = np.array([4.0, 30.0, 0.25, 2.0, 1.0, 0.05])
    cost, grad = R.ilt_iteration(theta, target, Wt, ks[0].support, Vt, [1 / 3] * 3, g["ilt_params"], pitch=4.0)
    g["ilt_cost"], g["ilt_grad"], g["ilt_theta1"] = np.array(cost), grad, theta
    # --- pupil known answers, test_imaging.cpp:64-89 ---
    fc = 0.33 / 13.5
    g["pupil_args"] = np.array([[0, 0, 0], [0.99 * fc, 0, 0], [1.01 * fc, 0, 0], [0.8 * fc, 0.8 * fc, 0],
                                [0.5 * fc, 0, 40], [0.5 * fc, 0, -40]])
    g["pupil_vals"] = np.array([R.pupil(a, b, c) for a, b, c in g["pupil_args"]])
    np.savez_compressed(OUT, **g)
    print(OUT, os.path.getsize(OUT), "bytes,", len(g), "arrays")


if __name__ == "__main__":
    main()
