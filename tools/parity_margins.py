#!/usr/bin/env python
"""Print the rel L-inf errors behind the north-star parity tests (margin to
the 1e-4 bar) for the ILT gradient at C2 / C3 / C5-shaped problems and the
forward image at C1, against the fp64 oracle.

  python tools/parity_margins.py [--out gpurun_out/parity_margins.json]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2602_15036_b200 as L  # noqa: E402
from oracle import oracle as O  # noqa: E402
from test_gpu_ilt_parity import ILT, PRM, bench_tile, euv, rel_linf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/parity_margins.json")
    a = ap.parse_args()
    O.set_threads(os.cpu_count() or 1)
    ctx = L.default_context(0)
    res = []
    for n, K, foci, name in [(2048, 16, (0.0,), "C2"), (2048, 16, (-40.0, -20.0, 0.0, 20.0, 40.0), "C3"),
                             (2048, 24, (-40.0, 0.0, 40.0), "C5 tile")]:
        F = len(foci)
        fw = [1.0 / F] * F
        ks = L.build_socs_kernels(euv(), L.Grid(n, n, 1.0), list(foci), k_fixed=K, backend="gpu", ctx=ctx)
        target, theta0 = bench_tile(n, seed=4242)
        theta0 = theta0 + np.random.default_rng(1).standard_normal(theta0.shape) * 0.25
        s = L.IltSolver(ks, L.IltParams(focus_weights=fw, **ILT), 1, "f32", ctx)
        s.set_tiles(target[None], theta0[None])
        cost, grad = s.gradient()
        th = np.ascontiguousarray(theta0, np.float64).copy()
        c_ref, g_ref = O.ilt_iteration(th, target, ks.weights, ks.support, ks.values, fw, PRM, 1.0)
        res.append({"case": name, "grad_rel_linf": rel_linf(grad[0], g_ref),
                    "cost_rel": abs(cost[0] - c_ref) / abs(c_ref)})
        print(json.dumps(res[-1]), flush=True)
    n = 1024
    ks = L.build_socs_kernels(euv(), L.Grid(n, n, 1.0), [0.0], k_fixed=8, backend="gpu", ctx=ctx)
    mask = O.rasterize(__import__("paper_2602_15036_b200.layouts", fromlist=["x"]).line_space_contacts(n, n, seed=3),
                       n, n)
    want = O.image_socs(mask, ks.weights[0], ks.support, ks.values[0])
    got = L.DeviceKernels(ks, "f32", ctx).image(mask)["intensity"]
    res.append({"case": "C1 aerial", "image_rel_linf": rel_linf(got, want)})
    print(json.dumps(res[-1]))
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
