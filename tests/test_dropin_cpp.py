"""GPU: the reference's OWN unmodified C++ test suites (test_imaging,
test_geometry, test_opc_ai, test_contour from /root/reference, built by
tests/cpp/build_dropin_tests.sh) linked against the drop-in
(host/litho_dropin.cpp replaces imaging.cpp + raster.cpp and contour.cpp's
marching_squares / measure_epe; everything else is the reference).  Every TEST_CASE runs its imaging / rasterization on the B200
through the C ABI, at the reference's own fp64 tolerances."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_bin")


@pytest.mark.parametrize("suite", ["test_imaging", "test_geometry", "test_opc_ai", "test_contour"])
def test_reference_suite_on_dropin(suite):
    exe = os.path.join(BIN, suite)
    if not os.path.exists(exe):
        pytest.skip("drop-in test binaries not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=1500)
    print(r.stdout[-4000:])
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 failed" in r.stdout


def test_reference_c_abi_image_and_ai_init_at_baseline_window(tmp_path):
    """The reference's own C ABI (litho_c.cpp, unmodified) on a 1024 x 1024 px
    window through the drop-in: litho_image (aerial, and resist at 30 nm
    defocus) and litho_ai_init.  The TCC support (6377) is above the
    reference's dense budget, so build_tcc returns the factored form and
    decompose_tcc takes the Abbe-SVD route; build_field_tensor's gradient is
    the GPU adjoint.  Files are checked against the oracle pipeline on the
    same kernels (the product's host generator == the factored route)."""
    import numpy as np

    import paper_2602_15036_b200 as L
    from oracle import oracle as O
    from oracle import refpy as R
    exe = os.path.join(BIN, "dropin_capi")
    if not os.path.exists(exe):
        pytest.skip("drop-in test binaries not built")
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    # the window litho_image used: make_window (opc.cpp:97-112), guard 24 nm, pitch 1
    lay = L.load_layout(str(tmp_path / "capi_layout.json"))
    polys = lay.layers[0][1]
    xy = np.concatenate(polys)
    x0, y0 = xy[:, 0].min() - 24, xy[:, 1].min() - 24
    n = int(np.ceil((xy[:, 0].max() + 24 - x0) / 1.0))
    assert n == 1024
    grid = L.Grid(n, n, 1.0, float(x0), float(y0))
    mask = R.rasterize(polys, n, n, 1.0, float(x0), float(y0), 1.0)
    model = L.OpticalModel(source=L.make_annular_source(0.4, 0.8, 21))
    O.set_threads(os.cpu_count() or 1)
    g0, aerial = L.read_aimg(str(tmp_path / "capi_aerial.aimg"))
    assert (g0.nx, g0.ny, g0.pitch_nm) == (1024, 1024, 1.0)
    ks = L.build_socs_kernels(model, grid, [0.0], energy_floor=0.995)
    want = O.image_socs(mask, ks.weights[0], ks.support, ks.values[0])
    assert np.abs(aerial - want).max() <= 1e-9 * np.abs(want).max()
    _, resist = L.read_aimg(str(tmp_path / "capi_resist.aimg"))
    ks30 = L.build_socs_kernels(model, grid, [30.0], energy_floor=0.995)
    want_r = O.gaussian_blur(O.image_socs(mask, ks30.weights[0], ks30.support, ks30.values[0], dose=1.1), 2.0, 1.0)
    assert np.abs(resist - want_r).max() <= 1e-9 * np.abs(want_r).max()
    _, m0 = L.read_aimg(str(tmp_path / "capi_ai_m0.aimg"))
    _, grad = L.read_aimg(str(tmp_path / "capi_ai_grad.aimg"))
    assert np.array_equal(m0, mask)
    g_want = O.weighted_gradient(mask, ks.weights[0], ks.support, ks.values[0], None, dose=1.0)
    # build_field_tensor normalises the channel to [0, 1] (ai.cpp:46-58)
    g_want = (g_want - g_want.min()) / (g_want.max() - g_want.min())
    assert np.abs(grad - g_want).max() <= 1e-9
