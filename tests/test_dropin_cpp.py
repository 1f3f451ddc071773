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
