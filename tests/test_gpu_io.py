"""AIMG tile I/O: files written from device tiles are
byte-identical to the reference write_aimg (io.cpp:317-330, oracle/_ref), and
read_aimg round-trips with the reference's header checks and messages."""
import os

import numpy as np
import pytest

import paper_2602_15036_b200 as L
from oracle import refpy as R

pytestmark = pytest.mark.gpu


def test_write_aimg_bytes_match_reference(ctx, tmp_path):
    import torch
    rng = np.random.default_rng(1)
    tiles = rng.standard_normal((3, 48, 64))
    g = L.Grid(64, 48, 0.75, 3.0, -2.0)
    ours = [str(tmp_path / f"t{i}.aimg") for i in range(3)]
    dev = torch.from_numpy(tiles).cuda()
    L.write_aimg(ours, g, dev, ctx)  # device tiles, pinned double buffer
    for i in range(3):
        ref = str(tmp_path / f"r{i}.aimg")
        R.write_aimg(ref, tiles[i], 0.75)
        assert open(ours[i], "rb").read() == open(ref, "rb").read()
    # f32 device tiles are widened to f64 on the device; host f64 path too
    L.write_aimg(ours, g, dev.float(), ctx)
    R.write_aimg(str(tmp_path / "r0.aimg"), tiles[0].astype(np.float32).astype(np.float64), 0.75)
    assert open(ours[0], "rb").read() == open(str(tmp_path / "r0.aimg"), "rb").read()
    L.write_aimg(ours[1], g, tiles[1], ctx)
    R.write_aimg(str(tmp_path / "r1.aimg"), tiles[1], 0.75)
    assert open(ours[1], "rb").read() == open(str(tmp_path / "r1.aimg"), "rb").read()


def test_read_aimg_roundtrip_and_errors(ctx, tmp_path):
    rng = np.random.default_rng(2)
    v = rng.random((33, 17))
    p = str(tmp_path / "a.aimg")
    R.write_aimg(p, v, 2.5)
    g, got = L.read_aimg(p, ctx)
    assert (g.nx, g.ny, g.pitch_nm, g.origin_x_nm) == (17, 33, 2.5, 0.0)
    assert np.array_equal(got, v)
    bad = str(tmp_path / "bad.aimg")
    open(bad, "wb").write(b"NOPE" + bytes(40))
    with pytest.raises(RuntimeError, match="not an AIMG file"):
        L.read_aimg(bad, ctx)
    trunc = str(tmp_path / "trunc.aimg")
    open(trunc, "wb").write(open(p, "rb").read()[:100])
    with pytest.raises(RuntimeError, match="truncated AIMG payload"):
        L.read_aimg(trunc, ctx)
    with pytest.raises(RuntimeError, match="cannot open"):
        L.read_aimg(str(tmp_path / "missing.aimg"), ctx)
    assert not os.path.exists(str(tmp_path / "missing.aimg"))
