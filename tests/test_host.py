"""CPU: the C-ABI boundary (library loads, exports every declared symbol,
error/status mapping), the host kernel generator against the reference's
build_tcc/decompose_tcc, synthetic layouts, halo tiling, and the multi-rank
sharding logic (world_size 2, gloo)."""
import os
import re

import numpy as np
import pytest

import paper_2602_15036_b200 as L
from paper_2602_15036_b200 import _lib, chip
from paper_2602_15036_b200 import layouts as LY
from oracle import oracle as O
from oracle import refpy as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "lithogpu.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lithogpu_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    import ctypes
    syms = header_symbols()
    assert len(syms) >= 25
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED), set(syms) ^ set(_lib.EXPORTED)


def test_status_mapping_without_gpu():
    import ctypes as C
    lib = _lib.lib()
    assert lib.lithogpu_ctx_create(0, None) == _lib.ERR_USAGE
    assert b"null" in lib.lithogpu_last_error()
    h = C.c_void_p()
    rc = lib.lithogpu_ctx_create(0, C.byref(h))
    if rc != _lib.OK:  # no GPU here: a CUDA failure must map to DOMAIN with a message
        assert rc == _lib.ERR_DOMAIN and b"CUDA" in lib.lithogpu_last_error()
    else:
        lib.lithogpu_ctx_destroy(h)
    assert lib.lithogpu_kernels_create(None, None, 0, 1, 1, None, 1, None, None, None) == _lib.ERR_USAGE
    assert lib.lithogpu_ilt_run(None, 1, None, None) == _lib.ERR_USAGE
    # contour / EPE / evaluate_epe / AIMG / GPU kernel generation entry points
    assert lib.lithogpu_marching_squares(None, None, None, 0.5, None) == _lib.ERR_USAGE
    assert lib.lithogpu_contours_size(None, None, None) == _lib.ERR_USAGE
    assert lib.lithogpu_contours_get(None, None, None, None) == _lib.ERR_USAGE
    assert lib.lithogpu_measure_epe(None, None, 1, 1.0, None, None) == _lib.ERR_USAGE
    assert lib.lithogpu_measure_epe_loops(None, None, 0, None, None, None, 1, 1.0, None, None) == _lib.ERR_USAGE
    assert lib.lithogpu_evaluate_epe(None, 0, 1, None, 1, 1.0, 2.0, 0.25, None, 0, 1.0, None, None,
                                     None) == _lib.ERR_USAGE
    assert lib.lithogpu_write_aimg(None, None, 1, None, None, 1) == _lib.ERR_USAGE
    assert lib.lithogpu_read_aimg(None, b"x", None, None, None, None) == _lib.ERR_USAGE
    assert lib.lithogpu_socs_kernels_gpu(None, 8, 8, 1.0, 13.5, 0.33, 0, None, 0, 1, None, 0, None, 0, 1.0, 1,
                                         None, None, None, None) == _lib.ERR_USAGE
    assert lib.lithogpu_kernels_fast_order(None, None) == _lib.ERR_USAGE
    assert lib.lithogpu_kernels_fast_stacks(None, None) == _lib.ERR_USAGE
    lib.lithogpu_contours_destroy(None)  # null-safe
    with pytest.raises(_lib.LithoUsageError):
        _lib.check(_lib.ERR_USAGE)


def test_source_matches_reference():
    for gn in (5, 7, 21):
        assert np.array_equal(L.make_annular_source(0.4, 0.8, gn), R.source(0.4, 0.8, gn))
    with pytest.raises(ValueError):
        L.make_annular_source(0.8, 0.4)


@pytest.mark.parametrize("n,pitch,focus", [(12, 4.0, 0.0), (16, 4.0, 30.0), (24, 4.0, -40.0), (32, 2.0, 20.0)])
def test_kernel_generator_matches_reference(n, pitch, focus):
    """Abbe-SVD kernels == reference build_tcc + decompose_tcc: same support
    (order included), same eigenvalues, and full rank reproduces the
    reference's Hopkins image (test_imaging.cpp:157-171)."""
    model = L.OpticalModel(source=L.make_annular_source(0.4, 0.8, 7))
    g = L.Grid(n, n, pitch)
    ks = L.build_socs_kernels(model, g, [focus], energy_floor=1.0)
    rk = R.RefKernels(n, n, pitch, focus=focus, energy_floor=1.0, full_rank=True)
    assert np.array_equal(ks.support, rk.support)
    k = min(ks.order(), 6)
    assert np.allclose(ks.weights[0][:k], rk.weights[:k], rtol=1e-9, atol=1e-12)
    mask = np.random.default_rng(n).random((n, n))
    img = O.image_socs(mask, ks.weights[0], ks.support, ks.values[0])
    hop = rk.hopkins(mask)
    assert np.abs(img - hop).max() / np.abs(hop).max() < 1e-9


def test_kernel_generator_truncation_semantics():
    model = L.OpticalModel(source=L.make_annular_source(0.4, 0.8, 7))
    g = L.Grid(16, 16, 4.0)
    one = L.build_socs_kernels(model, g, [0.0], k_fixed=1)
    assert one.order() == 1
    fl = L.build_socs_kernels(model, g, [0.0], energy_floor=0.95)
    assert fl.captured_energy[0] >= 0.95
    w = fl.weights[0]
    assert np.all(w >= 0) and np.all(np.diff(w) <= 0)
    # phase convention: largest-magnitude component real positive (imaging.cpp:192-196)
    for v in fl.values[0]:
        i = int(np.argmax(np.abs(v)))
        assert abs(v[i].imag) < 1e-12 and v[i].real > 0


@pytest.mark.parametrize("gen", [LY.line_space_contacts, LY.curvilinear])
def test_layouts_are_heal_canonical(gen):
    polys = gen(384, 256, seed=11, x0=-50, y0=20)
    healed = R.heal(polys)
    assert len(healed) == len(polys)
    assert all(np.array_equal(a, b) for a, b in zip(healed, polys))


def test_tile_halo_indexing_bit_exact():
    """Every tile raster is bitwise the matching sub-block of the raster of
    the halo-extended chip window."""
    chip_grid = L.Grid(200, 150, 1.0, -40.0, 10.0)
    tl = LY.Tiling(chip_grid, core=64, halo=16)
    polys = LY.line_space_contacts(260, 210, seed=3, x0=-70, y0=-20)
    ext = tl.extended_grid()
    full = O.rasterize(polys, ext.nx, ext.ny, ext.pitch_nm, ext.origin_x_nm, ext.origin_y_nm)
    assert len(tl) == tl.tx * tl.ty == 4 * 3
    for t in range(len(tl)):
        g = tl.tile_grid(t)
        tile = O.rasterize(tl.tile_polygons(polys, t), g.nx, g.ny, g.pitch_nm, g.origin_x_nm, g.origin_y_nm)
        i, j = tl.tile_ij(t)
        sub = full[j * tl.core:j * tl.core + tl.n, i * tl.core:i * tl.core + tl.n]
        assert np.array_equal(tile, sub), t
    # stitching the cores reproduces the chip window
    tiles = np.stack([O.rasterize(tl.tile_polygons(polys, t), tl.n, tl.n, 1.0, tl.tile_grid(t).origin_x_nm,
                                  tl.tile_grid(t).origin_y_nm) for t in range(len(tl))])
    st = tl.stitch(tiles)
    h = tl.halo
    assert np.array_equal(st, full[h:h + chip_grid.ny, h:h + chip_grid.nx])


@pytest.mark.parametrize("n,world", [(256, 8), (256, 3), (7, 4), (3, 5)])
def test_shard_partition(n, world):
    parts = [chip.shard(n, world, r) for r in range(world)]
    seen = [t for p in parts for t in p]
    assert seen == list(range(n))
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= 1


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = chip.shard(10, world, rank)
    cost = torch.tensor([float(sum(t * t for t in mine))], dtype=torch.float64)
    gmax = torch.tensor([float(max(mine) if len(mine) else 0)], dtype=torch.float64)
    chip.allreduce_scalars(cost, gmax)
    q.put((rank, list(mine), cost.item(), gmax.item()))
    dist.destroy_process_group()


def test_two_rank_cost_allreduce_gloo():
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[0][1] + res[1][1] == list(range(10))
    want = float(sum(t * t for t in range(10)))
    assert res[0][2] == res[1][2] == want
    assert res[0][3] == res[1][3] == 9.0


def _segment_worker(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist

    from paper_2602_15036_b200 import chip
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = list(chip.shard(5, world, rank))
    state = {"it": 0}

    def run_segment(k, cost, gmax):  # fake solver: cost = (iter+1)*(tile+1), decreasing gmax
        for j in range(k):
            it = state["it"] + j
            for a, t in enumerate(mine):
                cost[j, a] = (it + 1) * (t + 1) if it < 3 else 4.0 * (t + 1)
                gmax[j, a] = 1.0 / (it + 1) + t
        state["it"] += k

    c_all, g_all = chip.segmented_ilt(run_segment, 7, len(mine), sync_every=3)
    state["it"] = 0
    c_tol, _ = chip.segmented_ilt(run_segment, 7, len(mine), sync_every=2, tol=1e-12)
    q.put((rank, c_all.tolist(), g_all.tolist(), len(c_tol)))
    dist.destroy_process_group()


def test_segmented_ilt_allreduce_gloo():
    """per-iteration global cost / max|grad| of the sharded chip ILT, reduced
    once per segment, with the tolerance stop (world_size 2, gloo)."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_segment_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    tiles_sum = sum(t + 1 for t in range(5))
    want = [(it + 1) * tiles_sum if it < 3 else 4.0 * tiles_sum for it in range(7)]
    assert res[0][1] == res[1][1] == want
    assert res[0][2] == res[1][2] == [1.0 / (it + 1) + 4 for it in range(7)]
    # segments of 2: costs 15, 30 | 45, 60 | 60, 60 -> stop after the third segment
    assert res[0][3] == res[1][3] == 6


def test_layout_json_loader_round_trip_and_errors(tmp_path):
    """lithogpu_layout_load (reference load_layout, io.cpp:53-116): the
    reference JSON format in, flattened polygon buffers out; the reference's
    validation messages."""
    import json
    polys = LY.line_space_contacts(300, 200, seed=2)
    doc = {"format_version": 1, "dbu_per_nm": [2, 1],
           "layers": [{"name": "M1", "polygons": [p.tolist() for p in polys]}, {"name": "empty", "polygons": []}]}
    p = tmp_path / "l.json"
    p.write_text(json.dumps(doc, indent=1))
    lay = L.load_layout(str(p))
    assert (lay.dbu_num, lay.dbu_den) == (2, 1) and lay.dbu_per_nm() == 2.0
    assert [n for n, _ in lay.layers] == ["M1", "empty"]
    got = lay.layers[0][1]
    assert len(got) == len(polys) and all(np.array_equal(a, b) for a, b in zip(got, polys))
    assert lay.layers[1][1] == []
    bad = [({"format_version": 2, "dbu_per_nm": 1, "layers": []}, "missing or unsupported format_version"),
           ({"format_version": 1, "dbu_per_nm": 1, "layers": [], "x": 1}, 'unknown key "x"'),
           ({"format_version": 1, "layers": []}, "missing dbu_per_nm"),
           ({"format_version": 1, "dbu_per_nm": 0, "layers": []}, "dbu_per_nm must be positive"),
           ({"format_version": 1, "dbu_per_nm": 1, "layers": [{"name": "a", "polygons": [[[0, 0], [1.5, 0], [1, 1]]]}]},
            "non-integer coordinate in"),
           ({"format_version": 1, "dbu_per_nm": 1, "layers": [{"name": "a", "polygons": [[[0, 0, 1]]]}]},
            "bad vertex in")]
    for i, (d, msg) in enumerate(bad):
        q = tmp_path / f"bad{i}.json"
        q.write_text(json.dumps(d))
        with pytest.raises(RuntimeError, match=msg):
            L.load_layout(str(q))
    q = tmp_path / "malformed.json"
    q.write_text("{not json")
    with pytest.raises(RuntimeError, match="malformed JSON"):
        L.load_layout(str(q))
    with pytest.raises(RuntimeError, match="cannot open"):
        L.load_layout(str(tmp_path / "missing.json"))
