"""Seeded synthetic layouts (SURVEY.md §8d "Synthetic inputs") and the
halo-padded chip tiler.

Polygons are emitted directly in the reference heal() canonical form
(boolean.cpp finalize_layer :413-427): CCW outers, lexicographically smallest
vertex first, no repeated / collinear vertices, polygons sorted by vertex
list, all pairwise disjoint and non-touching — so heal(layer) == layer and the
GPU rasterizer's healed-input precondition holds (checked against the
reference heal in tests/test_layouts.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Sequence

import numpy as np

from .api import Grid


def _rect(x0, y0, x1, y1):
    return np.array([[x0, y0], [x1, y0], [x1, y1], [x0, y1]], np.int64)


def _canon(polys: List[np.ndarray]) -> List[np.ndarray]:
    out = []
    for p in polys:
        p = np.asarray(p, np.int64)
        if len(p) == 4 and p[0, 0] == p[3, 0] == min(p[0, 0], p[1, 0]) and p[1, 0] == p[2, 0] != p[0, 0] \
                and p[0, 1] == p[1, 1] < p[2, 1] == p[3, 1]:
            out.append(p)  # _rect output: CCW, smallest vertex first, already canonical
            continue
        # drop consecutive duplicates and collinear vertices (normalize_chain)
        changed = True
        while changed and len(p) >= 3:
            changed = False
            keep = []
            n = len(p)
            for i in range(n):
                a, b, c = p[i - 1], p[i], p[(i + 1) % n]
                if (b == a).all():
                    changed = True
                    continue
                cr = int(b[0] - a[0]) * int(c[1] - a[1]) - int(b[1] - a[1]) * int(c[0] - a[0])
                if cr == 0:
                    changed = True
                    continue
                keep.append(b)
            p = np.array(keep, np.int64).reshape(-1, 2)
        if len(p) < 3:
            continue
        area2 = int(np.sum(p[:, 0] * np.roll(p[:, 1], -1) - np.roll(p[:, 0], -1) * p[:, 1]))
        if area2 < 0:
            p = p[::-1]
        i = min(range(len(p)), key=lambda k: (int(p[k, 0]), int(p[k, 1])))
        out.append(np.roll(p, -i, axis=0))
    out.sort(key=lambda q: [tuple(v) for v in q.tolist()])
    return out


def line_space_contacts(width_nm: int, height_nm: int, seed: int = 0, x0: int = 0, y0: int = 0,
                        dbu_per_nm: int = 1) -> List[np.ndarray]:
    """Vertical lines (width 16-24 nm, pitch 40-64 nm) broken into segments
    with 20-40 nm tip-to-tip gaps, plus 16x16 nm contacts in the spaces that
    are wide enough to keep >= 4 nm clearance.  Integer nm vertices."""
    rng = np.random.default_rng(seed)
    polys = []
    x = x0 + int(rng.integers(0, 32))
    xe = x0 + width_nm
    lines = []
    while x < xe:
        pitch = int(rng.integers(40, 65))
        w = int(rng.integers(16, 25))
        lines.append((x, min(x + w, xe), pitch))
        x += pitch
    for lx0, lx1, pitch in lines:
        if lx1 - lx0 < 4:
            continue
        y = y0 + int(rng.integers(0, 40))
        while y < y0 + height_nm:
            seg = int(rng.integers(60, 400))
            ya, yb = y, min(y + seg, y0 + height_nm)
            if yb - ya >= 8:
                polys.append(_rect(lx0, ya, lx1, yb))
            y = yb + int(rng.integers(20, 41))
        # contacts in the space right of the line
        space0, space1 = lx1, lx0 + pitch
        if space1 - space0 >= 16 + 8 and space1 <= xe:
            cx = space0 + (space1 - space0 - 16) // 2
            cy = y0 + int(rng.integers(0, 80))
            while cy + 16 < y0 + height_nm:
                if rng.random() < 0.5:
                    polys.append(_rect(cx, cy, cx + 16, cy + 16))
                cy += int(rng.integers(40, 120))
    if dbu_per_nm != 1:
        polys = [p * dbu_per_nm for p in polys]
    return _canon(polys)


def curvilinear(width_nm: int, height_nm: int, seed: int = 0, x0: int = 0, y0: int = 0,
                cell_nm: int = 56) -> List[np.ndarray]:
    """All-angle blobs: ellipses (16-64 vertices, semi-axes 8-20 nm, random
    rotation) on a jittered grid of `cell_nm` cells, one per cell, disjoint."""
    rng = np.random.default_rng(seed)
    polys = []
    for cy in range(y0, y0 + height_nm - cell_nm + 1, cell_nm):
        for cx in range(x0, x0 + width_nm - cell_nm + 1, cell_nm):
            if rng.random() < 0.15:
                continue
            a = rng.uniform(8, 20)
            b = rng.uniform(8, 20)
            nv = int(rng.integers(16, 65))
            rot = rng.uniform(0, math.pi)
            mx = cx + cell_nm / 2 + rng.uniform(-3, 3)
            my = cy + cell_nm / 2 + rng.uniform(-3, 3)
            t = np.linspace(0, 2 * math.pi, nv, endpoint=False)
            px = mx + a * np.cos(t) * math.cos(rot) - b * np.sin(t) * math.sin(rot)
            py = my + a * np.cos(t) * math.sin(rot) + b * np.sin(t) * math.cos(rot)
            p = np.stack([np.rint(px), np.rint(py)], 1).astype(np.int64)
            polys.append(p)
    return _canon(polys)


def polygon_bboxes(polys: Sequence[np.ndarray]) -> np.ndarray:
    """[P, 4] int64 (xmin, ymin, xmax, ymax) per polygon."""
    if not len(polys):
        return np.zeros((0, 4), np.int64)
    xy, st = polygon_arrays(polys)
    idx = st[:-1]
    return np.stack([np.minimum.reduceat(xy[:, 0], idx), np.minimum.reduceat(xy[:, 1], idx),
                     np.maximum.reduceat(xy[:, 0], idx), np.maximum.reduceat(xy[:, 1], idx)], 1)


def chip_tiling(tile: int, tiles_x: int, tiles_y: int, halo: int, pitch_nm: float = 1.0,
                origin_nm=(0.0, 0.0)) -> "Tiling":
    """Tiling of a chip window into tiles_x x tiles_y halo-padded tiles of
    `tile` px (core = tile - 2 halo)."""
    core = tile - 2 * halo
    if core <= 0:
        raise ValueError("chip_tiling: halo leaves no core")
    chip = Grid(tiles_x * core, tiles_y * core, pitch_nm, origin_nm[0], origin_nm[1])
    return Tiling(chip, core, halo)


def chip_layout(tiling: "Tiling", seed: int = 0, curvilinear_layout: bool = False) -> List[np.ndarray]:
    """One seeded synthetic layout over the halo-extended chip window
    (integer nm; pitch 1 nm), heal-canonical."""
    ext = tiling.extended_grid()
    w = int(round(ext.nx * ext.pitch_nm))
    h = int(round(ext.ny * ext.pitch_nm))
    x0 = int(math.floor(ext.origin_x_nm))
    y0 = int(math.floor(ext.origin_y_nm))
    gen = curvilinear if curvilinear_layout else line_space_contacts
    return gen(w, h, seed=seed, x0=x0, y0=y0)


def polygon_arrays(polys: Sequence[np.ndarray]):
    """Flattened (xy [V,2] int64, starts [P+1] int64) for the C ABI."""
    if len(polys):
        xy = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int64).reshape(-1, 2) for p in polys]))
    else:
        xy = np.zeros((0, 2), np.int64)
    starts = np.zeros(len(polys) + 1, np.int64)
    starts[1:] = np.cumsum([len(p) for p in polys])
    return xy, starts


# ---------------------------------------------------------------------------
# halo-padded tiling
# ---------------------------------------------------------------------------
def blur_radius_px(resist_sigma_nm: float, pitch_nm: float) -> int:
    """Support of the reference resist blur: r = ceil(6 sigma_px) + 1
    (imaging.cpp:296-297; the min(N/2, .) cap does not bind at tile sizes)."""
    if resist_sigma_nm <= 0:
        return 0
    return int(math.ceil(6.0 * resist_sigma_nm / pitch_nm)) + 1


def optical_halo_px(wavelength_nm: float, na: float, pitch_nm: float, resist_sigma_nm: float,
                    ambit_lambda_over_na: float = 2.0, align: int = 64, minimum: int = 64) -> int:
    """Guard band of a halo-padded tile, in pixels: the optical ambit
    (`ambit_lambda_over_na` x lambda/NA, the coherent impulse response's main
    lobes) plus the resist-blur support (blur_radius_px), rounded up to
    `align` and at least `minimum` — the reference's window guard is this
    "pupil impulse-response support + resist sigma" band (SPEC.md:457,
    make_window opc.cpp:97-112).  EUV defaults (13.5 nm, NA 0.33, sigma 2 nm,
    1 nm pitch): 82 + 13 = 95 -> 128 px.

    The cores of halo-padded cyclic tiles equal a larger window's image only
    up to the hard-pupil tail, which decays slowly: measured on the oracle
    (tests/test_gpu_tiling.py) the core-vs-window aerial difference is a
    few 1e-2 of max I for halos from 64 to 384 px.  Tiles are therefore
    closed problems by definition (each cyclic window is imaged exactly, as
    the reference images each make_window window) and only cores are
    stitched."""
    ambit = ambit_lambda_over_na * wavelength_nm / na / pitch_nm
    h = int(math.ceil(ambit)) + blur_radius_px(resist_sigma_nm, pitch_nm)
    h = max(h, minimum)
    return -(-h // align) * align
@dataclass(frozen=True)
class Tiling:
    """Chip window `chip` split into tx x ty cores of `core` px; each tile is
    core + 2*halo px.  Tile (i, j) origin = chip origin + (i*core - halo)*pitch
    (exact: integer multiples of the pitch), so a tile raster is bitwise the
    matching sub-block of a raster of the halo-extended chip window."""
    chip: Grid
    core: int
    halo: int

    @property
    def tx(self) -> int:
        return -(-self.chip.nx // self.core)

    @property
    def ty(self) -> int:
        return -(-self.chip.ny // self.core)

    @property
    def n(self) -> int:
        return self.core + 2 * self.halo

    def __len__(self) -> int:
        return self.tx * self.ty

    def tile_ij(self, t: int):
        return t % self.tx, t // self.tx

    def tile_grid(self, t: int) -> Grid:
        i, j = self.tile_ij(t)
        p = self.chip.pitch_nm
        return Grid(self.n, self.n, p, self.chip.origin_x_nm + (i * self.core - self.halo) * p,
                    self.chip.origin_y_nm + (j * self.core - self.halo) * p)

    def extended_grid(self) -> Grid:
        """The halo-extended chip window every tile is a sub-block of."""
        p = self.chip.pitch_nm
        return Grid(self.tx * self.core + 2 * self.halo, self.ty * self.core + 2 * self.halo, p,
                    self.chip.origin_x_nm - self.halo * p, self.chip.origin_y_nm - self.halo * p)

    def tile_polygons(self, polys: Sequence[np.ndarray], t: int, dbu_per_nm: float = 1.0, bboxes=None):
        """Polygons whose bbox meets tile t's window, in layer order
        (`bboxes`: polygon_bboxes(polys), precomputed for many tiles)."""
        g = self.tile_grid(t)
        x0, y0 = g.origin_x_nm * dbu_per_nm, g.origin_y_nm * dbu_per_nm
        x1, y1 = x0 + g.nx * g.pitch_nm * dbu_per_nm, y0 + g.ny * g.pitch_nm * dbu_per_nm
        bb = polygon_bboxes(polys) if bboxes is None else bboxes
        hit = (bb[:, 2] >= x0) & (bb[:, 0] <= x1) & (bb[:, 3] >= y0) & (bb[:, 1] <= y1)
        return [polys[i] for i in np.nonzero(hit)[0]]

    def stitch(self, tiles: np.ndarray) -> np.ndarray:
        """Core regions of [T, n, n] tile images -> chip image [ny, nx]."""
        h, c = self.halo, self.core
        out = np.zeros((self.ty * c, self.tx * c), tiles.dtype)
        for t in range(len(self)):
            i, j = self.tile_ij(t)
            out[j * c:(j + 1) * c, i * c:(i + 1) * c] = tiles[t, h:h + c, h:h + c]
        return out[:self.chip.ny, :self.chip.nx]
