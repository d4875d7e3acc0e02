"""Seeded facet-soup generators for the five BASELINE configurations.

The generator is the single source of geometry: the oracle (C restatement and
the compiled reference behind its facet-soup adapter) and the CUDA path read
the very same float64 arrays, so RNG portability never matters.

Conventions:
  * one seed per config: ``2501027470 + k``; ``numpy.random.Generator(PCG64)``;
  * metres, float64; vertex rings wound CCW seen from outside, so the Newell
    normal (reference ``ConvexPolygon::from_points``, proj/src/geom.cpp:126-140)
    points outward; ground tiles face +z;
  * buildings are open shells (walls + roof, no base), walls emitted in the
    reference box order s, n, w, e (proj/src/scene.cpp:384-402), then the roof;
    ground tiles come last (the reference registers the ground face last,
    proj/src/scene.cpp:163-170);
  * footprints overlapping an earlier building are rejected by resampling;
    snapshot positions are kept off every footprint.

A :class:`FacetSoup` carries no building/edge topology: exactly what the
oracle's facet-soup adapter feeds the reference (no ``inside_building``, no
diffraction edges).  Closed-shell fixture scenes carry ``building`` indices.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence

import numpy as np

SEED_BASE = 2501027470


@dataclasses.dataclass
class FacetSoup:
    ids: List[str]
    vert_off: np.ndarray          # int32 [n+1]
    verts: np.ndarray             # float64 [total, 3]
    building: Optional[np.ndarray] = None   # int32 [n], -1 = none (None: pure soup)
    building_ids: Optional[List[str]] = None
    name: str = ""

    @property
    def nfaces(self) -> int:
        return len(self.ids)

    def face_points(self, i: int) -> np.ndarray:
        return self.verts[self.vert_off[i]:self.vert_off[i + 1]]


@dataclasses.dataclass
class Workload:
    config: int
    scene: FacetSoup
    tx: Optional[np.ndarray] = None     # [K, 3] float64 snapshot positions
    rx: Optional[np.ndarray] = None     # [K, 3] or [1, 3]
    trace_order: int = 0
    description: str = ""


class _Builder:
    def __init__(self) -> None:
        self.ids: List[str] = []
        self.rings: List[np.ndarray] = []

    def add(self, fid: str, pts: Sequence[Sequence[float]]) -> None:
        self.ids.append(fid)
        self.rings.append(np.asarray(pts, dtype=np.float64).reshape(-1, 3))

    def soup(self, name: str) -> FacetSoup:
        off = np.zeros(len(self.rings) + 1, dtype=np.int32)
        off[1:] = np.cumsum([len(r) for r in self.rings])
        verts = np.ascontiguousarray(np.concatenate(self.rings, axis=0))
        return FacetSoup(ids=list(self.ids), vert_off=off, verts=verts, name=name)


def _box(b: _Builder, bid: str, lo, hi) -> None:
    """Open box: the reference's make_box_building ring order without the base."""
    (lx, ly, lz), (hx, hy, hz) = lo, hi
    b.add(f"{bid}_s", [(lx, ly, lz), (hx, ly, lz), (hx, ly, hz), (lx, ly, hz)])
    b.add(f"{bid}_n", [(lx, hy, lz), (lx, hy, hz), (hx, hy, hz), (hx, hy, lz)])
    b.add(f"{bid}_w", [(lx, ly, lz), (lx, ly, hz), (lx, hy, hz), (lx, hy, lz)])
    b.add(f"{bid}_e", [(hx, ly, lz), (hx, hy, lz), (hx, hy, hz), (hx, ly, hz)])
    b.add(f"{bid}_roof", [(lx, ly, hz), (hx, ly, hz), (hx, hy, hz), (lx, hy, hz)])


def _tiles(b: _Builder, size: float, n: int) -> None:
    step = size / n
    for j in range(n):
        for i in range(n):
            x0, y0 = i * step, j * step
            x1, y1 = (i + 1) * step, (j + 1) * step
            b.add(f"T_{i}_{j}", [(x0, y0, 0.0), (x1, y0, 0.0), (x1, y1, 0.0), (x0, y1, 0.0)])


def _random_boxes(rng: np.random.Generator, size: float, count: int,
                  wlo=10.0, whi=30.0, hlo=10.0, hhi=40.0, keepout=None):
    """Axis-aligned footprints, centres uniform with the footprint inside the
    plane, overlaps (and keep-out hits) rejected by resampling."""
    rects = []
    while len(rects) < count:
        w, d = rng.uniform(wlo, whi), rng.uniform(wlo, whi)
        h = rng.uniform(hlo, hhi)
        cx = rng.uniform(w / 2, size - w / 2)
        cy = rng.uniform(d / 2, size - d / 2)
        lo = (cx - w / 2, cy - d / 2)
        hi = (cx + w / 2, cy + d / 2)
        if any(lo[0] < r[1][0] and r[0][0] < hi[0] and lo[1] < r[1][1] and r[0][1] < hi[1]
               for r in rects):
            continue
        if keepout is not None and keepout(lo, hi):
            continue
        rects.append((lo, hi, h))
    return rects


def _inside_any(rects, x: float, y: float, margin: float = 0.5) -> bool:
    return any(r[0][0] - margin <= x <= r[1][0] + margin and r[0][1] - margin <= y <= r[1][1] + margin
               for r in rects)


def _seg_hits_rect(p0, p1, lo, hi, margin: float) -> bool:
    """Conservative: does segment p0->p1 (xy) come within `margin` of the rect?"""
    lo = (lo[0] - margin, lo[1] - margin)
    hi = (hi[0] + margin, hi[1] + margin)
    t0, t1 = 0.0, 1.0
    d = (p1[0] - p0[0], p1[1] - p0[1])
    for k in range(2):
        if abs(d[k]) < 1e-12:
            if p0[k] < lo[k] or p0[k] > hi[k]:
                return False
            continue
        a = (lo[k] - p0[k]) / d[k]
        b = (hi[k] - p0[k]) / d[k]
        if a > b:
            a, b = b, a
        t0, t1 = max(t0, a), min(t1, b)
        if t0 > t1:
            return False
    return True


# ---------------------------------------------------------------------------
# Config 1 — small urban canyon (116 facets, 100 Tx snapshots, fixed Rx)
# ---------------------------------------------------------------------------

def config1(seed: int = SEED_BASE + 1) -> Workload:
    rng = np.random.Generator(np.random.PCG64(seed))
    size = 200.0
    # A straight "street" for the Tx track: keep a 6 m corridor clear.
    y_street = float(rng.uniform(40.0, 160.0))
    x0 = float(rng.uniform(20.0, 60.0))
    p0, p1 = (x0, y_street), (x0 + 99.0, y_street)
    rects = _random_boxes(rng, size, 20,
                          keepout=lambda lo, hi: _seg_hits_rect(p0, p1, lo, hi, 3.0))
    b = _Builder()
    for k, (lo, hi, h) in enumerate(rects):
        _box(b, f"B{k}", (lo[0], lo[1], 0.0), (hi[0], hi[1], h))
    _tiles(b, size, 4)
    soup = b.soup("config1")
    tx = np.array([[x0 + k * 1.0, y_street, 1.5] for k in range(100)], dtype=np.float64)
    while True:
        rxy = rng.uniform(10.0, size - 10.0, size=2)
        if not _inside_any(rects, rxy[0], rxy[1], 1.0):
            break
    rx = np.array([[rxy[0], rxy[1], 1.5]], dtype=np.float64)
    return Workload(1, soup, tx=tx, rx=rx, trace_order=2,
                    description="200 m plane, 4x4 tiles, 20 boxes; 100 Tx snapshots at 1 m, fixed Rx; order 2")


# ---------------------------------------------------------------------------
# Config 2 — medium city grid, matrix only (1,256 facets)
# ---------------------------------------------------------------------------

def config2(seed: int = SEED_BASE + 2) -> Workload:
    rng = np.random.Generator(np.random.PCG64(seed))
    size = 1000.0
    rects = _random_boxes(rng, size, 200)
    b = _Builder()
    for k, (lo, hi, h) in enumerate(rects):
        _box(b, f"B{k}", (lo[0], lo[1], 0.0), (hi[0], hi[1], h))
    _tiles(b, size, 16)
    return Workload(2, b.soup("config2"), description="1 km plane, 16x16 tiles, 200 boxes; matrix only")


# ---------------------------------------------------------------------------
# Config 3 — dynamic V2V street scene: Manhattan grid of 500 boxes
# ---------------------------------------------------------------------------

def _lognormal_height(rng: np.random.Generator) -> float:
    return float(min(100.0, rng.lognormal(mean=math.log(20.0), sigma=0.5)))


def config3(seed: int = SEED_BASE + 3) -> Workload:
    rng = np.random.Generator(np.random.PCG64(seed))
    size = 2000.0
    ncols, nrows = 25, 20           # 500 blocks
    # Street widths U[15, 30] for each street line (including the borders),
    # blocks share the remaining length equally.
    sx = rng.uniform(15.0, 30.0, size=ncols + 1)
    sy = rng.uniform(15.0, 30.0, size=nrows + 1)
    bw = (size - sx.sum()) / ncols
    bd = (size - sy.sum()) / nrows
    xs = [float(sx[: i + 1].sum() + i * bw) for i in range(ncols)]
    ys = [float(sy[: j + 1].sum() + j * bd) for j in range(nrows)]
    b = _Builder()
    k = 0
    for j in range(nrows):
        for i in range(ncols):
            h = _lognormal_height(rng)
            _box(b, f"B{k}", (xs[i], ys[j], 0.0), (xs[i] + bw, ys[j] + bd, h))
            k += 1
    _tiles(b, size, 16)
    soup = b.soup("config3")
    # Tx on a horizontal street (between block rows), Rx on a vertical street.
    jt = int(rng.integers(1, nrows))          # street line between rows jt-1 and jt
    ytx = ys[jt] - sy[jt] / 2.0
    ir = int(rng.integers(1, ncols))
    xrx = xs[ir] - sx[ir] / 2.0
    tx0 = float(rng.uniform(50.0, size - 1050.0))
    ry0 = float(rng.uniform(50.0, size - 1050.0))
    tx = np.array([[tx0 + s, ytx, 1.5] for s in range(1000)], dtype=np.float64)
    rx = np.array([[xrx, ry0 + s, 1.5] for s in range(1000)], dtype=np.float64)
    return Workload(3, soup, tx=tx, rx=rx, trace_order=3,
                    description="2 km Manhattan grid 25x20 blocks, 16x16 tiles; Tx/Rx 1000 snapshots each; order 3")


# ---------------------------------------------------------------------------
# Config 4/5 — large irregular city of convex prisms (~21k facets)
# ---------------------------------------------------------------------------

def _prism_city(rng: np.random.Generator, size: float, count: int, track):
    prisms = []   # (cx, cy, r, angles, h)
    cells = {}
    cell = 80.0

    def near(cx, cy, r):
        ix, iy = int(cx // cell), int(cy // cell)
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for (ox, oy, orr) in cells.get((ix + dx, iy + dy), ()):
                    if (cx - ox) ** 2 + (cy - oy) ** 2 < (r + orr) ** 2:
                        return True
        return False

    while len(prisms) < count:
        k = int(rng.integers(4, 9))
        r = float(rng.uniform(8.0, 40.0))
        ang = np.sort(rng.uniform(0.0, 2.0 * math.pi, size=k))
        h = _lognormal_height(rng)
        cx = float(rng.uniform(r, size - r))
        cy = float(rng.uniform(r, size - r))
        # Reject near-duplicate angles (degenerate wall) and overlaps.
        gaps = np.diff(np.concatenate([ang, [ang[0] + 2 * math.pi]]))
        if gaps.min() < 1e-3 or gaps.max() >= math.pi:
            continue
        if near(cx, cy, r):
            continue
        if track is not None and _seg_hits_rect(track[0], track[1], (cx - r, cy - r), (cx + r, cy + r), 6.0):
            continue
        prisms.append((cx, cy, r, ang, h))
        cells.setdefault((int(cx // cell), int(cy // cell)), []).append((cx, cy, r))
    return prisms


def _prism_soup(prisms, size: float, tiles: int, name: str) -> FacetSoup:
    b = _Builder()
    for n, (cx, cy, r, ang, h) in enumerate(prisms):
        fp = [(cx + r * math.cos(a), cy + r * math.sin(a)) for a in ang]   # CCW from above
        k = len(fp)
        for i in range(k):
            (ax, ay), (bx, by) = fp[i], fp[(i + 1) % k]
            b.add(f"P{n}_w{i}", [(ax, ay, 0.0), (bx, by, 0.0), (bx, by, h), (ax, ay, h)])
        for i in range(1, k - 1):
            b.add(f"P{n}_r{i - 1}", [(fp[0][0], fp[0][1], h), (fp[i][0], fp[i][1], h),
                                     (fp[i + 1][0], fp[i + 1][1], h)])
    _tiles(b, size, tiles)
    return b.soup(name)


def _config45_geometry(seed: int):
    rng = np.random.Generator(np.random.PCG64(seed))
    size = 4000.0
    # Train track along the diagonal (5 km fits only along a diagonal); the
    # generator keeps its corridor building-free.
    off = float(rng.uniform(-150.0, 150.0))
    start = (300.0 + off, 300.0 - off)
    d = (1.0 / math.sqrt(2.0), 1.0 / math.sqrt(2.0))
    L = 0.5 * 9999
    end = (start[0] + d[0] * L, start[1] + d[1] * L)
    prisms = _prism_city(rng, size, 2000, (start, end))
    return rng, size, prisms, start, d


def config4(seed: int = SEED_BASE + 4) -> Workload:
    _, size, prisms, _, _ = _config45_geometry(seed)
    return Workload(4, _prism_soup(prisms, size, 32, "config4"),
                    description="4 km plane, 32x32 tiles, 2000 convex prisms; matrix only")


def config5(seed: int = SEED_BASE + 4, snapshots: int = 10000) -> Workload:
    """Config-4 geometry (same seed), Tx on the diagonal track at z = 4 every
    0.5 m, Rx on a seeded helix between 50 m and 120 m altitude."""
    rng, size, prisms, start, d = _config45_geometry(seed)
    soup = _prism_soup(prisms, size, 32, "config5")
    tx = np.array([[start[0] + d[0] * 0.5 * k, start[1] + d[1] * 0.5 * k, 4.0]
                   for k in range(snapshots)], dtype=np.float64)
    hc = (float(rng.uniform(1500.0, 2500.0)), float(rng.uniform(1500.0, 2500.0)))
    hr = float(rng.uniform(300.0, 600.0))
    turns = 3.0
    rx = np.array([[hc[0] + hr * math.cos(2 * math.pi * turns * k / snapshots),
                    hc[1] + hr * math.sin(2 * math.pi * turns * k / snapshots),
                    50.0 + 70.0 * k / max(1, snapshots - 1)] for k in range(snapshots)],
                  dtype=np.float64)
    return Workload(5, soup, tx=tx, rx=rx, trace_order=3,
                    description="config-4 geometry; Tx track z=4 every 0.5 m, Rx helix 50-120 m; order 3")


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def workload(k: int, **kw) -> Workload:
    return CONFIGS[k](**kw)
