"""Edge cases of the hot path, GPU vs the CPU oracle (and the compiled
reference where built): ragged facets (3..8 vertices in one scene: the
MAXV = 8 record layout), degenerate scene sizes (1 and 2 facets), empty
batches (no sources / no snapshots), a blocker that hides a pair exactly, and
sources on a facet plane. Every comparison is bit-exact."""
import math

import numpy as np
import pytest

from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import Scene, Tracer, point_regions_array, unpack_bits

pytestmark = pytest.mark.gpu


def ragged_city(seed: int = 7, count: int = 10, size: float = 160.0):
    """Convex prisms with 4..8 walls whose roof is ONE k-gon (not
    fan-triangulated) plus a few triangular canopies, on a 2x2 tiled ground:
    facets of 3, 4, 5, 6, 7 and 8 vertices in one soup."""
    rng = np.random.Generator(np.random.PCG64(seed))
    b = scenes._Builder()
    placed = []
    while len(placed) < count:
        k = int(rng.integers(4, 9))
        r = float(rng.uniform(6.0, 16.0))
        cx, cy = float(rng.uniform(r + 2, size - r - 2)), float(rng.uniform(r + 2, size - r - 2))
        if any((cx - x) ** 2 + (cy - y) ** 2 < (r + rr + 3.0) ** 2 for x, y, rr in placed):
            continue
        ang = np.sort(rng.uniform(0.0, 2 * math.pi, k))
        gaps = np.diff(np.concatenate([ang, [ang[0] + 2 * math.pi]]))
        if gaps.min() < 0.05 or gaps.max() >= math.pi:
            continue
        h = float(rng.uniform(8.0, 30.0))
        n = len(placed)
        placed.append((cx, cy, r))
        fp = [(cx + r * math.cos(a), cy + r * math.sin(a)) for a in ang]
        for i in range(k):
            (ax, ay), (bx, by) = fp[i], fp[(i + 1) % k]
            b.add(f"P{n}_w{i}", [(ax, ay, 0.0), (bx, by, 0.0), (bx, by, h), (ax, ay, h)])
        b.add(f"P{n}_roof", [(x, y, h) for x, y in fp])
        if n % 3 == 0:   # a floating triangular canopy beside the prism
            z = h * 0.5
            b.add(f"P{n}_tri", [(cx + r + 1.0, cy, z), (cx + r + 1.0, cy + 4.0, z), (cx + r + 1.0, cy + 2.0, z + 3.0)])
    scenes._tiles(b, size, 2)
    return b.soup("ragged"), size


@pytest.fixture(scope="module")
def ragged():
    soup, size = ragged_city()
    nv = np.diff(soup.vert_off)
    assert nv.min() == 3 and nv.max() >= 7   # ragged indeed
    rng = np.random.default_rng(3)
    src = np.column_stack([rng.uniform(5, size - 5, 6), rng.uniform(5, size - 5, 6), rng.uniform(1.5, 40.0, 6)])
    return soup, src


def test_ragged_matrix_all_pairs(oracle_built, ragged):
    soup, _ = ragged
    n = soup.nfaces
    pi, pj = np.triu_indices(n, 1)
    kinds = oracle_built.Oracle(soup).occlusion_batch(pi.astype(np.int32), pj.astype(np.int32))
    with Scene(soup) as sc:
        bits, _ = sc.pair_visibility("all")
        M = unpack_bits(bits, n)
        assert np.array_equal(M, M.T)
        np.testing.assert_array_equal(M[pi, pj], kinds != 2)
        sel = np.arange(0, len(pi), 41)
        kind, blockers, _ = sc.pair_detail(pi[sel], pj[sel])
        o = oracle_built.Oracle(soup)
        for q, s in enumerate(sel):
            ek, eb = o.occlusion(int(pi[s]), int(pj[s]))
            assert (int(kind[q]), blockers[q]) == (ek, sorted(eb))


def test_ragged_matrix_prefiltered(oracle_built, ragged):
    soup, _ = ragged
    o = oracle_built.Oracle(soup)
    with Scene(soup) as sc:
        sc.pair_visibility("prefiltered")
        ci, cj, ad = sc.candidates()
    pi, pj = o.prefilter_all()
    np.testing.assert_array_equal(ci, pi)
    np.testing.assert_array_equal(cj, pj)
    if len(ci):
        kinds = o.occlusion_batch(ci, cj)
        assert set(np.nonzero(ad)[0]) <= set(np.nonzero(kinds != 2)[0])


def test_ragged_regions(oracle_built, ragged):
    soup, src = ragged
    o = oracle_built.Oracle(soup)
    with Scene(soup) as sc:
        arr, _ = point_regions_array(sc, src)
    for k in range(len(src)):
        for f in range(soup.nfaces):
            e = o.illuminated_region(src[k], f)
            g = arr[k, f]
            assert (int(g["present"]), [int(x) for x in g["has"]], [int(x) for x in g["clipped"]],
                    [float(x) for x in g["sub"]]) == (e["present"], e["has"], e["clipped"], e["sub"]), (k, f)
    assert (arr["present"] == 1).sum() > 0


def test_ragged_trace_order2(oracle_built, ragged):
    soup, src = ragged
    with Scene(soup) as sc:
        bits, _ = sc.pair_visibility("prefiltered")
        tr = Tracer(sc, 2, admitted_bits=bits)
        tx, rx = src[:3], src[3:6]
        paths, nodes, _ = tr.trace(tx, rx)
        tr.close()
    filt = oracle_built.chain_filter_arrays(soup.nfaces, unpack_bits(bits, soup.nfaces))
    o = oracle_built.Oracle(soup)
    key = lambda p: (tuple(p["faces"]), tuple(p["points"]), p["length"])
    for q in range(len(tx)):
        exp, est = o.trace(filt, 2, tx[q], rx[q])
        assert sorted(map(key, paths[q])) == sorted(map(key, exp))
        assert nodes[q] == est[0]


def _soup(rings):
    b = scenes._Builder()
    for i, r in enumerate(rings):
        b.add(f"F{i}", r)
    return b.soup("edge")


WALL_A = [(0, 0, 0), (10, 0, 0), (10, 0, 10), (0, 0, 10)]            # normal -y
WALL_B = [(0, -20, 0), (0, -20, 10), (10, -20, 10), (10, -20, 0)]     # normal +y, facing A
BLOCKER = [(-5, -10, -5), (-5, -10, 15), (15, -10, 15), (15, -10, -5)]  # between them, larger than both


def test_single_facet_scene(oracle_built):
    soup = _soup([WALL_A])
    with Scene(soup) as sc:
        bits, st = sc.pair_visibility("all")
        assert st["pairs"] == 0 and not bits.any()
        bits, st = sc.pair_visibility("prefiltered")
        assert st["candidates"] == 0 and not bits.any()
        src = np.array([[5.0, -3.0, 5.0], [5.0, 3.0, 5.0], [5.0, 0.0, 5.0]])   # front, back, on the plane
        arr, _ = point_regions_array(sc, src)
    o = oracle_built.Oracle(soup)
    for k in range(3):
        e = o.illuminated_region(src[k], 0)
        assert int(arr[k, 0]["present"]) == e["present"]
        assert [float(x) for x in arr[k, 0]["sub"]] == e["sub"]
    assert [int(arr[k, 0]["present"]) for k in range(3)] == [1, 0, -1]


def test_two_facets_and_exact_blocker(oracle_built):
    for rings, visible in (([WALL_A, WALL_B], True), ([WALL_A, WALL_B, BLOCKER], False)):
        soup = _soup(rings)
        o = oracle_built.Oracle(soup)
        with Scene(soup) as sc:
            bits, _ = sc.pair_visibility("all")
            M = unpack_bits(bits, soup.nfaces)
            kind, blockers, _ = sc.pair_detail([0], [1])
        ek, eb = o.occlusion(0, 1)
        assert bool(M[0, 1]) == (ek != 2) == visible
        assert (int(kind[0]), blockers[0]) == (ek, sorted(eb))
        if not visible:
            assert blockers[0] == [2]


def test_empty_batches():
    wl = scenes.workload(1)
    with Scene(wl.scene) as sc:
        arr, st = point_regions_array(sc, np.zeros((0, 3)))
        assert arr.shape == (0, sc.n)
        sc.pair_visibility("prefiltered")
        tr = Tracer(sc, 2)
        paths, nodes, st = tr.trace(np.zeros((0, 3)), np.zeros((0, 3)))
        tr.close()
        assert paths == [] and len(nodes) == 0 and st["nodes"] == 0
