"""GPU (through the C-ABI) vs the committed golden vectors of the reference:
every fixture scene (closed-shell reference fixtures and the config-1 soup)
through all three subsystems, bit-exact."""
import numpy as np
import pytest

import golden_util as G
from paper_2501_02747_b200.core import (Scene, Tracer, chain_triples, path_identity, point_regions_array,
                                        unpack_bits)

pytestmark = pytest.mark.gpu

FIX = ["two_buildings", "street_canyon", "screened_wall", "manhattan", "config1"]


@pytest.fixture(scope="module", params=FIX)
def fx(request):
    d = G.load(request.param)
    s = G.soup(d)
    sc = Scene(s)
    yield d, s, sc
    sc.close()


def test_matrix_B_bits(fx):
    d, s, sc = fx
    bits, _ = sc.pair_visibility("all")
    M = unpack_bits(bits, s.nfaces)
    pi, pj = G.pairs(s.nfaces)
    np.testing.assert_array_equal(M[pi, pj], G.kinds(d) != 2)


def test_matrix_A_admitted(fx):
    d, s, sc = fx
    bits, _ = sc.pair_visibility("prefiltered")
    np.testing.assert_array_equal(unpack_bits(bits, s.nfaces), G.admitted_matrix(d))


def test_verdicts_and_blockers(fx):
    d, s, sc = fx
    pi, pj = G.pairs(s.nfaces)
    sel = np.arange(len(pi)) if len(pi) < 4000 else np.arange(0, len(pi), 7)
    kind, blockers, _ = sc.pair_detail(pi[sel], pj[sel])
    np.testing.assert_array_equal(kind, G.kinds(d)[sel])
    exp = d.get("blockers", {})
    for q, k in enumerate(sel):
        key = f"{pi[k]},{pj[k]}"
        if key in exp:
            assert blockers[q] == sorted(exp[key]), key


def test_regions(fx):
    d, s, sc = fx
    src = np.array([G.unhex(r["source"]) for r in d["regions"]])
    arr, _ = point_regions_array(sc, src)
    for k, rec in enumerate(d["regions"]):
        for f, row in enumerate(rec["regions"]):
            exp = G.region_tuple(row)
            g = arr[k, f]
            got = (int(g["present"]), [int(x) for x in g["has"]], [int(x) for x in g["clipped"]],
                   [float(x) for x in g["sub"]])
            if exp[0] != 1:
                assert got[0] == exp[0], (k, f)
            else:
                assert got == exp, (k, f)


def test_chain_triples(fx):
    d, s, sc = fx
    sc.pair_visibility("prefiltered")
    tri, _ = chain_triples(sc)
    assert sorted(map(tuple, tri.tolist())) == sorted(map(tuple, d["triples"]))


def test_traces(fx):
    d, s, sc = fx
    sc.pair_visibility("prefiltered")
    tri, _ = chain_triples(sc)
    for order in sorted({t["order"] for t in d["traces"]}):
        ts = [t for t in d["traces"] if t["order"] == order]
        tr = Tracer(sc, order, triples=tri if order == 3 else None)
        tx = np.array([G.unhex(t["tx"]) for t in ts])
        rx = np.array([G.unhex(t["rx"]) for t in ts])
        paths, nodes, _ = tr.trace(tx, rx)
        tr.close()
        for q, t in enumerate(ts):
            got = sorted((path_identity(s.ids, p["faces"]), p["points"], p["length"]) for p in paths[q])
            exp = sorted((p["identity"], G.unhex(p["points"]), G.unhex(p["length"])) for p in t["paths"])
            assert got == exp, (order, q)
            assert nodes[q] == t["nodes"]
