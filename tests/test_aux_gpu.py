"""(3) image_tree (proj/src/raytracer.cpp:458-486) and closest_diffraction_edge
(proj/src/vistable.cpp:545-561) on the GPU vs the compiled reference's
answers (tests/golden/aux.json, made by tests/golden/make_golden_aux.py) and
the reference's known-answer test (proj/tests/test_raytracer.cpp:297-329)."""
import json
import os

import numpy as np
import pytest

import golden_util as G
from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import Scene, closest_diffraction_edges, image_tree

pytestmark = pytest.mark.gpu
AUX = json.load(open(os.path.join(G.GOLDEN, "aux.json")))


def soup_of(name):
    return scenes.workload(1).scene if name == "config1" else G.soup(G.load(name))


@pytest.mark.parametrize("k", range(len(AUX["image_trees"])))
def test_image_tree_vs_reference(k):
    t = AUX["image_trees"][k]
    with Scene(soup_of(t["scene"])) as sc:
        nodes = image_tree(sc, t["source"], t["depth"])
    assert [n["face"] for n in nodes] == t["face"]
    assert [n["parent"] for n in nodes] == t["parent"]
    assert [n["depth"] for n in nodes] == t["node_depth"]
    assert [[float.fromhex(x) for x in p] for p in t["image"]] == [n["image"] for n in nodes]


def test_image_tree_front_side_known_answer():
    """proj/tests/test_raytracer.cpp:297-329: from (5,-5,2) at depth 2, two
    depth-1 nodes (B1_s, B2_s) and three depth-2 nodes."""
    s = soup_of("two_buildings")
    with Scene(s) as sc:
        nodes = image_tree(sc, [5, -5, 2], 2, ids=s.ids)
    d1 = [n for n in nodes if n["depth"] == 1]
    d2 = [n for n in nodes if n["depth"] == 2]
    assert len(d1) == 2 and len(d2) == 3
    assert {n["face"] for n in d1} == {"B1_s", "B2_s"}
    for n in d2:
        assert nodes[n["parent"]]["depth"] == 1 and nodes[n["parent"]]["face"] != n["face"]


@pytest.mark.parametrize("k", range(len(AUX["closest_edges"])))
def test_closest_edges_vs_reference(k):
    c = AUX["closest_edges"][k]
    d = G.load(c["scene"])
    with Scene(G.soup(d)) as sc:
        got = closest_diffraction_edges(sc, c["receivers"], d["edges"])
    assert got.tolist() == c["edge"]


DIFF = AUX["diffraction_traces"]


@pytest.mark.parametrize("k", range(len(DIFF)), ids=[f"{t['scene']}-o{t['order']}-{i}" for i, t in enumerate(DIFF)])
def test_trace_with_diffraction_vs_reference(k):
    """TraceAccelerator::trace(tx, rx, allow_diffraction=true): the receiver's
    closest edge adds the Fermat-point sequences; path identities, points,
    lengths and the node / sequence counters equal the reference's."""
    from paper_2501_02747_b200._capi import PlacementError
    from paper_2501_02747_b200.core import Tracer, chain_triples, path_identity
    t = DIFF[k]
    d = G.load(t["scene"])
    s = G.soup(d)
    with Scene(s) as sc:
        bits, _ = sc.pair_visibility("prefiltered")
        tri, _ = chain_triples(sc, bits)
        tr = Tracer(sc, t["order"], admitted_bits=bits, triples=tri, edges=d["edges"])
        if "error" in t:
            with pytest.raises(PlacementError, match=t["error"]):
                tr.trace([t["tx"]], [t["rx"]], allow_diffraction=True)
            return
        paths, nodes, st = tr.trace([t["tx"]], [t["rx"]], allow_diffraction=True)
    got = sorted([{"identity": path_identity(s.ids, p["faces"], d["edges"][p["edge"]]["id"] if p["edge"] >= 0 else None),
                   "points": [float(x).hex() for x in p["points"]], "length": float(p["length"]).hex()}
                  for p in paths[0]], key=lambda p: p["identity"])
    assert got == t["paths"]
    assert int(nodes[0]) == t["nodes"]
    assert st["sequences"] == t["sequences"]


BRUTE = AUX["brute_traces"]


@pytest.mark.parametrize("k", range(len(BRUTE)),
                         ids=[f"{t['scene']}-o{t['order']}-d{int(t['diffraction'])}-{i}" for i, t in enumerate(BRUTE)])
def test_brute_force_trace_vs_reference(k):
    """brute_force_trace (proj/src/raytracer.cpp:488-493) on the GPU: the
    unpruned, unfiltered tree (N(N-1)^(d-1) nodes) gives the reference's path
    set and counters; and the accelerated trace finds the same path set
    (proj/tests/test_raytracer.cpp:134-168, acceptance c1)."""
    from paper_2501_02747_b200.core import Tracer, brute_force_trace, chain_triples, path_identity
    t = BRUTE[k]
    d = G.load(t["scene"])
    s = G.soup(d)

    def ident(p):
        return path_identity(s.ids, p["faces"], d["edges"][p["edge"]]["id"] if p["edge"] >= 0 else None)

    with Scene(s) as sc:
        paths, nodes, st = brute_force_trace(sc, [t["tx"]], [t["rx"]], t["order"], t["diffraction"], d["edges"])
        got = sorted([{"identity": ident(p), "points": [float(x).hex() for x in p["points"]],
                       "length": float(p["length"]).hex()} for p in paths[0]], key=lambda p: p["identity"])
        assert got == t["paths"]
        assert int(nodes[0]) == t["nodes"] and st["sequences"] == t["sequences"]
        bits, _ = sc.pair_visibility("prefiltered")
        tri, _ = chain_triples(sc, bits)
        acc = Tracer(sc, t["order"], admitted_bits=bits, triples=tri, edges=d["edges"])
        apaths, _, _ = acc.trace([t["tx"]], [t["rx"]], allow_diffraction=t["diffraction"])
        assert sorted(ident(p) for p in apaths[0]) == [p["identity"] for p in t["paths"]]


def _route_position(wps, s):
    """Trajectory::position_at (proj/src/scene.cpp:459-469) in float64."""
    w = np.asarray(wps, np.float64)
    if s <= 0:
        return w[0]
    for i in range(len(w) - 1):
        d = w[i + 1] - w[i]
        seg = np.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])
        if s <= seg:
            return w[i] + (w[i + 1] - w[i]) * (s / seg)
        s -= seg
    return w[-1]


@pytest.mark.parametrize("k", range(len(AUX["dynamic"])),
                         ids=[f"{t['scene']}-d{int(t['diffraction'])}" for t in AUX["dynamic"]])
def test_resolve_keys_vs_reference_dynamic_trace(k):
    """dynamic_trace's re-solve (proj/src/raytracer.cpp:554-570, 590-643): the
    keys of each coherence segment's retraced sample, re-solved on the GPU at
    every later sample of the segment in ONE batched call, give the
    reference's paths (identity, points, length) bit for bit."""
    from paper_2501_02747_b200.core import resolve_keys, path_identity
    t = AUX["dynamic"][k]
    d = G.load(t["scene"])
    s = G.soup(d)
    fid = {f: i for i, f in enumerate(s.ids)}
    eid = {e["id"]: i for i, e in enumerate(d["edges"])}

    def key_of(ident):
        if ident == "LOS":
            return [], -1
        import re
        faces, edge = [], -1
        for kind, name in re.findall(r"(R|D):(.*?)(?=/(?:R|D):|$)", ident):   # edge ids contain '/'
            if kind == "R":
                faces.append(fid[name])
            else:
                edge = eid[name]
        return faces, edge

    seg_keys, tx, keys, expect = {}, [], [], []
    for smp in t["samples"]:
        if smp["retraced"]:
            seg_keys[smp["segment"]] = [key_of(p["identity"]) for p in smp["paths"]]
            continue
        tx.append(_route_position(t["waypoints"], float.fromhex(smp["s"])))
        keys.append(seg_keys[smp["segment"]])
        expect.append(smp["paths"])
    assert tx, "no re-solved samples"
    with Scene(s) as sc:
        got, st = resolve_keys(sc, np.array(tx), [t["rx"]], keys, d["edges"])
    for g, e in zip(got, expect):
        gp = sorted([{"identity": path_identity(s.ids, p["faces"], d["edges"][p["edge"]]["id"] if p["edge"] >= 0 else None),
                      "points": [float(x).hex() for x in p["points"]], "length": float(p["length"]).hex()} for p in g],
                    key=lambda p: p["identity"])
        assert gp == e


O4 = AUX["order4_traces"]


@pytest.mark.parametrize("k", range(len(O4)), ids=[f"{t['scene']}-d{int(t['diffraction'])}-{i}" for i, t in enumerate(O4)])
def test_trace_order4_vs_reference(k):
    """TraceAccelerator(max_refl = 4) (proj/include/rt/raytracer.hpp:96-118):
    depth-4 continuations follow the order-3 chains (Markov-2 growth of the
    order-2 triples); path sets and counters equal the reference's."""
    from paper_2501_02747_b200.core import Tracer, chain_triples, path_identity
    t = O4[k]
    if t["scene"] == "config1":
        s, edges = scenes.workload(1).scene, []
    else:
        d = G.load(t["scene"])
        s, edges = G.soup(d), d["edges"]
    with Scene(s) as sc:
        bits, _ = sc.pair_visibility("prefiltered")
        tri, _ = chain_triples(sc, bits)
        tr = Tracer(sc, 4, admitted_bits=bits, triples=tri, edges=edges)
        paths, nodes, st = tr.trace([t["tx"]], [t["rx"]], allow_diffraction=t["diffraction"])
    got = sorted([{"identity": path_identity(s.ids, p["faces"], edges[p["edge"]]["id"] if p["edge"] >= 0 else None),
                   "points": [float(x).hex() for x in p["points"]], "length": float(p["length"]).hex()}
                  for p in paths[0]], key=lambda p: p["identity"])
    assert got == t["paths"]
    assert int(nodes[0]) == t["nodes"] and st["sequences"] == t["sequences"]
