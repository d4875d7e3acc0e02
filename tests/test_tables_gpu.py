"""(2) (A)-semantics per-snapshot tables: point_vis_table rows from the GPU
regions + beam cascade vs the compiled reference (order 1 and 2 entries),
the street-canyon published rows, and the batched sightline_clear primitive."""
import numpy as np
import pytest

import golden_util as G
from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import ENTRY_DTYPE, Scene, point_tables, point_vis_table, segments_clear

pytestmark = pytest.mark.gpu


def entries_of(ents, max_order):
    out = [(e["order"], e["chain"] + [0] * (5 - len(e["chain"])), e["plane"]) for e in ents
           if e["order"] <= max_order]
    return np.array(out, dtype=ENTRY_DTYPE)


def test_point_vis_table_config1_vs_reference(oracle_built):
    if not oracle_built.have_ref():
        pytest.skip("oracle/_ref not built")
    wl = scenes.workload(1)
    soup = wl.scene
    r = oracle_built.RefOracle(soup)
    m = r.build_matrix(2)
    ents = r.matrix_entries(m)
    E = entries_of(ents, 2)
    ids = soup.ids
    srcs = list(wl.tx[::9]) + [wl.rx[0]]
    with Scene(soup) as sc:
        for src in srcs:
            for order in (1, 2):
                sel = E[E["order"] <= order]
                got = point_vis_table(sc, src, sel, ids)
                exp = r.point_vis_table(m, np.asarray(src), order)
                exp_rows = [{"order": x["order"], "chain": [ids[f] for f in x["chain"]], "aim": ids[x["aim"]],
                             "plane": x["plane"], "verdict": "Full" if x["verdict"] == 0 else "Partial",
                             "ref_display": x["ref_display"], "aim_display": x["aim_display"]} for x in exp]
                assert got == exp_rows, (src, order)


def test_street_canyon_published_rows():
    """proj/tests/test_vistable.cpp:98-128 / acceptance.cpp:209-228:
    {AB->EF, AC'->EG, AC'->EI, AC'->CG, EI->AC'} from (5, 28, 11)."""
    d = G.load("street_canyon")
    s = G.soup(d)
    E = np.array([(1, [e["ref"], e["aim"], 0, 0, 0], e["plane"]) for e in d["matrix1"]], dtype=ENTRY_DTYPE)
    labels = [(f["label_xy"], f["label_vert"]) for f in d["faces"]]
    with Scene(s) as sc:
        rows = point_vis_table(sc, [5.0, 28.0, 11.0], E, s.ids, labels)
    pairs = sorted((r["ref_display"], r["aim_display"]) for r in rows)
    assert pairs == sorted([("AB", "EF"), ("AC'", "EG"), ("AC'", "EI"), ("AC'", "CG"), ("EI", "AC'")])
    for r in rows:
        if r["ref_display"] == "AB":
            assert r["verdict"] == "Full" and r["plane"] == 0
        if r["ref_display"] == "AC'":
            assert r["verdict"] == "Partial" and r["plane"] == 1


def test_segments_clear_vs_oracle(oracle_built):
    wl = scenes.workload(1)
    soup = wl.scene
    o = oracle_built.Oracle(soup)
    rng = np.random.default_rng(11)
    # face vertices (MobileSampler vertex keys) and random street points
    verts = soup.verts[rng.choice(len(soup.verts), 300)]
    a = np.repeat(wl.tx[::10], 30, axis=0)[:300]
    b = verts
    with Scene(soup) as sc:
        clear, st = segments_clear(sc, a, b)
    for k in range(len(a)):
        hit = any(o.lib().vo_segment_hits_face(o.h, np.ascontiguousarray(a[k]), np.ascontiguousarray(b[k]), f)
                  for f in range(soup.nfaces))
        assert clear[k] == (not hit), k


def test_point_tables_full_bits_consistent():
    """Order-1 rows exist exactly where the head face has a region; Full
    exactly where that region is unclipped in the entry's plane."""
    wl = scenes.workload(1)
    d = G.load("config1")
    E = np.array([(1, [e["ref"], e["aim"], 0, 0, 0], e["plane"]) for e in d["matrix1"]], dtype=ENTRY_DTYPE)
    with Scene(wl.scene) as sc:
        rows, full, regs, _ = point_tables(sc, wl.tx[:5], E, want_regions=True)
    for k in range(5):
        for e, ent in enumerate(E):
            r = regs[k, ent["chain"][0]]
            assert rows[k, e] == (r["present"] == 1)
            assert full[k, e] == (r["present"] == 1 and bool(r["has"][ent["plane"]]) and not r["clipped"][ent["plane"]])


@pytest.mark.parametrize("name,order", [("two_buildings", 3), ("street_canyon", 3), ("screened_wall", 4)])
def test_point_vis_table_higher_orders_vs_reference(oracle_built, name, order):
    """point_vis_table of orders 3 and 4 (the beam cascade through 3-4
    reflectors, src/vistable.cpp:404-467) vs the compiled reference."""
    if not oracle_built.have_ref():
        pytest.skip("oracle/_ref not built")
    d = G.load(name)
    soup = G.soup(d, with_buildings=False)
    r = oracle_built.RefOracle(soup)
    m = r.build_matrix(order)
    E = entries_of(r.matrix_entries(m), order)
    ids = soup.ids
    srcs = [G.unhex(x["source"]) for x in d["regions"]]
    with Scene(soup) as sc:
        for src in srcs:
            got = point_vis_table(sc, src, E, ids)
            exp = r.point_vis_table(m, np.asarray(src), order)
            exp_rows = [{"order": x["order"], "chain": [ids[f] for f in x["chain"]], "aim": ids[x["aim"]],
                         "plane": x["plane"], "verdict": "Full" if x["verdict"] == 0 else "Partial",
                         "ref_display": x["ref_display"], "aim_display": x["aim_display"]} for x in exp]
            assert got == exp_rows, src
