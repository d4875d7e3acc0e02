"""(2) Trajectory visibility tables (rt::trajectory_vis_table, src/vistable.cpp:822-960)
on the GPU vs the compiled reference's rows (tests/golden/trajectories.json,
made by tests/golden/make_golden_traj.py): every row bit-identical — nodes,
parents, labels (incl. primes), blocking buildings and the bisected s values.
Plus the reference's own known answers (proj/tests/test_vistable.cpp:181-236,
286-319) on the GPU rows, and the chain-reach primitive vs point tables."""
import json
import os

import numpy as np
import pytest

import golden_util as G
from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200._capi import UsageError, VisibilityError
from paper_2501_02747_b200.core import ENTRY_DTYPE, Scene, chain_reach, point_tables, trajectory_vis_table

CASES = json.load(open(os.path.join(G.GOLDEN, "trajectories.json")))


def case_scene(c):
    if c["scene"] == "config1":
        soup = scenes.workload(1).scene
        return soup, None
    if "faces" in c:
        faces = c["faces"]
        off = np.zeros(len(faces) + 1, np.int32)
        off[1:] = np.cumsum([len(f["pts"]) for f in faces])
        soup = scenes.FacetSoup(ids=[f["id"] for f in faces], vert_off=off,
                                verts=np.array([p for f in faces for p in f["pts"]], np.float64),
                                building=np.array([f["building"] for f in faces], np.int32), name=c["scene"])
        return soup, [""] * len(faces)
    d = G.load(c["scene"])
    return G.soup(d), [f["label_xy"] for f in d["faces"]]


def entries_of(c):
    e = np.zeros(len(c["entries"]), ENTRY_DTYPE)
    for k, row in enumerate(c["entries"]):   # [order, chain..., plane]
        ch = list(row[1:-1]) + [0] * 5
        e[k] = (row[0], ch[:5], row[-1])
    return e


def run_case(c, sc=None):
    soup, labels = case_scene(c)
    own = sc is None
    sc = sc or Scene(soup)
    try:
        return trajectory_vis_table(sc, c["waypoints"], entries_of(c), c["max_order"], soup.ids, labels,
                                    soup.building, c["building_names"], return_stats=True)
    finally:
        if own:
            sc.close()


def expected_rows(c):
    out = []
    for r in c["rows"]:
        r = dict(r)
        r["s_start"] = float.fromhex(r["s_start"])
        r["s_end"] = float.fromhex(r["s_end"])
        out.append(r)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(CASES)), ids=[f"{c['scene']}-o{c['max_order']}-{i}" for i, c in enumerate(CASES)])
def test_trajectory_table_vs_reference(k):
    c = CASES[k]
    got, st = run_case(c)
    exp = expected_rows(c)
    assert len(got) == len(exp)
    for g, e in zip(got, exp):
        assert g == e, (g, e)
    assert st["pairs"] >= 2


@pytest.mark.gpu
def test_drive_by_known_answers():
    """proj/tests/test_vistable.cpp:181-236 on the GPU rows: 18 rows, every
    labelled boundary within kBoundaryTolerance of 10/3, 4, 46 or 140/3; the
    wall W_s seen on [0, 10/3] and [140/3, 50]; corner nodes blocked by K;
    order-2 rows hang off W_s -> K_n."""
    c = next(c for c in CASES if c["scene"] == "screened_wall" and c["max_order"] == 2)
    rows, _ = run_case(c)
    assert len(rows) == 18
    expected = [10 / 3, 4.0, 46.0, 140 / 3]
    events = 0
    for e in rows:
        assert e["s_start"] < e["s_end"]
        for lab, s in ((e["label_start"], e["s_start"]), (e["label_end"], e["s_end"])):
            if lab != "-":
                assert min(abs(s - x) for x in expected) <= 1e-3
                events += 1
        if "#" in e["node"]:
            assert e["blockage"] == "K"
        if e["order"] == 2:
            assert e["node"] == "K_n" and e["parent"] == "W_s"
    assert events == 18
    wall = sorted((e["s_start"], e["s_end"]) for e in rows if e["node"] == "W_s")
    assert len(wall) == 2
    assert wall[0][0] == pytest.approx(0.0) and abs(wall[0][1] - 10 / 3) <= 1e-3
    assert abs(wall[1][0] - 140 / 3) <= 1e-3 and wall[1][1] == pytest.approx(50.0)


@pytest.mark.gpu
def test_primed_vertical_boundary():
    """proj/tests/test_vistable.cpp:286-319: three W3_s rows ending at s = 4
    with a primed label; corner rows blocked by K2."""
    c = next(c for c in CASES if c["scene"] == "primed")
    rows, _ = run_case(c)
    assert len(rows) == 3
    for e in rows:
        assert e["node"].startswith("W3_s")
        assert e["s_start"] == pytest.approx(0.0) and abs(e["s_end"] - 4.0) <= 1e-3
        assert e["label_start"] == "-" and e["label_end"].endswith("'")
        if "#" in e["node"]:
            assert e["blockage"] == "K2"


@pytest.mark.gpu
def test_trajectory_errors():
    c = next(c for c in CASES if c["scene"] == "screened_wall")
    soup, labels = case_scene(c)
    with Scene(soup) as sc:
        with pytest.raises(VisibilityError, match="at least two distinct waypoints"):
            trajectory_vis_table(sc, [[1, 2, 3], [1, 2, 3]], entries_of(c), 1, soup.ids, labels)
        with pytest.raises(VisibilityError, match="matrix holds orders up to 1, requested 2"):
            trajectory_vis_table(sc, c["waypoints"], entries_of(c), 2, soup.ids, labels, matrix_max_order=1)
        with pytest.raises(UsageError):
            trajectory_vis_table(sc, c["waypoints"], entries_of(c), 5, soup.ids, labels)


@pytest.mark.gpu
def test_chain_reach_matches_point_tables():
    """The paired query path (K4 task list + K5 paired) equals the dense
    point-table path on every (source, entry) of config 1."""
    c = next(c for c in CASES if c["scene"] == "config1" and c["max_order"] == 2)
    wl = scenes.workload(1)
    E = entries_of(c)
    rng = np.random.default_rng(3)
    sel = E[rng.choice(len(E), 2000, replace=False)]
    src = wl.tx[rng.integers(0, len(wl.tx), len(sel))]
    with Scene(wl.scene) as sc:
        reach, full, _ = chain_reach(sc, src, sel)
        for k in range(0, len(sel), 97):
            rows, fb, _, _ = point_tables(sc, src[k:k + 1], sel[k:k + 1])
            assert reach[k] == rows[0, 0] and full[k] == fb[0, 0], k
