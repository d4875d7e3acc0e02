"""Generate tests/golden/trajectories.json from the UNMODIFIED reference
(oracle/_ref): rt::trajectory_vis_table (proj/src/vistable.cpp:822-960) on
the reference's own route fixtures (proj/data/fixtures/route_*.json) over its
scene fixtures, the primed-label walk of proj/tests/test_vistable.cpp:286-319
(two box buildings), and the seeded config-1 soup along its Tx line.
Run in the build container (needs /root/reference):

    python tests/golden/make_golden_traj.py

Per case: the scene (a golden fixture name, or inline faces), building names,
waypoints, max_order, the matrix entries of order <= max_order in matrix order
([order, chain ids..., plane] — the input a caller hands the GPU path) and the
reference's rows, doubles as float.hex() for bit-exact comparison.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import bindings  # noqa: E402
from paper_2501_02747_b200 import scenes  # noqa: E402
from make_golden import FIXTURES, soup_from_ref  # noqa: E402


def route(name: str):
    with open(os.path.join(FIXTURES, name + ".json")) as fh:
        return [w[:3] for w in json.load(fh)["waypoints"]]


def box_faces(bid: str, lo, hi):
    """The closed box of proj/tests/test_vistable.cpp:24-42 (ids <bid>_<side>)."""
    (x0, y0, z0), (x1, y1, z1) = lo, hi
    return [(f"{bid}_s", [[x0, y0, z0], [x1, y0, z0], [x1, y0, z1], [x0, y0, z1]]),
            (f"{bid}_n", [[x0, y1, z0], [x0, y1, z1], [x1, y1, z1], [x1, y1, z0]]),
            (f"{bid}_w", [[x0, y0, z0], [x0, y0, z1], [x0, y1, z1], [x0, y1, z0]]),
            (f"{bid}_e", [[x1, y0, z0], [x1, y1, z0], [x1, y1, z1], [x1, y0, z1]]),
            (f"{bid}_roof", [[x0, y0, z1], [x1, y0, z1], [x1, y1, z1], [x0, y1, z1]]),
            (f"{bid}_base", [[x0, y0, z0], [x0, y1, z0], [x1, y1, z0], [x1, y0, z0]])]


def entries(r, m, max_order):
    out = []
    for e in r.matrix_entries(m):
        if e["order"] > max_order:
            continue
        ch = list(e["chain"]) + [0] * (3 - len(e["chain"]))
        out.append([e["order"]] + ch + [e["plane"]])   # [order, chain (>= 3 ids), plane]
    return out


def case(r, name, wps, max_order, building_names, faces=None):
    m = r.build_matrix(max_order)
    rows = r.trajectory_vis_table(m, np.asarray(wps, np.float64), max_order)
    for row in rows:
        row["s_start"] = float(row["s_start"]).hex()
        row["s_end"] = float(row["s_end"]).hex()
    d = {"scene": name, "building_names": building_names, "waypoints": wps, "max_order": max_order,
         "entries": entries(r, m, max_order), "rows": rows}
    if faces is not None:
        d["faces"] = faces
    print(name, "order", max_order, len(rows), "rows", len(d["entries"]), "entries")
    return d


def main() -> None:
    bindings.build(ref=True)
    cases = []
    jobs = [("screened_wall", "route_drive_by", 2), ("screened_wall", "route_drive_by", 1),
            ("screened_wall", "route_corridor", 1), ("manhattan", "route_manhattan", 2),
            ("street_canyon", "route_corridor", 2), ("two_buildings", "route_drive_by", 2),
            ("screened_wall", "route_drive_by", 3), ("street_canyon", "route_corridor", 3),
            ("two_buildings", "route_drive_by", 4)]
    for scene, rt_name, order in jobs:
        r = bindings.RefOracle(path=os.path.join(FIXTURES, scene + ".json"))
        soup = soup_from_ref(r, scene)
        cases.append(case(r, scene, route(rt_name), order, soup.building_ids))
    # primed-label walk (proj/tests/test_vistable.cpp:286-319)
    faces = box_faces("K2", (10, 20, 0), (40, 22, 10)) + box_faces("W3", (24, 40, 0), (26, 42, 20))
    off = np.zeros(len(faces) + 1, np.int32)
    off[1:] = np.cumsum([len(p) for _, p in faces])
    soup = scenes.FacetSoup(ids=[i for i, _ in faces], vert_off=off,
                            verts=np.array([q for _, p in faces for q in p], np.float64),
                            building=np.array([0] * 6 + [1] * 6, np.int32), building_ids=["K2", "W3"],
                            name="primed")
    r = bindings.RefOracle(soup)
    fx = [{"id": i, "pts": p, "building": b} for (i, p), b in zip(faces, [0] * 6 + [1] * 6)]
    cases.append(case(r, "primed", [[25, 0, 2], [25, 18, 2]], 1, ["K2", "W3"], faces=fx))
    # config 1: the seeded soup along its Tx line (100 m), orders 1 and 2
    wl = scenes.workload(1)
    r = bindings.RefOracle(wl.scene)
    wps = [wl.tx[0].tolist(), wl.tx[-1].tolist()]
    for order in (1, 2):
        cases.append(case(r, "config1", wps, order, []))
    with open(os.path.join(HERE, "trajectories.json"), "w") as fh:
        json.dump(cases, fh, separators=(",", ":"))


if __name__ == "__main__":
    main()
