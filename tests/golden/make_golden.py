"""Generate tests/golden/*.json from the UNMODIFIED reference (oracle/_ref,
compiled from /root/reference by oracle/Makefile). Run in the build container:

    python tests/golden/make_golden.py

Each fixture records the scene (faces converted from the reference's own
fixture files proj/data/fixtures/*.json via its load_scene, or the seeded
config-1 soup) and the reference's outputs on the hot path:
  * kinds  : occlusion_judgment(F_i, F_j).kind for every i < j ("0/1/2" string)
  * blockers: occlusion_judgment blocker sets (face indices) for Partial pairs
  * matrix1: build_matrix(scene, 1) entries (ref, aim, plane, PAR/PER, angles, blockers)
  * triples: the order-2 chains (p, t, a) of build_matrix(scene, 2)
  * regions: illuminated_region(source, face) for sampled sources x all faces
  * traces : TraceAccelerator(max_refl).trace(tx, rx, false) path sets + node counts
Doubles are stored with float.hex() so the comparison is bit-exact.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import bindings  # noqa: E402
from paper_2501_02747_b200 import scenes  # noqa: E402

FIXTURES = "/root/reference/proj/data/fixtures"


def hx(v: float) -> str:
    return float(v).hex()


def soup_from_ref(r: bindings.RefOracle, name: str) -> scenes.FacetSoup:
    faces, _ = r.export()
    bids = []
    building = []
    for f in faces:
        b = f["building"]
        if b == "":
            building.append(-1)
        else:
            if b not in bids:
                bids.append(b)
            building.append(bids.index(b))
    off = np.zeros(len(faces) + 1, np.int32)
    off[1:] = np.cumsum([len(f["pts"]) for f in faces])
    verts = np.array([p for f in faces for p in f["pts"]], np.float64)
    return scenes.FacetSoup(ids=[f["id"] for f in faces], vert_off=off, verts=verts,
                            building=np.array(building, np.int32), building_ids=bids, name=name)


def record(r: bindings.RefOracle, soup: scenes.FacetSoup, sources, traces, orders=(1, 2, 3),
           blockers=True, extra=None) -> dict:
    n = soup.nfaces
    faces, edges = r.export()
    out = {"name": soup.name, "faces": [{"id": f["id"], "pts": f["pts"], "building": b,
                                         "label_xy": f["label_xy"], "label_vert": f["label_vert"]}
                                        for f, b in zip(faces, soup.building.tolist()
                                                        if soup.building is not None else [-1] * n)],
           "edges": edges}
    pi, pj = np.triu_indices(n, 1)
    kinds = r.occlusion_batch(pi.astype(np.int32), pj.astype(np.int32))
    out["kinds"] = "".join(str(int(k)) for k in kinds)
    if blockers:
        out["blockers"] = {f"{i},{j}": r.occlusion(int(i), int(j))[1]
                           for i, j, k in zip(pi, pj, kinds) if k == 1}
    m1 = r.build_matrix(1)
    out["matrix1"] = [{"ref": e["chain"][0], "aim": e["chain"][1], "plane": e["plane"],
                       "kind": "PAR" if e["kind"] == 0 else "PER",
                       "ranges": [hx(e["ranges"][q]) for q in (2, 3, 8, 9)],
                       "blockers": e["blockers"], "edge_a": e["edge_a"], "edge_b": e["edge_b"]}
                      for e in r.matrix_entries(m1)]
    m2 = r.build_matrix(2)
    ents2 = r.matrix_entries(m2)
    out["matrix2_entries"] = len(ents2)
    out["triples"] = sorted({tuple(e["chain"]) for e in ents2 if e["order"] == 2})
    regs = []
    for src in sources:
        row = []
        for f in range(n):
            d = r.illuminated_region(np.asarray(src, np.float64), f)
            row.append([d["present"], d["has"], d["clipped"], [hx(x) for x in d["sub"]]])
        regs.append({"source": [hx(x) for x in src], "regions": row})
    out["regions"] = regs
    trs = []
    r.lib().vref_matrix_set_max_order(m2, 3)
    for order in orders:
        acc = r.accel(m2, order)
        for tx, rx in traces:
            paths, st = r.trace(acc, np.asarray(tx, np.float64), np.asarray(rx, np.float64))
            trs.append({"order": order, "tx": [hx(x) for x in tx], "rx": [hx(x) for x in rx],
                        "nodes": int(st[0]), "sequences": int(st[1]),
                        "paths": sorted([{"identity": p["identity"], "faces": p["faces"],
                                          "points": [hx(x) for x in p["points"]], "length": hx(p["length"])}
                                         for p in paths], key=lambda p: p["identity"])})
        r.lib().vref_accel_free(acc)
    out["traces"] = trs
    if extra:
        out.update(extra)
    return out


def main() -> None:
    bindings.build(ref=True)
    os.makedirs(HERE, exist_ok=True)
    jobs = {
        "two_buildings": ([(5, 15, 2), (5, -5, 2), (20, 25, 40)], [((3, 15, 2), (7, 16, 3)), ((5, -5, 2), (5, 15, 2))]),
        "street_canyon": ([(5, 28, 11), (5, 15, 2), (-4, 12, 6)], [((3, 15, 2), (7, 16, 3)), ((5, 15, 1.5), (5, 35, 1.5))]),
        "screened_wall": ([(2, 2, 2), (25, -5, 1.5)], [((2, -3, 1.5), (20, 8, 1.5))]),
        "open_field": ([(0, 0, 2), (30, 5, 10)], [((0, 0, 10), (50, 0, 2))]),
        "manhattan": ([(12.5, 2.5, 1.5), (50, 50, 30)], [((2.5, 12.5, 1.5), (97.5, 62.5, 1.5)),
                                                       ((30, 2.5, 2), (50, 97.5, 2))]),
    }
    for name, (sources, traces) in jobs.items():
        r = bindings.RefOracle(path=os.path.join(FIXTURES, name + ".json"))
        soup = soup_from_ref(r, name)
        data = record(r, soup, sources, traces)
        with open(os.path.join(HERE, name + ".json"), "w") as fh:
            json.dump(data, fh, separators=(",", ":"))
        print(name, soup.nfaces, "faces", len(data["matrix1"]), "entries", len(data["triples"]), "triples")
    # config 1 (seeded soup through the facet-soup adapter)
    wl = scenes.workload(1)
    r = bindings.RefOracle(wl.scene)
    soup = wl.scene
    soup.name = "config1"
    data = record(r, soup, [wl.tx[0], wl.tx[57], wl.rx[0]],
                  [(wl.tx[k], wl.rx[0]) for k in (0, 31, 64, 99)], orders=(2, 3), blockers=False,
                  extra={"sha_verts": hx(float(np.sum(soup.verts * np.arange(soup.verts.size).reshape(soup.verts.shape))))})
    with open(os.path.join(HERE, "config1.json"), "w") as fh:
        json.dump(data, fh, separators=(",", ":"))
    print("config1", soup.nfaces, "faces", len(data["matrix1"]), "entries", len(data["triples"]), "triples")


if __name__ == "__main__":
    main()
