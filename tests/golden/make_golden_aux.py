"""Generate tests/golden/aux.json from the UNMODIFIED reference (oracle/_ref):
image_tree(scene, source, depth) (proj/src/raytracer.cpp:458-486) node lists
and closest_diffraction_edge(receiver, scene) (proj/src/vistable.cpp:545-561)
answers on the reference's fixture scenes and the seeded config-1 soup.
Run in the build container:  python tests/golden/make_golden_aux.py"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from oracle import bindings  # noqa: E402
from paper_2501_02747_b200 import scenes  # noqa: E402
from make_golden import FIXTURES  # noqa: E402


def main() -> None:
    bindings.build(ref=True)
    trees, edges = [], []
    jobs = [("two_buildings", (5, -5, 2), 2), ("two_buildings", (5, 15, 2), 3), ("street_canyon", (5, 28, 11), 3),
            ("screened_wall", (2, 2, 2), 3), ("manhattan", (12.5, 2.5, 1.5), 2), ("open_field", (0, 0, 2), 3)]
    for name, src, depth in jobs:
        r = bindings.RefOracle(path=os.path.join(FIXTURES, name + ".json"))
        face, parent, dep, image = r.image_tree(np.asarray(src, np.float64), depth)
        trees.append({"scene": name, "source": list(src), "depth": depth, "face": face.tolist(),
                      "parent": parent.tolist(), "node_depth": dep.tolist(),
                      "image": [[float(x).hex() for x in p] for p in image]})
        print(name, depth, len(face), "nodes")
    wl = scenes.workload(1)
    r = bindings.RefOracle(wl.scene)
    face, parent, dep, image = r.image_tree(wl.tx[3], 2)
    trees.append({"scene": "config1", "source": wl.tx[3].tolist(), "depth": 2, "face": face.tolist(),
                  "parent": parent.tolist(), "node_depth": dep.tolist(),
                  "image": [[float(x).hex() for x in p] for p in image]})
    print("config1", 2, len(face), "nodes")
    rng = np.random.default_rng(7)
    for name in ("two_buildings", "street_canyon", "screened_wall", "manhattan", "open_field"):
        r = bindings.RefOracle(path=os.path.join(FIXTURES, name + ".json"))
        _, es = r.export()
        pts = [(5, 12, 1), (5, 5, 2), (5, -5, 2), (5, 28, 11), (12.5, 2.5, 1.5), (50, 50, 30)]
        lo = np.min([e["a"] for e in es], axis=0) if es else np.zeros(3)
        hi = np.max([e["a"] for e in es], axis=0) if es else np.ones(3)
        pts += [tuple((lo + (hi - lo) * rng.random(3) * 1.2 - 0.1 * (hi - lo)).tolist()) for _ in range(24)]
        edges.append({"scene": name, "receivers": [list(p) for p in pts],
                      "edge": [r.closest_edge(np.asarray(p, np.float64)) for p in pts]})
        print(name, len(es), "edges")
    # TraceAccelerator::trace with allow_diffraction = true (proj/src/raytracer.cpp:342-444)
    diff = []
    djobs = {"two_buildings": [((3, 15, 2), (7, 16, 3)), ((5, -5, 2), (5, 15, 2)), ((-5, 5, 2), (35, 5, 2))],
             "street_canyon": [((3, 15, 2), (7, 16, 3)), ((5, 15, 1.5), (5, 35, 1.5)), ((5, 5, 1.5), (5, 40, 8))],
             "screened_wall": [((2, -3, 1.5), (20, 8, 1.5)), ((0, 10, 2), (50, 10, 2)), ((25, -5, 1.5), (5, 12, 1))],
             "manhattan": [((2.5, 12.5, 1.5), (97.5, 62.5, 1.5)), ((30, 2.5, 2), (50, 97.5, 2))]}
    for name, trs in djobs.items():
        r = bindings.RefOracle(path=os.path.join(FIXTURES, name + ".json"))
        m = r.build_matrix(2)
        r.lib().vref_matrix_set_max_order(m, 3)
        for order in (1, 2, 3):
            acc = r.accel(m, order)
            for tx, rx in trs:
                try:
                    paths, st = r.trace(acc, np.asarray(tx, np.float64), np.asarray(rx, np.float64), diffraction=True)
                except RuntimeError as e:   # PlacementError: the GPU path must raise it too
                    diff.append({"scene": name, "order": order, "tx": list(tx), "rx": list(rx), "error": str(e)})
                    continue
                diff.append({"scene": name, "order": order, "tx": list(tx), "rx": list(rx), "nodes": int(st[0]),
                             "sequences": int(st[1]),
                             "paths": sorted([{"identity": p["identity"], "points": [float(x).hex() for x in p["points"]],
                                               "length": float(p["length"]).hex()} for p in paths],
                                             key=lambda p: p["identity"])})
            r.lib().vref_accel_free(acc)
        print(name, "diffraction traces", sum(len(d.get("paths", [])) for d in diff if d["scene"] == name), "paths")
    # brute_force_trace (proj/src/raytracer.cpp:488-493)
    brute = []
    for name in ("two_buildings", "street_canyon", "screened_wall"):
        r = bindings.RefOracle(path=os.path.join(FIXTURES, name + ".json"))
        for order in (1, 2, 3):
            for tx, rx in djobs[name]:
                for dif in (False, True):
                    try:
                        paths, st = r.brute_trace(np.asarray(tx, np.float64), np.asarray(rx, np.float64), order, dif)
                    except RuntimeError as e:
                        continue
                    brute.append({"scene": name, "order": order, "tx": list(tx), "rx": list(rx), "diffraction": dif,
                                  "nodes": int(st[0]), "sequences": int(st[1]),
                                  "paths": sorted([{"identity": p["identity"],
                                                    "points": [float(x).hex() for x in p["points"]],
                                                    "length": float(p["length"]).hex()} for p in paths],
                                                  key=lambda p: p["identity"])})
    print("brute traces", len(brute))
    # TraceAccelerator(max_refl = 4): the order-3 chains of build_matrix(scene, 3)
    # restrict depth-4 continuations (proj/src/raytracer.cpp:319-340)
    order4 = []
    o4jobs = [("two_buildings", djobs["two_buildings"][:2]), ("street_canyon", djobs["street_canyon"][:2]),
              ("screened_wall", djobs["screened_wall"][:2])]
    for name, trs in o4jobs:
        r = bindings.RefOracle(path=os.path.join(FIXTURES, name + ".json"))
        m = r.build_matrix(3)
        r.lib().vref_matrix_set_max_order(m, 4)
        acc = r.accel(m, 4)
        for tx, rx in trs:
            for dif in (False, True):
                try:
                    paths, st = r.trace(acc, np.asarray(tx, np.float64), np.asarray(rx, np.float64), diffraction=dif)
                except RuntimeError:
                    continue
                order4.append({"scene": name, "tx": list(tx), "rx": list(rx), "diffraction": dif, "nodes": int(st[0]),
                               "sequences": int(st[1]),
                               "paths": sorted([{"identity": p["identity"], "points": [float(x).hex() for x in p["points"]],
                                                 "length": float(p["length"]).hex()} for p in paths],
                                               key=lambda p: p["identity"])})
        r.lib().vref_accel_free(acc)
    wl = scenes.workload(1)
    r = bindings.RefOracle(wl.scene)
    m = r.build_matrix(3)
    r.lib().vref_matrix_set_max_order(m, 4)
    acc = r.accel(m, 4)
    for k in (0, 50):
        paths, st = r.trace(acc, wl.tx[k], wl.rx[0])
        order4.append({"scene": "config1", "tx": wl.tx[k].tolist(), "rx": wl.rx[0].tolist(), "diffraction": False,
                       "nodes": int(st[0]), "sequences": int(st[1]),
                       "paths": sorted([{"identity": p["identity"], "points": [float(x).hex() for x in p["points"]],
                                         "length": float(p["length"]).hex()} for p in paths],
                                       key=lambda p: p["identity"])})
    r.lib().vref_accel_free(acc)
    print("order-4 traces", len(order4), [t["nodes"] for t in order4])
    # dynamic_trace against a fixed receiver (proj/src/raytracer.cpp:590-643): the
    # non-retraced samples are resolve_keys of their segment's first trace
    dyn = []
    djobs2 = [("screened_wall", "route_drive_by", (25, -5, 1.5)), ("street_canyon", "route_corridor", (5, 35, 1.5)),
              ("two_buildings", "route_drive_by", (35, 5, 2))]
    for name, route_name, rx in djobs2:
        r = bindings.RefOracle(path=os.path.join(FIXTURES, name + ".json"))
        m = r.build_matrix(2)
        with open(os.path.join(FIXTURES, route_name + ".json")) as fh:
            wps = [w[:3] for w in json.load(fh)["waypoints"]]
        for dif in (False, True):
            try:
                smp = r.dynamic_trace(m, np.asarray(wps, np.float64), np.asarray(rx, np.float64), 2, dif, 0.5)
            except RuntimeError as e:
                print(name, "dynamic", e)
                continue
            dyn.append({"scene": name, "waypoints": wps, "rx": list(rx), "diffraction": dif,
                        "samples": [{"s": float(q["s"]).hex(), "segment": q["segment"], "retraced": q["retraced"],
                                     "paths": [{"identity": p["identity"], "points": [float(x).hex() for x in p["points"]],
                                                "length": float(p["length"]).hex()} for p in q["paths"]]}
                                    for q in smp]})
            print(name, "dynamic", dif, len(smp), "samples")
    with open(os.path.join(HERE, "aux.json"), "w") as fh:
        json.dump({"image_trees": trees, "closest_edges": edges, "diffraction_traces": diff, "brute_traces": brute,
                   "dynamic": dyn, "order4_traces": order4},
                  fh, separators=(",", ":"))


if __name__ == "__main__":
    main()
