"""Generate tests/golden/em.json from the UNMODIFIED reference (oracle/_ref):
ray_gains + channel_stats (proj/src/em.cpp:194-277) of accelerated traces on
the reference's fixture scenes (with their materials and edge faces), for TE /
TM polarisation and antenna gains. Run in the build container:
    python tests/golden/make_golden_em.py"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from oracle import bindings  # noqa: E402
from make_golden import FIXTURES  # noqa: E402


def main() -> None:
    bindings.build(ref=True)
    out = []
    jobs = {"two_buildings": [((3, 15, 2), (7, 16, 3)), ((-5, 5, 2), (35, 5, 2))],
            "street_canyon": [((3, 15, 2), (7, 16, 3)), ((5, 15, 1.5), (5, 35, 1.5))],
            "screened_wall": [((2, -3, 1.5), (20, 8, 1.5)), ((0, 10, 2), (50, 10, 2)), ((25, -5, 1.5), (5, 12, 1))],
            "manhattan": [((2.5, 12.5, 1.5), (30, 12.5, 1.5))]}
    cfgs = [(5.5e9, 0.0, 0.0, 0), (2.4e9, 3.0, 1.5, 1)]
    for name, trs in jobs.items():
        r = bindings.RefOracle(path=os.path.join(FIXTURES, name + ".json"))
        mats = r.face_materials()
        efaces = r.edge_faces()
        m = r.build_matrix(2)
        acc = r.accel(m, 2)
        cases = []
        for tx, rx in trs:
            for dif in (False, True):
                paths, _ = r.trace(acc, np.asarray(tx, np.float64), np.asarray(rx, np.float64), diffraction=dif)
                for freq, gt, gr, tm in cfgs:
                    amp, dl, st = r.trace_em(acc, tx, rx, dif, freq, gt, gr, tm)
                    cases.append({"tx": list(tx), "rx": list(rx), "diffraction": dif, "freq": freq, "tx_gain": gt,
                                  "rx_gain": gr, "tm": tm,
                                  "paths": [{"identity": p["identity"], "re": float(a[0]).hex(), "im": float(a[1]).hex(),
                                             "delay": float(d).hex()} for p, a, d in zip(paths, amp, dl)],
                                  "stats": [float(x).hex() for x in st]})
        r.lib().vref_accel_free(acc)
        out.append({"scene": name, "materials": mats.tolist(), "edge_faces": efaces, "cases": cases})
        print(name, len(cases), "cases", sum(len(c["paths"]) for c in cases), "rays")
    with open(os.path.join(HERE, "em.json"), "w") as fh:
        json.dump(out, fh, separators=(",", ":"))


if __name__ == "__main__":
    main()
