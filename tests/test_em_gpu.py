"""EM consumer: ray_gains + channel_stats
(proj/src/em.cpp:194-235) on the GPU vs the compiled reference's values
(tests/golden/em.json, made by tests/golden/make_golden_em.py) for the same
traces (path sets bit-identical, pinned elsewhere). Transcendentals are CUDA's,
so amplitudes and path loss are compared with a relative tolerance of 1e-9
(the RMS delay spread with 1e-7 of the delays, for the m2 - m1^2 cancellation);
delays (length / c) are exact."""
import json
import os

import numpy as np
import pytest

import golden_util as G
from paper_2501_02747_b200.core import Scene, Tracer, channel_stats, chain_triples, path_identity, ray_gains

pytestmark = pytest.mark.gpu
EM = json.load(open(os.path.join(G.GOLDEN, "em.json")))
RTOL = 1e-9


@pytest.mark.parametrize("k", range(len(EM)), ids=[e["scene"] for e in EM])
def test_ray_gains_and_channel_stats_vs_reference(k):
    e = EM[k]
    d = G.load(e["scene"])
    s = G.soup(d)
    edges = d["edges"]
    with Scene(s) as sc:
        bits, _ = sc.pair_visibility("prefiltered")
        tri, _ = chain_triples(sc, bits)
        tr = Tracer(sc, 2, admitted_bits=bits, triples=tri, edges=edges)
        for c in e["cases"]:
            paths, _, _ = tr.trace([c["tx"]], [c["rx"]], allow_diffraction=c["diffraction"])

            def ident(p):
                return path_identity(s.ids, p["faces"], edges[p["edge"]]["id"] if p["edge"] >= 0 else None)

            ps = sorted(paths[0], key=ident)   # the reference's ray order (paths sorted by identity)
            assert [ident(p) for p in ps] == [r["identity"] for r in c["paths"]]
            amp, dl = ray_gains(sc, ps, e["materials"], edges, e["edge_faces"], c["freq"], c["tx_gain"],
                                c["rx_gain"], "TM" if c["tm"] else "TE")
            for a, t, r in zip(amp, dl, c["paths"]):
                ref = complex(float.fromhex(r["re"]), float.fromhex(r["im"]))
                assert abs(a - ref) <= RTOL * abs(ref), (r["identity"], a, ref)
                assert t == float.fromhex(r["delay"])
            out, loss, rms = channel_stats(sc, [amp], [dl])
            es = [float.fromhex(x) for x in c["stats"]]
            assert bool(out[0]) == bool(es[0])
            if not out[0]:
                assert abs(loss[0] - es[1]) <= RTOL * abs(es[1])
                # m2 - m1^2 cancels: sqrt(eps) x delay of absolute slack (1e-7 relative to the delays)
                assert abs(rms[0] - es[2]) <= RTOL * abs(es[2]) + 1e-7 * float(np.max(dl))
