"""Small invocations of the table / chain / tree kernels (for ncu captures)."""
import sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import Scene, Tracer, chain_triples, point_regions_array
what = sys.argv[1]
wl = scenes.workload(3)
with Scene(wl.scene) as sc:
    if what == "regions":
        arr, st = point_regions_array(sc, np.concatenate([wl.tx[::100], wl.rx[::100]]))
    elif what == "chains":
        sc.pair_visibility("prefiltered", copy_bits=False)
        tri, st = chain_triples(sc)
    elif what == "tree":
        sc.pair_visibility("prefiltered", copy_bits=False)
        tri, _ = chain_triples(sc)
        tr = Tracer(sc, 3, triples=tri)
        st = tr.trace_raw(wl.tx[:8], wl.rx[:8])[3]
    print(what, st)
