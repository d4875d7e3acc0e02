"""Quick trajectory-table timing at config scale (development aid)."""
import sys, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np
from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import ENTRY_DTYPE, Scene, chain_triples, trajectory_vis_table, unpack_bits
for arg in sys.argv[1:] or ["3:1:200", "3:2:200"]:
    cfg, order, length = (int(x) for x in arg.split(":"))
    wl = scenes.workload(cfg)
    with Scene(wl.scene) as sc:
        bits, _ = sc.pair_visibility("prefiltered")
        adm = unpack_bits(bits, sc.n)
        ai, aj = np.nonzero(adm)
        tri, _ = chain_triples(sc, bits) if order >= 2 else (np.zeros((0, 3), np.int32), None)
        ent = np.zeros(len(ai) + len(tri), ENTRY_DTYPE)
        ent["order"][: len(ai)] = 1
        ent["chain"][: len(ai), 0] = ai
        ent["chain"][: len(ai), 1] = aj
        ent["order"][len(ai):] = 2
        ent["chain"][len(ai):, :3] = tri
        d = wl.tx[-1] - wl.tx[0]
        wps = np.array([wl.tx[0], wl.tx[0] + d / np.linalg.norm(d) * length])
        for rep in range(2):   # second call timed (first-call init excluded)
            t0 = time.perf_counter()
            rows, st = trajectory_vis_table(sc, wps, ent, order, wl.scene.ids, return_stats=True)
            wall = time.perf_counter() - t0
        print(f"cfg{cfg} order{order} route {length} m: samples {st['pairs']} boundaries {st['candidates']} rows {len(rows)} "
              f"device {st['ms']:.1f} ms wall {1e3*wall:.1f} ms launches {st['sweeps']} entries {len(ent)}", flush=True)
