"""Quick image-tree timing (development aid)."""
import sys, time
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import Scene, Tracer
for arg in sys.argv[1:] or ["1:2:100"]:
    cfg, order, nsnap = (int(x) for x in arg.split(":"))
    wl = scenes.workload(cfg)
    with Scene(wl.scene) as sc:
        sc.pair_visibility("prefiltered")
        tr = Tracer(sc, order)
        rx = wl.rx if len(wl.rx) == 1 else wl.rx[:nsnap]
        for rep in range(2):
            t0 = time.perf_counter()
            off, paths, nodes, st = tr.trace_raw(wl.tx[:nsnap], rx)
            t1 = time.perf_counter()
        print(f"cfg{cfg} order{order} nsnap={nsnap}: device {st['ms']:.2f} ms wall {1e3*(t1-t0):.1f} ms "
              f"nodes {st['nodes']} ({st['nodes']/max(1,nsnap):.0f}/snap) paths {st['paths']} "
              f"leg tests {st['leg_tests']} -> {st['nodes']/st['ms']*1e3:.3e} nodes/s", flush=True)
