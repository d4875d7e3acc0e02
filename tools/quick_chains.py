"""Quick order-2 chain timing (development aid)."""
import hashlib, sys, time
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import Scene, chain_triples
for cfg in [int(a) for a in sys.argv[1:]] or [1, 2, 3]:
    wl = scenes.workload(cfg)
    with Scene(wl.scene) as sc:
        _, st0 = sc.pair_visibility("prefiltered", copy_bits=False)
        t0 = time.perf_counter()
        tri, st = chain_triples(sc)
        t1 = time.perf_counter()
        print(f"cfg{cfg} N={wl.scene.nfaces}: admitted pairs {st['pairs']} candidate triples {st['candidates']} "
              f"feasible {st['admitted']} kernel {st['ms']:.1f} ms wall {1e3*(t1-t0):.0f} ms "
              f"sha {hashlib.sha256(np.ascontiguousarray(tri).tobytes()).hexdigest()[:16]}", flush=True)
