"""Row block of a config's (B) matrix, culled or brute force (VISRT_NOCULL=1): time + sha (development aid).
usage: python tools/quick_rows.py cfg row0 row1"""
import hashlib, sys, time
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import Scene
cfg, r0, r1 = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
with Scene(scenes.workload(cfg).scene) as sc:
    t0 = time.perf_counter()
    b, st = sc.pair_visibility("all", rows=(r0, r1))
    print(f"cfg{cfg} rows [{r0},{r1}): pairs {st['pairs']} kernel {st['ms']:.1f} ms wall {1e3*(time.perf_counter()-t0):.0f} ms "
          f"exec {st['tests_exec']:.3e} sha {hashlib.sha256(b.tobytes()).hexdigest()[:16]}", flush=True)
