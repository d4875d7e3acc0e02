"""Break down the e2e step (development aid): ingest+upload, build, D2H, free."""
import sys, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np
from paper_2501_02747_b200 import scenes, _capi
from paper_2501_02747_b200.core import Scene
soup = scenes.workload(2).scene
for rep in range(5):
    t0 = time.perf_counter()
    s = Scene(soup)
    t1 = time.perf_counter()
    bits, st = s.pair_visibility("all")
    t2 = time.perf_counter()
    s.close()
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} ms  build+D2H {1e3*(t2-t1):.2f} ms (kernel {st['ms']:.2f})  destroy {1e3*(t3-t2):.2f} ms")
