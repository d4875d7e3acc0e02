"""Quick matrix timing on one GPU (development aid)."""
import hashlib, sys, time
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import Scene

for cfg in [int(a) for a in sys.argv[1:]] or [1, 2]:
    soup = scenes.workload(cfg).scene
    with Scene(soup) as sc:
        for mode in ("all", "prefiltered"):
            for rep in range(3):
                t0 = time.perf_counter()
                bits, st = sc.pair_visibility(mode, copy_bits=rep == 2)
                t1 = time.perf_counter()
            sha = hashlib.sha256(np.asarray(bits).tobytes()).hexdigest()[:16]
            print(f"cfg{cfg} N={soup.nfaces} {mode}: kernel {st['ms']:.3f} ms wall {1e3*(t1-t0):.2f} ms "
                  f"cand {st['candidates']} tests_alg {st['tests_alg']:.3e} exec {st['tests_exec']:.3e} "
                  f"alg/s {st['tests_alg']/st['ms']*1e3:.3e} sweeps {st['sweeps']:.3e} tiles {st['tiles']:.3e} sha {sha}", flush=True)
