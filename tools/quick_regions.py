"""Quick per-snapshot region timing (development aid)."""
import hashlib, sys, time
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import Scene, point_regions_array
for arg in sys.argv[1:] or ["1:101", "3:200"]:
    f = arg.split(":")
    cfg, nsrc = int(f[0]), int(f[1])
    which = f[2] if len(f) > 2 else "txrx"   # txrx | tx | rx | mix (half Tx, half Rx)
    wl = scenes.workload(cfg)
    if which == "mix":
        src = np.concatenate([wl.tx[:nsrc // 2], wl.rx[:nsrc - nsrc // 2]])
    else:
        src = {"txrx": np.concatenate([wl.tx, wl.rx]), "tx": wl.tx, "rx": wl.rx}[which][:nsrc]
    with Scene(wl.scene) as sc:
        for rep in range(2):
            t0 = time.perf_counter()
            arr, st = point_regions_array(sc, src)
            t1 = time.perf_counter()
        pres = (arr["present"] == 1).sum()
        print(f"cfg{cfg}/{which} N={wl.scene.nfaces} nsrc={len(src)}: kernel {st['ms']:.2f} ms wall {1e3*(t1-t0):.1f} ms "
              f"regions {arr.size} present {pres} sightlines {st['candidates']:.3e} exact {st['tests_exec']:.3e} "
              f"-> {arr.size/st['ms']*1e3:.3e} regions/s sha {hashlib.sha256(arr.tobytes()).hexdigest()[:16]}", flush=True)
