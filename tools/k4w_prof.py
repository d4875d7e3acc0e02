"""K4w phase breakdown (build with VISRT_NVCC_FLAGS=-DVISRT_K4W_PROF; development aid):
cycles in the column scan vs the boundary bisection, sweeps (clear / blocked) per phase."""
import ctypes as C, sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import Scene, point_regions_array
from paper_2501_02747_b200._capi import lib
for arg in sys.argv[1:] or ["5:20:rx", "5:20:tx", "3:200:mix"]:
    f = arg.split(":")
    cfg, nsrc, which = int(f[0]), int(f[1]), f[2]
    wl = scenes.workload(cfg)
    src = {"tx": wl.tx, "rx": wl.rx, "mix": np.concatenate([wl.tx[:nsrc // 2], wl.rx[:nsrc - nsrc // 2]])}[which][:nsrc]
    with Scene(wl.scene) as sc:
        out = (C.c_ulonglong * 24)()
        lib().visrt_debug_k4w_prof(out)   # reset
        arr, st = point_regions_array(sc, src)
        lib().visrt_debug_k4w_prof(out)
    o = list(out)
    tot = max(o[8], 1)
    print(f"cfg{cfg}/{which} nsrc={nsrc}: {st['ms']:.1f} ms; task cycles {o[8]:.3e}: scan {100*o[0]/tot:.1f}% "
          f"refine {100*o[1]/tot:.1f}% present-tasks {100*o[10]/tot:.1f}% ({o[11]} of {o[9]} front-facing); "
          f"scan sweeps {o[2]} clear {o[3]}; refine calls {o[6]} iters {o[7]} sweeps {o[4]} clear {o[5]}; "
          f"cycles/sweep scan {o[0]/max(o[2],1):.0f} refine {o[1]/max(o[4],1):.0f}; "
          f"cone lists {o[12]} overflow {o[13]} mean length {o[14]/max(o[12]-o[13],1):.0f} scan iterations {o[15]:.3e}; "
          f"refine fan build {100*o[16]/tot:.1f}% fans {o[18]} mean T {o[17]/max(o[18],1):.1f}; "
          f"scan split: cone build {100*o[19]/tot:.1f}% cone scan {100*o[20]/tot:.1f}% sweeps {100*o[21]/tot:.1f}%; "
          f"refine steps: sample {100*o[22]/tot:.1f}% whole steps {100*o[23]/tot:.1f}%", flush=True)
