"""K2w phase breakdown (build with VISRT_NVCC_FLAGS=-DVISRT_K2W_PROF; development aid)."""
import ctypes as C, sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import Scene
from paper_2501_02747_b200._capi import lib
for cfg in [int(a) for a in sys.argv[1:]] or [2, 3]:
    with Scene(scenes.workload(cfg).scene) as sc:
        out = (C.c_ulonglong * 16)()
        sc.pair_visibility("all")
        lib().visrt_debug_k2w_prof(out)
        _, st = sc.pair_visibility("all")
        lib().visrt_debug_k2w_prof(out)
    o = list(out)
    T = max(o[0], 1)
    print(f"cfg{cfg}: {st['ms']:.2f} ms; pairs {o[7]} visible {o[10]} ({100*o[8]/T:.1f}% of cycles); "
          f"cache-only pairs {o[9]}; cache settle {100*o[1]/T:.1f}%; sweeps {o[3]} ({100*o[2]/T:.1f}%), "
          f"clear sweeps {o[5]} ({100*o[4]/T:.1f}%); post-sweep settle {100*o[6]/T:.1f}%; "
          f"cycles/pair {T/max(o[7],1):.0f}, /sweep {o[2]/max(o[3],1):.0f}, /clear sweep {o[4]/max(o[5],1):.0f}",
          flush=True)
