"""Reject-reason histogram of the exact predicate in K2w (build with -DVISRT_SEG_STATS; development aid)."""
import ctypes as C, sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import Scene
from paper_2501_02747_b200._capi import lib
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
with Scene(scenes.workload(cfg).scene) as sc:
    sc.pair_visibility("all")
    out = (C.c_ulonglong * 8)()
    lib().visrt_debug_seg_stats(out)
names = ["total", "eps", "same_side", "off_plane", "edge0", "edge_k", "hit"]
tot = out[0]
print(f"cfg{cfg}: " + ", ".join(f"{n} {out[i]} ({100*out[i]/max(tot,1):.1f}%)" for i, n in enumerate(names)))
