"""Run one config's matrix build a few times (for ncu captures)."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import Scene
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mode = sys.argv[2] if len(sys.argv) > 2 else "all"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
with Scene(scenes.workload(cfg).scene) as sc:
    for _ in range(reps):
        _, st = sc.pair_visibility(mode, copy_bits=False)
    print(st)
