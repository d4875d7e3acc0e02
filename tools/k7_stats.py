"""K7 stage counts (build with VISRT_NVCC_FLAGS=-DVISRT_K7_STATS; development aid)."""
import ctypes as C, sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import Scene, chain_triples
from paper_2501_02747_b200._capi import lib
for cfg in [int(a) for a in sys.argv[1:]] or [3]:
    with Scene(scenes.workload(cfg).scene) as sc:
        sc.pair_visibility("prefiltered", copy_bits=False)
        out = (C.c_ulonglong * 8)()
        lib().visrt_debug_k7_stats(out)
        tri, st = chain_triples(sc)
        lib().visrt_debug_k7_stats(out)
    o = list(out)
    print(f"cfg{cfg}: candidates {st['candidates']} feasible-calls {o[0]} past pre-reject {o[1]} clip-c ok {o[2]} "
          f"mean section {o[3]/max(o[2],1):.1f} hull ok {o[4]} mean hull {o[7]/max(o[4],1):.1f} overlap {o[5]} "
          f"finite {o[6]} triples {len(tri)} ms {st['ms']:.1f}", flush=True)
