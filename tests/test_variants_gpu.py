"""Every traversal variant of the sweeping kernels gives bit-identical outputs
on FULL matrices / region tables (sha-256 of the whole output):

  * K2w member boxes: fp32 resident (N <= 6,144), streamed with the group
    level, and 8-bit quantised in shared memory (sweep.h qsat; the default
    for 6,144 < N <= 24,576, forced on small scenes with VISRT_QUANT=2);
  * K2w grabs: 16-pair rows vs pair-matrix tiles (VISRT_K2W_TILED) of the resident
    (2 x 16) and the big-scene (16 x 8, 8-entry cache) shapes and an odd one (5 x 3);
  * K4w task walk: face-major (default) vs source-major
    (VISRT_K4W_FACEMAJOR=0), and the same three member-box residencies;
  * K4w refinement: fan candidate lists (default) vs one sweep per sightline
    (VISRT_K4W_FAN=0);
  * K4w cone lists (the face's candidate list once it is partly visible,
    default) vs every sample swept through the hierarchy (VISRT_K4W_CONE=0),
    and a cone capacity small enough to overflow (VISRT_K4W_CONE=48).

Each variant runs in its own process (the knobs are read once per process).
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MATRIX = ("import sys, json, hashlib; sys.path.insert(0, %r);"
          "from paper_2501_02747_b200 import scenes;"
          "from paper_2501_02747_b200.core import Scene;"
          "sc = Scene(scenes.workload(%d).scene); b, st = sc.pair_visibility('all');"
          "a, _ = sc.pair_visibility('prefiltered');"
          "print(json.dumps([hashlib.sha256(b.tobytes()).hexdigest(), hashlib.sha256(a.tobytes()).hexdigest(),"
          " st['tests_exec']]))")

REGIONS = ("import sys, json, hashlib; import numpy as np; sys.path.insert(0, %r);"
           "from paper_2501_02747_b200 import scenes;"
           "from paper_2501_02747_b200.core import Scene, point_regions_array;"
           "wl = scenes.workload(%d); src = np.concatenate([wl.tx[::%d], wl.rx[::%d]]);"
           "sc = Scene(wl.scene); arr, st = point_regions_array(sc, src);"
           "print(json.dumps([hashlib.sha256(arr.tobytes()).hexdigest(), int((arr['present'] == 1).sum())]))")


def run(code, **env):
    e = dict(os.environ)
    e.update({k: str(v) for k, v in env.items()})
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


MATRIX_VARIANTS = [
    {},
    {"VISRT_QUANT": 2},
    {"VISRT_QUANT": 0, "VISRT_FORCE_STREAM": 1},
    {"VISRT_K2W_TILED": 1},
    {"VISRT_K2W_TILED": 1, "VISRT_QUANT": 2},
    {"VISRT_K2W_TILED": 0, "VISRT_QUANT": 0, "VISRT_FORCE_STREAM": 1},
    # the big-scene launch shape (16 x 8 tiles, 8-entry cache, streamed boxes) forced on small scenes
    {"VISRT_K2W_TILED": 1, "VISRT_K2W_TR": 16, "VISRT_K2W_TC": 8, "VISRT_K2W_WCT": 8, "VISRT_QUANT": 0,
     "VISRT_FORCE_STREAM": 1},
    {"VISRT_K2W_TILED": 1, "VISRT_K2W_TR": 5, "VISRT_K2W_TC": 3, "VISRT_K2W_SERP": 1},
    {"VISRT_K2W_TILED": 1, "VISRT_K2W_TR": 48, "VISRT_K2W_TC": 4, "VISRT_K2W_SERP": 1, "VISRT_K2W_TMORTON": 0},
]


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_matrix_variants_agree(cfg):
    code = MATRIX % (ROOT, cfg)
    out = [run(code, **v) for v in MATRIX_VARIANTS]
    for v, o in zip(MATRIX_VARIANTS[1:], out[1:]):
        assert o[:2] == out[0][:2], (v, o, out[0])


@pytest.mark.slow
def test_matrix_config4_quantised_vs_streamed():
    """Config 4 (22,096 facets): the quantised shared-memory sweep and the
    streamed sweep (default) give the same full (A) and (B) matrices."""
    code = MATRIX % (ROOT, 4)
    q = run(code, VISRT_QUANT=1)
    st = run(code)
    assert q[:2] == st[:2]


MATRIX_B = ("import sys, json, hashlib; sys.path.insert(0, %r);"
            "from paper_2501_02747_b200 import scenes;"
            "from paper_2501_02747_b200.core import Scene;"
            "sc = Scene(scenes.workload(%d).scene); b, st = sc.pair_visibility('all');"
            "print(json.dumps([hashlib.sha256(b.tobytes()).hexdigest(), st['tests_exec']]))")


@pytest.mark.slow
@pytest.mark.parametrize("cfg", [3, 4])
def test_matrix_full_size_brute_force_vs_culled(cfg):
    """The whole (B) matrix of configs 3 and 4 (3.8 M / 244 M pairs) built twice: with the
    fp32 culling hierarchy, blocker caches and grouped sweeps (default), and brute force
    (VISRT_NOCULL=1: every culling test passes, every occluder reached runs the exact FP64
    predicate — config 4: ~270x the exact tests, ~15 s). Culling is only allowed to
    skip work, never to change a verdict: the bit matrices are identical."""
    code = MATRIX_B % (ROOT, cfg)
    culled = run(code)
    brute = run(code, VISRT_NOCULL=1)
    assert brute[0] == culled[0]
    assert brute[1] > 20 * culled[1]   # the brute-force build really ran unculled


ROWS = ("import sys, json, hashlib; import numpy as np; sys.path.insert(0, %r);"
        "from paper_2501_02747_b200 import scenes;"
        "from paper_2501_02747_b200.core import Scene;"
        "from paper_2501_02747_b200.dist import pair_row_blocks;"
        "sc = Scene(scenes.workload(%d).scene); full, st = sc.pair_visibility('all');"
        "acc = np.zeros_like(full); pairs = 0; tests = 0.0; overlap = 0\n"
        "for r0, r1 in pair_row_blocks(sc.n, %d):\n"
        "    if r1 <= r0: continue\n"
        "    b, s = sc.pair_visibility('all', rows=(r0, r1)); overlap += int(np.bitwise_count(acc & b).sum());"
        " acc |= b; pairs += s['pairs']; tests += s['tests_alg']\n"
        "print(json.dumps([bool((acc == full).all()), overlap, pairs == st['pairs'],"
        " abs(tests - st['tests_alg']) <= 1e-9 * st['tests_alg']]))")


@pytest.mark.parametrize("cfg,world,env", [(1, 3, {}), (2, 4, {}), (2, 5, {"VISRT_K2W_TILED": 1}),
                                           (2, 3, {"VISRT_K2W_TILED": 1, "VISRT_K2W_TR": 16, "VISRT_K2W_TC": 8}),
                                           (3, 2, {}), (3, 7, {"VISRT_K2W_TILED": 0})])
def test_matrix_row_blocks_or_to_the_full_matrix(cfg, world, env):
    """visrt_pair_visibility_rows: the row blocks of a partition (the strong-scaling
    shard of one scene) carry disjoint bits and OR into the full (B) matrix, for the
    row-grab and the tiled K2w walk; their pair and reference-test counts add up."""
    assert run(ROWS % (ROOT, cfg, world), **env) == [True, 0, True, True]


REGION_VARIANTS = [
    {},
    {"VISRT_K4W_FAN": 0},
    {"VISRT_QUANT": 2},
    {"VISRT_QUANT": 0, "VISRT_FORCE_STREAM": 1},
    {"VISRT_K4W_FACEMAJOR": 0},
    {"VISRT_K4W_FACEMAJOR": 0, "VISRT_QUANT": 2},
    {"VISRT_K4W_CONE": 0},
    {"VISRT_K4W_CONE": 48},
]


@pytest.mark.parametrize("cfg,step", [(1, 7), (3, 50)])
def test_region_variants_agree(cfg, step):
    code = REGIONS % (ROOT, cfg, step, step)
    out = [run(code, **v) for v in REGION_VARIANTS]
    for v, o in zip(REGION_VARIANTS[1:], out[1:]):
        assert o == out[0], (v, o, out[0])


@pytest.mark.slow
def test_region_config5_quantised_vs_streamed():
    code = REGIONS % (ROOT, 5, 2500, 2500)
    assert run(code, VISRT_QUANT=1) == run(code)
