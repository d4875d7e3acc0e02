"""(1) Inter-visibility matrix: GPU (through the C-ABI) vs the CPU oracle.

Bit-exact: (B) bits = occlusion_judgment(F_i, F_j).kind != Occluded for every
i<j; (A) candidates = first_order_pair's gate, admitted = pair_admitted of
build_matrix(scene, 1); detail = verdict kind + blocker set.
"""
import numpy as np
import pytest

from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import Scene, unpack_bits

pytestmark = pytest.mark.gpu


def _all_pairs(n):
    pi, pj = np.triu_indices(n, 1)
    return pi.astype(np.int32), pj.astype(np.int32)


@pytest.fixture(scope="module")
def cfg1():
    return scenes.workload(1)


def test_matrix_all_pairs_config1(oracle_built, cfg1):
    soup = cfg1.scene
    o = oracle_built.Oracle(soup)
    pi, pj = _all_pairs(soup.nfaces)
    kinds = o.occlusion_batch(pi, pj)
    with Scene(soup) as sc:
        bits, st = sc.pair_visibility("all")
    M = unpack_bits(bits, soup.nfaces)
    assert np.array_equal(M, M.T)
    assert not M.diagonal().any()
    np.testing.assert_array_equal(M[pi, pj], kinds != 2)
    assert st["pairs"] == len(pi)
    assert st["tests_exec"] > 0


def test_matrix_prefiltered_config1(oracle_built, cfg1):
    soup = cfg1.scene
    o = oracle_built.Oracle(soup)
    pi, pj = _all_pairs(soup.nfaces)
    pref = np.array([o.prefilter(i, j) for i, j in zip(pi, pj)])
    with Scene(soup) as sc:
        bits, st = sc.pair_visibility("prefiltered")
        ci, cj, ad = sc.candidates()
    # ordered (i, j) candidate list identical to the oracle gate
    np.testing.assert_array_equal(ci, pi[pref])
    np.testing.assert_array_equal(cj, pj[pref])
    kinds = o.occlusion_batch(ci, cj)
    np.testing.assert_array_equal(ad.astype(bool), kinds != 2)   # no degenerate ranges here
    M = unpack_bits(bits, soup.nfaces)
    expect = np.zeros_like(M)
    expect[ci[ad == 1], cj[ad == 1]] = True
    expect = expect | expect.T
    np.testing.assert_array_equal(M, expect)


def test_matrix_prefiltered_matches_reference_build_matrix(oracle_built, cfg1):
    if not oracle_built.have_ref():
        pytest.skip("oracle/_ref not built")
    soup = cfg1.scene
    r = oracle_built.RefOracle(soup)
    entries = r.matrix_entries(r.build_matrix(1))
    admitted = {(e["chain"][0], e["chain"][1]) for e in entries}
    with Scene(soup) as sc:
        bits, _ = sc.pair_visibility("prefiltered")
    M = unpack_bits(bits, soup.nfaces)
    got = {(int(i), int(j)) for i, j in zip(*np.nonzero(M))}
    assert got == admitted


def test_pair_detail_config1(oracle_built, cfg1):
    soup = cfg1.scene
    o = oracle_built.Oracle(soup)
    pi, pj = _all_pairs(soup.nfaces)
    sel = np.arange(0, len(pi), 3)
    with Scene(soup) as sc:
        kind, blockers, st = sc.pair_detail(pi[sel], pj[sel])
    for k, s in enumerate(sel):
        ek, eb = o.occlusion(int(pi[s]), int(pj[s]))
        assert kind[k] == ek, (pi[s], pj[s])
        assert blockers[k] == sorted(eb), (pi[s], pj[s])


@pytest.mark.parametrize("cfg", [2])
def test_matrix_all_pairs_sampled_rows(oracle_built, cfg):
    """Full-size (B) matrix of config 2 on the GPU; a seeded sample of pairs
    re-decided by the oracle (the full CPU pass takes minutes)."""
    soup = scenes.workload(cfg).scene
    n = soup.nfaces
    with Scene(soup) as sc:
        bits, st = sc.pair_visibility("all")
    M = unpack_bits(bits, n)
    assert np.array_equal(M, M.T)
    rng = np.random.default_rng(7)
    pi = rng.integers(0, n, 3000).astype(np.int32)
    pj = rng.integers(0, n, 3000).astype(np.int32)
    keep = pi != pj
    pi, pj = np.minimum(pi, pj)[keep], np.maximum(pi, pj)[keep]
    kinds = oracle_built.Oracle(soup).occlusion_batch(pi, pj)
    np.testing.assert_array_equal(M[pi, pj], kinds != 2)


def test_matrix_stream_path_config1(oracle_built, cfg1, monkeypatch):
    """The streamed-tile sweep (used when the culling boxes exceed shared
    memory, e.g. config 4) must give the same bits as the resident sweep."""
    import subprocess, sys, os, json
    code = ("import sys, json; sys.path.insert(0, %r);"
            "from paper_2501_02747_b200 import scenes;"
            "from paper_2501_02747_b200.core import Scene;"
            "sc = Scene(scenes.workload(1).scene); b, st = sc.pair_visibility('all');"
            "k, bl, _ = sc.pair_detail([0, 3, 5], [40, 77, 100]);"
            "print(json.dumps([b.tolist(), k.tolist(), bl]))") % os.path.dirname(os.path.dirname(__file__))
    out = {}
    for force in ("0", "1"):
        env = dict(os.environ, VISRT_FORCE_STREAM=force)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True)
        out[force] = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["0"] == out["1"]


@pytest.mark.parametrize("cfg", [1, 2])
def test_matrix_lane_and_warp_kernels_agree(cfg):
    """K2w (warp per pair, default) and K2 (lane per pair, VISRT_K2_WARP=0)
    give identical (A) and (B) bits; both resident and global box paths."""
    import subprocess, sys, os, json
    code = ("import sys, json, hashlib; sys.path.insert(0, %r);"
            "from paper_2501_02747_b200 import scenes;"
            "from paper_2501_02747_b200.core import Scene;"
            "sc = Scene(scenes.workload(%d).scene); b, _ = sc.pair_visibility('all');"
            "a, _ = sc.pair_visibility('prefiltered');"
            "print(json.dumps([hashlib.sha256(b.tobytes()).hexdigest(), hashlib.sha256(a.tobytes()).hexdigest()]))"
            ) % (os.path.dirname(os.path.dirname(__file__)), cfg)
    out = {}
    # lane kernel; warp kernel resident; streamed with the group level; streamed flat
    for warp, force, grouped in (("0", "0", "1"), ("1", "0", "1"), ("1", "1", "1"), ("1", "1", "0")):
        env = dict(os.environ, VISRT_K2_WARP=warp, VISRT_FORCE_STREAM=force, VISRT_K2W_GROUPED=grouped)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True)
        out[warp + force + grouped] = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["001"] == out["101"] == out["111"] == out["110"]
