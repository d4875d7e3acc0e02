"""Culling stress test: near-grazing scenes (tests/adversarial.py) decided on
the GPU under every member-box residency (fp32 shared memory, streamed
through L1/L2, 8-bit quantised in shared memory) and with culling switched
off, against the UNMODIFIED reference (oracle/_ref):

  * (B) occlusion bits of every pair inside a group and of seeded
    cross-group pairs (occlusion_judgment, src/vismatrix.cpp:253-302);
  * (A) admitted bits of the whole matrix (build_matrix(scene, 1));
  * sightline_clear of the stressed segments (src/vistable.cpp:38-44);
  * illuminated_region of every group face from sources on and behind the
    grazing line (src/vistable.cpp:287-334).

Any one-sidedness failure of the fp32 box dilation (ingest.cpp box_margin,
quantise_members) would show up as a GPU 'visible' / 'clear' where the
reference finds a blocker."""
import os
import subprocess
import sys

import numpy as np
import pytest

import adversarial as ADV
import golden_util as G

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MODES = {"default": {}, "quantised": {"VISRT_QUANT": "2"},
         "streamed": {"VISRT_QUANT": "0", "VISRT_FORCE_STREAM": "1"}, "nocull": {"VISRT_NOCULL": "1"}}

RUNNER = r'''
import sys, numpy as np
sys.path.insert(0, %(root)r); sys.path.insert(0, %(tests)r)
import adversarial as ADV
from paper_2501_02747_b200.core import Scene, point_regions_array, segments_clear
soup, meta = ADV.build()
A, B = ADV.stressed_segments(meta)
src = ADV.sources(meta)
with Scene(soup) as sc:
    bb, _ = sc.pair_visibility("all")
    ba, _ = sc.pair_visibility("prefiltered")
    clear, _ = segments_clear(sc, A, B)
    reg, _ = point_regions_array(sc, src)
np.savez(%(out)r, bb=bb, ba=ba, clear=clear, reg=reg)
'''


@pytest.fixture(scope="module")
def scene():
    return ADV.build()


@pytest.fixture(scope="module")
def reference(scene, oracle_built):
    if not oracle_built.have_ref():
        pytest.skip("oracle/_ref not built")
    soup, meta = scene
    r = oracle_built.RefOracle(soup)
    n = soup.nfaces
    pi, pj = [], []
    for m in meta:
        f = m["faces"]
        for a in range(len(f)):
            for b in range(a + 1, len(f)):
                pi.append(f[a])
                pj.append(f[b])
    rng = np.random.default_rng(2501027470 + 90)
    i = rng.integers(0, n, 6000)
    j = rng.integers(0, n, 6000)
    keep = i != j
    pi = np.concatenate([pi, np.minimum(i, j)[keep]]).astype(np.int32)
    pj = np.concatenate([pj, np.maximum(i, j)[keep]]).astype(np.int32)
    kinds = r.occlusion_batch(pi, pj)
    adm = np.zeros((n, n), bool)
    for e in r.matrix_entries(r.build_matrix(1)):
        if e["order"] == 1:
            adm[e["chain"][0], e["chain"][1]] = True
    A, B = ADV.stressed_segments(meta)
    blocked = r.segments_blocked(A, B)
    src = ADV.sources(meta)
    qs, qf = [], []
    for g, m in enumerate(meta):
        for k in (2 * g, 2 * g + 1):
            for f in m["faces"]:
                qs.append(k)
                qf.append(f)
    regs = r.regions_batch(src[qs], np.array(qf, np.int32))
    return {"pi": pi, "pj": pj, "kinds": kinds, "adm": adm, "blocked": blocked, "qs": qs, "qf": qf, "regs": regs}


def run_mode(tmp_path, mode):
    out = str(tmp_path / f"{mode}.npz")
    code = RUNNER % {"root": ROOT, "tests": os.path.join(ROOT, "tests"), "out": out}
    env = dict(os.environ, **MODES[mode])
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("mode", list(MODES))
def test_adversarial_vs_reference(scene, reference, tmp_path, mode):
    soup, meta = scene
    n = soup.nfaces
    got = run_mode(tmp_path, mode)
    from paper_2501_02747_b200.core import unpack_bits
    MB = unpack_bits(got["bb"], n)
    ref = reference
    exp_b = ref["kinds"] != 2
    bad = np.nonzero(MB[ref["pi"], ref["pj"]] != exp_b)[0]
    assert len(bad) == 0, f"{mode}: (B) differs on {[(int(ref['pi'][k]), int(ref['pj'][k])) for k in bad[:5]]}"
    np.testing.assert_array_equal(unpack_bits(got["ba"], n), ref["adm"], err_msg=f"{mode}: (A) differs")
    np.testing.assert_array_equal(got["clear"], ~ref["blocked"], err_msg=f"{mode}: sightline_clear differs")
    reg = got["reg"]
    for q, (k, f) in enumerate(zip(ref["qs"], ref["qf"])):
        g = reg[k, f]
        e = ref["regs"][q]
        assert (int(g["present"]), [int(x) for x in g["has"]], [int(x) for x in g["clipped"]],
                [float(x) for x in g["sub"]]) == (e["present"], e["has"], e["clipped"], e["sub"]), (mode, k, f)


def test_adversarial_scene_is_sensitive(scene, reference):
    """The stress is real: the grazing offsets flip the reference's decisions
    (both visible and occluded window pairs, both clear and blocked segments)."""
    soup, meta = scene
    ref = reference
    kinds = dict(zip(zip(ref["pi"].tolist(), ref["pj"].tolist()), ref["kinds"].tolist()))
    pq = [kinds[(m["faces"][0], m["faces"][1])] for m in meta]
    assert 2 in pq and any(k != 2 for k in pq)
    assert ref["blocked"].any() and (~ref["blocked"]).any()
