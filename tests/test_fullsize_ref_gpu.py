"""Full-size parity against the compiled reference's committed outputs
(tests/golden/full/*.npz, made by tests/golden/make_golden_full.py from
oracle/_ref = the unmodified reference): the GPU runs the BASELINE
workloads of configs 3-5 and every boolean / index / interval output is
compared bit for bit.

  * config 3 (B): all 3,796,390 pairs            (src/vismatrix.cpp:253-302)
  * config 3 (A): build_matrix(scene,1) admitted (src/vismatrix.cpp:638-675)
  * config 4 (A): build_matrix(scene,1) admitted, all 2.44e8 pairs
  * config 4 (B): 100,000 seeded pairs of the full GPU matrix
  * config 3 regions: 100 sources x all faces    (src/vistable.cpp:287-334)
  * config 5 regions: 100 sources x all 22,096 faces (digest per source)
  * config 3 point_vis_table, 50 sources         (src/vistable.cpp:478-521)
  * config 3 trajectory_vis_table, 100 m          (src/vistable.cpp:845-987)
  * config 3 / 5 order-3 traces, 100 snapshots each (src/raytracer.cpp:496-514)
  * config 3 order-2 chains: all 15,021,972 triples     (src/vismatrix.cpp:715-797)
"""
import glob
import hashlib
import os

import numpy as np
import pytest

import golden_util as G
from paper_2501_02747_b200 import scenes
from paper_2501_02747_b200.core import (ENTRY_DTYPE, Scene, Tracer, chain_triples, point_regions_array,
                                        point_tables, trajectory_vis_table, unpack_bits)

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

FULL = os.path.join(G.GOLDEN, "full")


def fixture(name):
    p = os.path.join(FULL, name + ".npz")
    if not os.path.exists(p):
        pytest.skip(f"fixture {name}.npz not generated (tests/golden/make_golden_full.py)")
    return np.load(p)


def scene_sha(soup) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(soup.vert_off, np.int32).tobytes())
    h.update(np.ascontiguousarray(soup.verts, np.float64).tobytes())
    return h.hexdigest()


_WL = {}


def workload(cfg, d):
    if cfg not in _WL:
        _WL[cfg] = scenes.workload(cfg)
    wl = _WL[cfg]
    assert scene_sha(wl.scene) == str(d["scene_sha"]), "scene generator drifted from the fixture"
    return wl


def admitted_from_entries(E, n):
    adm = np.zeros((n, n), bool)
    adm[E[:, 0], E[:, 1]] = True
    return adm


def entries_dtype(E):
    out = np.zeros(len(E), ENTRY_DTYPE)
    out["order"] = 1
    out["chain"][:, 0] = E[:, 0]
    out["chain"][:, 1] = E[:, 1]
    out["plane"] = E[:, 2]
    return out


def test_config3_matrix_B_all_pairs():
    d = fixture("c3B")
    wl = workload(3, d)
    n = wl.scene.nfaces
    with Scene(wl.scene) as sc:
        bits, _ = sc.pair_visibility("all")
    M = unpack_bits(bits, n)
    pi, pj = G.pairs(n)
    exp = np.unpackbits(d["bits"])[: len(pi)].astype(bool)
    got = M[pi, pj]
    bad = np.nonzero(got != exp)[0]
    assert len(bad) == 0, f"{len(bad)} of {len(pi)} pairs differ, first {[(int(pi[k]), int(pj[k])) for k in bad[:5]]}"
    np.testing.assert_array_equal(M, M.T)


@pytest.mark.parametrize("cfg", [3, 4])
def test_matrix_A_all_pairs(cfg):
    d = fixture(f"c{cfg}A")
    wl = workload(cfg, d)
    n = wl.scene.nfaces
    with Scene(wl.scene) as sc:
        bits, _ = sc.pair_visibility("prefiltered")
    got = unpack_bits(bits, n)
    exp = admitted_from_entries(d["entries"], n)
    assert int(got.sum()) == int(exp.sum())
    np.testing.assert_array_equal(got, exp)


def test_config4_matrix_B_seeded_pairs():
    d = fixture("c4B")
    wl = workload(4, d)
    n = wl.scene.nfaces
    with Scene(wl.scene) as sc:
        bits, _ = sc.pair_visibility("all")
    M = unpack_bits(bits, n)
    pi, pj = d["pi"], d["pj"]
    np.testing.assert_array_equal(M[pi, pj], d["kinds"] != 2)
    np.testing.assert_array_equal(M[pi, pj], M[pj, pi])


def test_config3_chains_all():
    """Every order-2 chain of build_matrix(scene, 2) on config 3 (src/vismatrix.cpp:715-797):
    15.0 M (p, t, a) triples, compared by count, sha-256 of the sorted int32 array and a
    1/997 sample."""
    d = fixture("c3chains")
    wl = workload(3, d)
    with Scene(wl.scene) as sc:
        bits, _ = sc.pair_visibility("prefiltered")
        tri, _ = chain_triples(sc, bits)
    tri = np.ascontiguousarray(tri, np.int32)
    assert len(tri) == int(d["count"])
    np.testing.assert_array_equal(tri[d["sample_idx"]], d["sample"])
    assert hashlib.sha256(tri.tobytes()).hexdigest() == str(d["sha"])


def _regions_check(cfg, d, sc):
    src = d["src"]
    arr, _ = point_regions_array(sc, src)
    P = arr["present"]
    np.testing.assert_array_equal(P, d["present"])
    for q in range(len(src)):
        dig = G.region_digest(arr["present"][q], arr["has"][q], arr["clipped"][q], arr["sub"][q])
        assert dig == str(d["digest"][q]), f"config {cfg} source {q} ({src[q]}): regions differ"
    if "has" in d.files:
        pres = d["present"] == 1
        np.testing.assert_array_equal(arr["has"][pres], d["has"][pres])
        np.testing.assert_array_equal(arr["sub"][pres].view(np.uint64), d["sub"].view(np.uint64))


def test_config3_regions_all_faces():
    d = fixture("c3regions")
    wl = workload(3, d)
    with Scene(wl.scene) as sc:
        _regions_check(3, d, sc)


def test_config5_regions_all_faces():
    files = sorted(glob.glob(os.path.join(FULL, "c5regions_*.npz")))
    if not files:
        pytest.skip("config-5 region fixtures not generated")
    d0 = np.load(files[0])
    wl = workload(5, d0)
    nsrc = 0
    with Scene(wl.scene) as sc:
        for f in files:
            d = np.load(f)
            _regions_check(5, d, sc)
            nsrc += len(d["src"])
    assert nsrc >= 4


def test_config3_point_vis_table():
    d = fixture("c3tables")
    wl = workload(3, d)
    E = entries_dtype(fixture("c3A")["entries"])
    src = d["src"]
    with Scene(wl.scene) as sc:
        rows, full, regs, _ = point_tables(sc, src, E, want_regions=True)
    off = d["off"]
    for q in range(len(src)):
        ee = np.cumsum(d["entry_delta"][off[q]:off[q + 1]])   # ascending entry indices of the rows
        got_e = np.nonzero(rows[q])[0]
        np.testing.assert_array_equal(got_e, ee)
        o = np.arange(len(ee))
        np.testing.assert_array_equal(full[q, ee], d["full"][off[q]:off[q + 1]][o])
        # display primes: clipped region of the named face in the entry's plane
        pl = E["plane"][ee]
        for col, key in ((0, "ref_primed"), (1, "aim_primed")):
            f = E["chain"][ee, col]
            r = regs[q, f]
            primed = (r["present"] == 1) & (r["has"][np.arange(len(f)), pl] == 1) & \
                     (r["clipped"][np.arange(len(f)), pl] == 1)
            np.testing.assert_array_equal(primed, d[key][off[q]:off[q + 1]][o])


def test_config3_trajectory_table():
    d = fixture("c3traj")
    wl = workload(3, d)
    E = entries_dtype(fixture("c3A")["entries"])
    with Scene(wl.scene) as sc:
        rows = trajectory_vis_table(sc, d["waypoints"], E, 1, wl.scene.ids)
    keys = ["order", "node", "node_display", "s_start", "s_end", "label_start", "label_end", "parent", "blockage"]
    got = "\n".join("\t".join(str(x[k]) if k not in ("s_start", "s_end") else float(x[k]).hex() for k in keys)
                    for x in rows)
    exp = bytes(d["rows"]).decode()
    assert got.split("\n") == exp.split("\n")


@pytest.mark.parametrize("cfg", [3, 5])
def test_trace_order3(cfg):
    d = fixture(f"c{cfg}trace")
    wl = workload(cfg, d)
    ks = d["snap"]
    with Scene(wl.scene) as sc:
        bits, _ = sc.pair_visibility("prefiltered")
        tri, _ = chain_triples(sc, bits)
        tr = Tracer(sc, 3, admitted_bits=bits, triples=tri)
        paths, nodes, _ = tr.trace(wl.tx[ks], wl.rx[ks])
        tr.close()
    np.testing.assert_array_equal(np.asarray(nodes, np.int64), d["nodes"])
    off = d["off"]
    for q in range(len(ks)):
        exp = []
        for p in range(off[q], off[q + 1]):
            nf = int((d["faces"][p] >= 0).sum())
            exp.append((tuple(int(x) for x in d["faces"][p][:nf]),
                        tuple(float(x) for x in d["points"][p][: 3 * (nf + 2)]), float(d["length"][p])))
        got = [(tuple(p["faces"]), tuple(p["points"]), p["length"]) for p in paths[q]]
        assert sorted(got) == sorted(exp), f"snapshot {ks[q]}"
