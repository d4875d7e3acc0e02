"""CPU-only checks: the C-ABI library loads and exports every symbol
include/visrt.h declares, the host-side ingest (run through the library with a
host-only handle, device = -1) matches the oracle and the reference, the
seeded generators are deterministic, and the product fails loudly (no CPU
fallback) when the CUDA path is asked for work without a device."""
import ctypes
import os
import re

import numpy as np
import pytest

import golden_util as G
from paper_2501_02747_b200 import _capi, scenes
from paper_2501_02747_b200.core import Scene

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "visrt.h")).read()
    return sorted(set(re.findall(r"\b(visrt_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_2501_02747_b200 import build
    build.build()
    lib = ctypes.CDLL(_capi.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_capi.EXPORTS)


def test_sm100a_only_and_no_fma_in_predicate():
    """cuobjdump: the fatbin carries sm_100a SASS only; the FP64 predicate
    uses no DFMA (bit-exact FP64)."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump absent")
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in l for l in out.splitlines() if ".cubin" in l)
    full = subprocess.run(["cuobjdump", "-sass", _capi.LIB_PATH], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", full)
    hot = [f for f in funcs if re.match(r"\S*(k_pair_bits|k_pair_detail|k_point_regions|k_tree_unfold|"
                                        r"k_tree_legs|k_chain_triples)", f)]
    assert len(hot) >= 6
    for f in hot:
        assert "DMUL" in f or "DADD" in f
    assert any("UBLKCP" in f for f in hot)        # TMA bulk copies of the culling boxes
    # FP64 arithmetic is never contracted: the PTX holds separate mul/add/sub
    # .rn.f64 and no fma.*.f64 (SASS DFMA appears only inside the correctly
    # rounded div.rn.f64 / sqrt.rn.f64 expansions).
    from paper_2501_02747_b200 import build
    for src in ("matrix.cu", "tree.cu", "chains.cu", "regions.cu", "trajectory.cu"):
        ptx = subprocess.run([build.NVCC, "-std=c++17", "-ptx", "--fmad=false", "-gencode",
                              "arch=compute_100a,code=sm_100a", "-I", os.path.join(ROOT, "include"),
                              os.path.join(build.CSRC, src), "-o", "-"], capture_output=True, text=True, check=True).stdout
        assert "mul.rn.f64" in ptx and "add.rn.f64" in ptx
        assert not re.search(r"\bfma\.rn\.f64", ptx), src


@pytest.mark.parametrize("name", ["two_buildings", "street_canyon", "manhattan", "config1"])
def test_host_ingest_matches_oracle(oracle_built, name):
    d = G.load(name)
    s = G.soup(d)
    o = oracle_built.Oracle(s)
    with Scene(s, device=-1) as sc:
        nrm, ori, seg, ok = sc.ingest()
    np.testing.assert_array_equal(ori, o.orientation())
    for i in range(s.nfaces):
        for pl in range(3):
            e = o.plane_segment(i, pl)
            assert bool(ok[i, pl]) == (e is not None)
            if e is not None:
                assert seg[i, pl].tolist() == e.tolist()


def test_host_only_handle_refuses_device_work():
    s = scenes.workload(1).scene
    with Scene(s, device=-1) as sc:
        with pytest.raises(_capi.UsageError):
            sc.pair_visibility("all")


def test_scene_rejects_bad_faces():
    s = scenes.workload(1).scene
    bad = scenes.FacetSoup(ids=["x"], vert_off=np.array([0, 2], np.int32), verts=s.verts[:2].copy())
    with pytest.raises(_capi.SceneError, match="fewer than 3 vertices"):
        Scene(bad, device=-1)


def test_generators_deterministic_and_sized():
    a = scenes.workload(1)
    b = scenes.workload(1)
    assert np.array_equal(a.scene.verts, b.scene.verts) and np.array_equal(a.tx, b.tx)
    assert a.scene.nfaces == 116 and len(a.tx) == 100
    assert scenes.workload(2).scene.nfaces == 1256
    w3 = scenes.workload(3)
    assert w3.scene.nfaces == 2756 and len(w3.tx) == 1000 and len(w3.rx) == 1000
    d = G.load("config1")
    assert G.soup(d).verts.tolist() == a.scene.verts.tolist()   # golden pinned to this generator


def test_generated_normals_point_outward(oracle_built):
    """CCW-from-outside rings: every wall/roof normal points away from its
    box centre, tiles face +z (Scene::finalize's outward rule, scene.cpp:118-123)."""
    s = scenes.workload(1).scene
    o = oracle_built.Oracle(s)
    nrm = np.zeros(3)
    ori = ctypes.c_int32()
    for i, fid in enumerate(s.ids):
        o.lib().vo_face_info(o.h, i, nrm, ctypes.byref(ori))
        pts = s.face_points(i)
        if fid.startswith("T_"):
            assert nrm[2] == 1.0
            continue
        b = fid.split("_")[0]
        idx = [k for k, x in enumerate(s.ids) if x.split("_")[0] == b]
        centre = np.concatenate([s.face_points(k) for k in idx]).mean(axis=0)
        assert np.dot(nrm, pts.mean(axis=0) - centre) > 0


def test_matrix_cache_roundtrip_cpu(tmp_path):
    """Binary matrix / pair-graph cache, host-only:
    the reference's admitted pairs + order-2 chains of config 1 round-trip
    exactly; another scene is refused (SceneError); a corrupt file is a
    VisibilityError."""
    from paper_2501_02747_b200.core import load_matrix_cache, save_matrix_cache
    d = G.load("config1")
    s = G.soup(d)
    n = s.nfaces
    words = (n + 63) // 64
    bits = np.zeros((n, words), np.uint64)
    for e in d["matrix1"]:
        i, j = e["ref"], e["aim"]
        bits[i, j // 64] |= np.uint64(1) << np.uint64(j % 64)
    tri = np.array(d["triples"], np.int32)
    path = str(tmp_path / "m.bin")
    with Scene(s, device=-1) as sc:
        save_matrix_cache(sc, path, bits, tri, max_order=2)
        b2, t2, mo = load_matrix_cache(sc, path)
    assert mo == 2 and np.array_equal(b2, bits) and np.array_equal(t2, tri)
    other = G.soup(G.load("street_canyon"))
    with Scene(other, device=-1) as sc2:
        with pytest.raises(_capi.SceneError, match="different scene"):
            load_matrix_cache(sc2, path)
    raw = bytearray(open(path, "rb").read())
    raw[100] ^= 0xFF
    open(path, "wb").write(bytes(raw))
    with Scene(s, device=-1) as sc:
        with pytest.raises(_capi.VisibilityError, match="corrupt"):
            load_matrix_cache(sc, path)
