"""The C++ drop-in layer (paper_2501_02747_b200/cpp/rt.hpp, namespace rt on
the GPU C-ABI) against the unmodified reference (visrt_ref::) in one C++
program: build_matrix entries (every field: chains, PAR/PER, verdicts,
angle records incl. edge ids, criterion, subranges, blockers, aim images),
occlusion_judgment, illuminated_region (all fields incl. atan2 angles),
point_vis_table rows, image_tree, closest_diffraction_edge, trajectory_vis_table and
TraceAccelerator path sets/stats — bit-exact."""
import os
import subprocess

import pytest

import golden_util as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2501_02747_b200")
REF = os.path.join(ROOT, "oracle", "_ref")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def parity_bin(tmp_path_factory):
    from paper_2501_02747_b200 import build
    build.build()
    if not os.path.exists(os.path.join(REF, "libvisrt_ref.so")):
        pytest.skip("oracle/_ref not built")
    exe = str(tmp_path_factory.mktemp("cpp") / "parity_rt")
    subprocess.run(["g++", "-std=c++17", "-O2", "-o", exe, os.path.join(ROOT, "tests", "cpp", "parity_rt.cpp"),
                    "-L", PKG, "-lrt_b200", "-lvisrt_cuda", "-L", REF, "-lvisrt_ref",
                    f"-Wl,-rpath,{PKG}:{REF}"], check=True)
    return exe


def write_scene(path, d, sources, traces, max_order):
    faces = d["faces"]
    bids = []
    for f in faces:
        if f["building"] >= 0 and f["building"] >= len(bids):
            bids.extend(["B?"] * (f["building"] + 1 - len(bids)))
    # building ids: the prefix of the face ids of that building (reference fixtures: "<bid>_<suffix>")
    for f in faces:
        if f["building"] >= 0:
            bids[f["building"]] = f["id"].rsplit("_", 1)[0]
    with open(path, "w") as fh:
        fh.write(f"{len(faces)} {len(bids)}\n")
        for b in bids:
            fh.write(b + "\n")
        for f in faces:
            fh.write(f"{f['id']} {f['building']} {len(f['pts'])} " +
                     " ".join(float(c).hex() for p in f["pts"] for c in p) + "\n")
        fh.write(f"{len(sources)}\n")
        for s in sources:
            fh.write(" ".join(float(c).hex() for c in s) + "\n")
        fh.write(f"{len(traces)}\n")
        for tx, rx in traces:
            fh.write(" ".join(float(c).hex() for c in list(tx) + list(rx)) + "\n")
        fh.write(f"{max_order}\n")


@pytest.mark.parametrize("name", ["two_buildings", "street_canyon", "screened_wall", "manhattan", "config1"])
def test_cpp_dropin_parity(parity_bin, tmp_path, name):
    d = G.load(name)
    if name == "config1":
        for f in d["faces"]:
            f["building"] = -1 if f["id"].startswith("T_") else f["building"]
        d = dict(d)
        d["faces"] = [dict(f, building=-1) for f in d["faces"]]   # facet soup: no shells
    sources = [G.unhex(r["source"]) for r in d["regions"]]
    traces = sorted({(tuple(G.unhex(t["tx"])), tuple(G.unhex(t["rx"]))) for t in d["traces"]})
    scene = tmp_path / "scene.txt"
    write_scene(scene, d, sources, traces, max_order=2)
    r = subprocess.run([parity_bin, str(scene)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK 0 mismatches" in r.stdout
