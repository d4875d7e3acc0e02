"""rt::load_scene / rt::save_scene of the C++ drop-in layer vs the unmodified
reference (include/rt/scene.hpp:108-109, src/scene.cpp:258-375) on the
reference's own scene fixtures: identical faces, edges, saved JSON text and
SceneError messages. Host-only (no GPU): runs where /root/reference exists."""
import glob
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2501_02747_b200")
REF = os.path.join(ROOT, "oracle", "_ref")
FIXTURES = "/root/reference/proj/data/fixtures"
SCENES = [p for p in sorted(glob.glob(os.path.join(FIXTURES, "*.json"))) if "route_" not in p]


@pytest.fixture(scope="module")
def scene_io_bin(tmp_path_factory, oracle_built):
    from paper_2501_02747_b200 import build
    build.build()
    if not oracle_built.have_ref():
        pytest.skip("oracle/_ref not built")
    exe = str(tmp_path_factory.mktemp("cpp") / "scene_io")
    subprocess.run(["g++", "-std=c++17", "-O2", "-o", exe, os.path.join(ROOT, "tests", "cpp", "scene_io.cpp"),
                    "-L", PKG, "-lrt_b200", "-lvisrt_cuda", "-L", REF, "-lvisrt_ref",
                    f"-Wl,-rpath,{PKG}:{REF}"], check=True)
    return exe


@pytest.mark.skipif(not SCENES, reason="reference fixtures not present (GPU box)")
@pytest.mark.parametrize("path", SCENES, ids=[os.path.basename(p) for p in SCENES])
def test_scene_io_matches_reference(scene_io_bin, tmp_path, path):
    r = subprocess.run([scene_io_bin, path, str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK 0 mismatches" in r.stdout
