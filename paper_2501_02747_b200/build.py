"""Build recipe for the in-tree sm_100a library ``libvisrt_cuda.so``.

nvcc cross-compiles without a GPU; the .so is git-ignored but travels to the
GPU box with the gpurun snapshot. Flags:
  * ``-gencode arch=compute_100a,code=sm_100a`` — B200 only, no PTX fallback;
  * ``--fmad=false`` + explicit ``__d*_rn`` intrinsics — no FMA contraction in
    the FP64 predicate (bit-exact against the reference's x86-64 build);
  * host code with ``-ffp-contract=off`` for the same reason (ingest, angles).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libvisrt_cuda.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

SOURCES = ["ingest.cpp", "matrix.cu", "regions.cu", "trajectory.cu", "imagetree.cu", "chains.cu", "tree.cu", "peaks.cu", "capi.cu", "cache.cu", "em.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def sources():
    return [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".h")]
    deps.append(os.path.join(INCLUDE, "visrt.h"))
    deps += [os.path.join(HERE, "cpp", f) for f in ("rt.cpp", "rt.hpp")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    objdir = os.path.join(HERE, "_obj")
    os.makedirs(objdir, exist_ok=True)
    common = [NVCC, "-std=c++17", "-O3", "-lineinfo", "--fmad=false",
              "-gencode", "arch=compute_100a,code=sm_100a",
              "-Xcompiler", "-fPIC,-ffp-contract=off", "-I", INCLUDE, "-I", CSRC]
    common += os.environ.get("VISRT_NVCC_FLAGS", "").split()   # tuning experiments (-DVISRT_K2_MINB=2 ...)
    if verbose:
        common += ["-Xptxas", "-v"]
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        procs.append((src, subprocess.Popen(common + ["-c", src, "-o", obj],
                                            stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose and out:
            sys.stderr.write(out.decode())
    subprocess.run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB] + objs +
                   ["-lcudart"], check=True)
    build_rt()
    return LIB


RT_LIB = os.path.join(HERE, "librt_b200.so")


def json_include() -> str:
    """nlohmann json.hpp for rt::load_scene / save_scene: the copy vendored in the
    image's site-packages (cudnn_frontend); VISRT_JSON_INCLUDE overrides."""
    if os.environ.get("VISRT_JSON_INCLUDE"):
        return os.environ["VISRT_JSON_INCLUDE"]
    import sysconfig
    return os.path.join(sysconfig.get_paths()["purelib"], "include", "cudnn_frontend", "thirdparty", "nlohmann")


def build_rt() -> str:
    """The C++ drop-in layer (namespace rt over the C-ABI), host code only."""
    src = os.path.join(HERE, "cpp", "rt.cpp")
    subprocess.run(["g++", "-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-shared", "-o", RT_LIB, src,
                    "-I", os.path.join(HERE, "cpp"), "-I", json_include(), "-L", HERE, "-lvisrt_cuda",
                    "-Wl,-rpath,$ORIGIN"], check=True)
    return RT_LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
