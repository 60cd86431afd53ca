"""Build libslm_b200.so in-tree (sm_100a kernels + C++ runtime + C ABI).

    python -m paper_2504_12905_b200.build [--force]

nvcc cross-compiles for sm_100a without a GPU.  preprocess.cu is compiled
with -fmad=false so the FP64 preparation rounds like the reference's
-ffp-contract=off build (proj/src/CMakeLists.txt:23-25); everything else uses
-O3 with FMA.  The runtime is plain C++ compiled by g++ so its <random>
distributions are libstdc++'s, exactly like the reference's.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libslm_b200.so")
INCLUDE = os.path.join(ROOT, "include")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_SOURCES = {
    "preprocess.cu": ["-fmad=false"],
    "raster.cu": [],
    "chain.cu": [],
    "cg.cu": [],
    "sort.cu": [],
    "metrics.cu": [],
    "sampler.cu": [],
    "first_order.cu": [],
}
CPP_SOURCES = ["runtime.cpp"]
HEADERS = ["common.cuh", "layout.hpp", "runtime.hpp"]


def _newer(src_paths, out):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(p) > t for p in src_paths)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {os.path.basename(cmd[-1])}")
    return r.stdout + r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    deps = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "slm_types.h"),
                                                       os.path.join(INCLUDE, "slm_b200.h")]
    objs = []
    for src, extra in CU_SOURCES.items():
        sp = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if force or _newer([sp, *deps, __file__], obj):
            out = _run([NVCC, "-std=c++17", "-O3", "-lineinfo", *ARCH, *extra, "-Xcompiler", "-fPIC",
                        "-Xptxas", "-v", f"-I{INCLUDE}", f"-I{CSRC}", "-c", sp, "-o", obj])
            if verbose:
                print(out)
    for src in CPP_SOURCES:
        sp = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if force or _newer([sp, *deps, __file__], obj):
            _run(["g++", "-std=c++17", "-O2", "-fPIC", "-Wall", f"-I{INCLUDE}", f"-I{CSRC}",
                  f"-I{CUDA}/include", "-c", sp, "-o", obj])
    if force or _newer(objs, LIB):
        _run([NVCC, "-shared", *ARCH, "-cudart", "static", "-o", LIB, *objs, "-ldl"])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
