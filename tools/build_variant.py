"""Build an experimental libslm_b200 variant: one .cu (raster.cu, or $SRC)
recompiled with extra flags (e.g. -DSLM_E1), linked with the normal objects,
written to exp/NAME.so.

    [SRC=sort.cu] [SRCPATH=/tmp/old_raster.cu] python tools/build_variant.py NAME [-DFLAG ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_12905_b200 import build as B  # noqa: E402


def main():
    name, flags = sys.argv[1], sys.argv[2:]
    B.build()
    os.makedirs(os.path.join(ROOT, "exp"), exist_ok=True)
    src = os.environ.get("SRC", "raster.cu")
    obj = os.path.join(ROOT, "exp", f"{name}_{src}.o")
    B._run([B.NVCC, "-std=c++17", "-O3", "-lineinfo", *B.ARCH, "-Xcompiler", "-fPIC", "-Xptxas", "-v",
            f"-I{B.INCLUDE}", f"-I{B.CSRC}", *B.CU_SOURCES[src], *flags, "-c",
            os.environ.get("SRCPATH") or os.path.join(B.CSRC, src),
            "-o", obj])
    objs = [obj if s == src else os.path.join(B.BUILD, s + ".o") for s in B.CU_SOURCES]
    objs += [os.path.join(B.BUILD, s + ".o") for s in B.CPP_SOURCES]
    out = os.path.join(ROOT, "exp", f"{name}.so")
    B._run([B.NVCC, "-shared", *B.ARCH, "-cudart", "static", "-o", out, *objs, "-ldl"])
    print(out)


if __name__ == "__main__":
    main()
