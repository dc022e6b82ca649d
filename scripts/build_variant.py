"""Build a probe variant of libsfv.so: one source file recompiled with extra defines,
linked with the regular objects, written to scripts/probes/variants/libsfv_<name>.so
(git-ignored; load it with SFV_LIB=... for timing experiments only).

    python scripts/build_variant.py <name> <file.cu> -DMACRO=value ...
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_17217_b200 import build as B  # noqa: E402


def main():
    name, fname, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
    B.build()
    out_dir = os.path.join(ROOT, "build", "var", name)
    os.makedirs(out_dir, exist_ok=True)
    obj = os.path.join(out_dir, fname + ".o")
    B._run([B.NVCC, *B.ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC", *defs, *B.INC,
            "-c", os.path.join(B.CSRC, fname), "-o", obj])
    objs = [obj if f == fname else os.path.join(B.OBJ, f + ".o") for f in B.CU] + [
        os.path.join(B.OBJ, f + ".o") for f in B.CPP]
    lib_dir = os.path.join(ROOT, "scripts", "probes", "variants")
    os.makedirs(lib_dir, exist_ok=True)
    lib = os.path.join(lib_dir, f"libsfv_{name}.so")
    B._run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs, "-L/usr/local/cuda/lib64", "-lcusolver",
            "-Xlinker", "-rpath=/usr/local/cuda/lib64"])
    print(lib)


if __name__ == "__main__":
    main()
