"""Build a probe variant of libsfv.so with every source recompiled under extra defines
(scripts/probes/variants/libsfv_<name>.so, git-ignored; load with SFV_LIB=... for timing
experiments only).

    python scripts/build_full_variant.py <name> -DMACRO=value ...
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2502_17217_b200 import build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out_dir = os.path.join(ROOT, "build", "var", name)
    os.makedirs(out_dir, exist_ok=True)
    objs, jobs = [], []
    for f in B.CU:
        obj = os.path.join(out_dir, f + ".o")
        jobs.append([B.NVCC, *B.ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC", *defs,
                     *B.INC, "-c", os.path.join(B.CSRC, f), "-o", obj])
        objs.append(obj)
    for f in B.CPP:
        obj = os.path.join(out_dir, f + ".o")
        jobs.append(["g++", "-O2", "-ffp-contract=off", "-fPIC", "-std=c++17", *defs, *B.INC,
                     "-I/usr/local/cuda/include", "-c", os.path.join(B.CSRC, f), "-o", obj])
        objs.append(obj)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(B._run, jobs))
    lib_dir = os.path.join(ROOT, "scripts", "probes", "variants")
    os.makedirs(lib_dir, exist_ok=True)
    lib = os.path.join(lib_dir, f"libsfv_{name}.so")
    B._run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o", lib, *objs, "-L/usr/local/cuda/lib64", "-lcusolver",
            "-Xlinker", "-rpath=/usr/local/cuda/lib64"])
    print(lib)


if __name__ == "__main__":
    main()
