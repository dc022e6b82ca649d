"""Build libsfv.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

Host geometry/mesh code is compiled like the reference (-O2, no FMA contraction on
baseline x86-64) so it is bit-identical to it; CUDA kernels are compiled with
-fmad=false for the same reason (see csrc/residual.cu).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "libsfv.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INC = ["-I" + os.path.join(ROOT, "include"), "-I" + CSRC]

CU = ["residual.cu", "jv_fused.cu", "jv_pair.cu", "krylov.cu", "precond.cu", "precond_stream.cu", "precond_pipe.cu",
      "geometry.cu", "segregated.cu", "precond_dev.cu", "mesh_dev.cu"]
CPP = ["host_mesh.cpp", "precond_host.cpp", "capi.cpp"]
HEADERS = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))] + [
    os.path.join(ROOT, "include", h) for h in ("sfv.h", "sfv_case.h")]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd: list[str]) -> None:
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    objs, jobs = [], []
    for f in CU:
        src = os.path.join(CSRC, f)
        obj = os.path.join(OBJ, f + ".o")
        if _stale(obj, [src] + HEADERS):
            jobs.append([NVCC, *ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                         "-Xptxas", "-v" if verbose else "-O3", *INC, "-c", src, "-o", obj])
        objs.append(obj)
    for f in CPP:
        src = os.path.join(CSRC, f)
        obj = os.path.join(OBJ, f + ".o")
        if _stale(obj, [src] + HEADERS):
            jobs.append(["g++", "-O2", "-ffp-contract=off", "-fPIC", "-std=c++17", "-Wall", "-Wno-unused-function",
                         *INC, "-I/usr/local/cuda/include", "-c", src, "-o", obj])
        objs.append(obj)
    if jobs:  # translation units compile independently
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            list(ex.map(_run, jobs))
    if _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-L/usr/local/cuda/lib64", "-lcusolver",
              "-Xlinker", "-rpath=/usr/local/cuda/lib64"])
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv)
