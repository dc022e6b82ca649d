"""Component timings on one GPU (CUDA events on the context stream):
J.v, R(u), ILU(k) apply, and one GMRES(30) cycle, on a BASELINE config.

    python scripts/microbench.py [--config c2] [--n N] [--reps 20] [--what jv,ilu,gmres]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_17217_b200 import cases  # noqa: E402
from paper_2502_17217_b200 import solver as sv  # noqa: E402


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--what", default="jv,res,ilu,gmres")
    ap.add_argument("--precond", default="ilu1")
    args = ap.parse_args()
    what = set(args.what.split(","))
    case = cases.config(args.config, n=args.n)
    t0 = time.time()
    mesh = case.mesh()
    ev = sv.ResidualEvaluator(mesh, case.physics)
    ev.set_time(1.0)
    out = {"config": args.config, "cells": mesh.n_cells, "setup_s": time.time() - t0,
           "env": {k: v for k, v in os.environ.items() if k.startswith("SFV_")}}
    u_h, v_h = cases.jv_inputs(mesh, extent=case.mesh_args.get("extents"))
    u, v = sv.to_device(u_h), sv.to_device(v_h)
    r_u = ev.residual(u)
    o = ev.empty()
    if "jv" in what:
        ms = timed(lambda: ev.L.sfv_jv_async(ev.h, u.data_ptr(), r_u.data_ptr(), v.data_ptr(), o.data_ptr()),
                   args.reps)
        out["jv_ms"] = ms
        out["jv_GBps_algorithmic"] = ev.jv_bytes / (ms * 1e-3) / 1e9
    if "res" in what:
        import ctypes as C
        cell = C.c_int(0)
        out["residual_ms_incl_sync"] = timed(
            lambda: ev.L.sfv_residual(ev.h, u.data_ptr(), o.data_ptr(), C.byref(cell)), args.reps)
    if "ilu" in what or "gmres" in what:
        t1 = time.time()
        pc = sv.make_preconditioner(ev, args.precond)
        out["precond_setup_s"] = time.time() - t1
        out["precond_info"] = pc.info()
    if "ilu" in what:
        r = sv.to_device(cases.uniform(3, ev.n))
        z = ev.empty()
        out["precond_apply_ms_incl_sync"] = timed(lambda: ev.L.sfv_precond_apply(ev.h, r.data_ptr(), z.data_ptr()),
                                                  max(3, args.reps // 2))
    if "gmres" in what:
        b = -r_u
        t1 = time.time()
        x, it, st, rel = sv.gmres_jv(ev, u, r_u, b, restart=30, rel_reduction=1e-12, max_iters=30)
        torch.cuda.synchronize()
        dt = time.time() - t1
        out["gmres_cycle"] = {"iters": it, "status": st, "rel": rel, "s": dt, "ms_per_iter": 1e3 * dt / max(it, 1)}
    out["launches"] = ev.launch_count
    print(json.dumps(out))


if __name__ == "__main__":
    main()
