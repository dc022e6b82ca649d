"""J.v throughput over the BASELINE configurations and the C5 size sweep (1e5 .. 2.46e7
cells), with the per-stage breakdown (CUDA events, sfv_jv_stage_times) — one JSON line per
case, collected into profiles/<tag>_jv_sweep.json by --out.

    python scripts/jv_sweep.py [--cases c2,c3,c4,c5:26,c5:56,c5:118,c5:160] [--reps 50] [--out F]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_17217_b200 import cases  # noqa: E402
from paper_2502_17217_b200 import solver as sv  # noqa: E402

NAMES = ["norm_partials_kernel", "eps_perturb_kernel", "grad_cell_kernel", "boundary_kernel", "flux_pair_kernel"]


def peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"])
    return 6650.0


def run(spec, reps):
    name, _, n = spec.partition(":")
    case = cases.config(name, n=int(n) if n else None)
    t0 = time.time()
    mesh = case.mesh()
    ev = sv.ResidualEvaluator(mesh, case.physics)
    ev.set_time(1.0)
    setup = time.time() - t0
    u_h, v_h = cases.jv_inputs(mesh, extent=case.mesh_args.get("extents"))
    u, v = sv.to_device(u_h), sv.to_device(v_h)
    r_u = ev.residual(u)
    out = ev.empty()
    L, h = ev.L, ev.h
    for _ in range(5):
        ev._check(L.sfv_jv_async(h, u.data_ptr(), r_u.data_ptr(), v.data_ptr(), out.data_ptr()))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        L.sfv_jv_async(h, u.data_ptr(), r_u.data_ptr(), v.data_ptr(), out.data_ptr())
    b.record()
    torch.cuda.synchronize()
    ev._check(L.sfv_check_errors(h, None))
    ms = a.elapsed_time(b) / reps
    st_ms, st_b = (C.c_double * 5)(), (C.c_double * 5)()
    L.sfv_jv_stage_bytes(h, st_b)
    ev._check(L.sfv_jv_stage_times(h, u.data_ptr(), r_u.data_ptr(), v.data_ptr(), out.data_ptr(), max(5, reps // 2),
                                   st_ms))
    pk = peak()
    jvb = ev.jv_bytes
    stages = [{"kernel": NAMES[k], "us": round(1e3 * st_ms[k], 2), "MB": round(st_b[k] / 1e6, 1),
               "frac_of_peak": round(st_b[k] / (st_ms[k] / 1e3) / 1e9 / pk, 3) if st_ms[k] > 0 else None}
              for k in range(5)]
    return {"case": spec, "cells": mesh.n_cells, "faces": mesh.n_faces, "jv_ms": round(ms, 4),
            "jv_per_s": round(1e3 / ms, 1), "cell_dof_per_s": 3 * mesh.n_cells * 1e3 / ms,
            "jv_frac_of_peak_survey_model": round(jvb / (ms / 1e3) / 1e9 / pk, 3), "setup_s": round(setup, 1),
            "stages": stages, "notes": case.notes}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="c2,c3,c4,c5:26,c5:56,c5:118,c5:160")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    for spec in args.cases.split(","):
        row = run(spec, args.reps)
        print(json.dumps(row), flush=True)
        rows.append(row)
        torch.cuda.empty_cache()
    if args.out:
        json.dump({"peak_gbs": peak(), "rows": rows}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
