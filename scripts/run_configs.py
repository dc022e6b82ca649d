"""Full BASELINE solves on one GPU: every load increment / time step of a configuration
through sfv_run_steps_host, with the per-step Newton and GMRES counts.

    python scripts/run_configs.py [--cases c1,c2,c3,c4] [--out F]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2502_17217_b200 import cases  # noqa: E402
from paper_2502_17217_b200 import solver as sv  # noqa: E402


def run(name, algorithm="jfnk", max_outer=0):
    case = cases.config(name)
    t0 = time.time()
    mesh = case.mesh()
    ev = sv.ResidualEvaluator(mesh, case.physics)
    setup = time.time() - t0
    f0 = case.initial_field(mesh)
    sv.run_steps_host(ev, f0, case.solver(max_outer=1, max_krylov=3, algorithm=algorithm), 1)  # warm-up
    f, reps, wall = sv.run_steps_host(ev, f0, case.solver(algorithm=algorithm, max_outer=max_outer), case.n_steps)
    s = [r.summary() for r in reps]
    return {"case": name, "algorithm": algorithm, "cells": mesh.n_cells, "steps": len(s), "solve_seconds": wall,
            "setup_seconds": setup, "outer_total": sum(x["outer_iters"] for x in s),
            "status": sorted(set(x["status"] for x in s)), "newton": [x["outer_iters"] for x in s],
            "krylov_total": sum(x["krylov_iters"] for x in s),
            "final_rel_residual_max": max(x["final_residual"] / max(x["initial_residual"], 1e-300) for x in s),
            "notes": case.notes}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="c1,c2,c3,c4")
    ap.add_argument("--out", default=None)
    ap.add_argument("--algorithm", default="jfnk", choices=["jfnk", "segregated"])
    ap.add_argument("--max-outer", type=int, default=0)
    args = ap.parse_args()
    rows = []
    for name in args.cases.split(","):
        row = run(name, args.algorithm, args.max_outer)
        print(json.dumps(row), flush=True)
        rows.append(row)
    if args.out:
        json.dump(rows, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
