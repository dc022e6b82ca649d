"""How sensitive is the C2 Newton count to the summation order of GMRES's inner products?

Runs the C restatement (oracle/sfv_oracle.c — bit-identical to the reference with its own
sequential std::inner_product order) on the full C2 solve with ORC_DOT_BLOCK=k, i.e. GMRES
dot products and norms summed in blocks of k (an equally valid order), and prints the
per-Newton relative residuals.  Test infrastructure / evidence only.

    ORC_DOT_BLOCK=4096 python scripts/order_sensitivity.py [--n 100] [--out F]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.bind import OracleCase  # noqa: E402
from paper_2502_17217_b200 import cases  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    case = cases.config("c2", n=a.n)
    mesh = case.mesh()
    orc = OracleCase(mesh, case.physics)
    t0 = time.time()
    f, reps, wall = orc.run_steps(case.initial_field(mesh), case.solver(), 1)
    s = reps[0].summary()
    r = s["r_norms"]
    row = {"n": a.n, "dot_block": os.environ.get("ORC_DOT_BLOCK", "0 (sequential, the reference's order)"),
           "newton": s["outer_iters"], "krylov_per_newton": s["krylov_per_newton"],
           "rel_residuals": [x / r[0] for x in r], "seconds": time.time() - t0}
    print(json.dumps(row), flush=True)
    if a.out:
        json.dump(row, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
