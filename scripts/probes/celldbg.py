import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2502_17217_b200 import cases, solver as sv
case = cases.config("c2", n=24); mesh = case.mesh(); u, v = cases.jv_inputs(mesh)
res = {}
for fused in ("0", "1"):
    os.environ["SFV_EPS_FUSED"] = fused
    ev = sv.ResidualEvaluator(mesh, case.physics); ev.set_time(1.0)
    r_u = ev.residual(u)
    a = sv.jacobian_vector_product(ev, u, r_u, v).cpu().numpy()
    b = sv.jacobian_vector_product(ev, u, r_u, v).cpu().numpy()
    print(os.environ.get("SFV_FLUX"), fused, "repeat-equal", np.array_equal(a, b), np.abs(a - b).max())
    res[fused] = a
print("fused-vs-unfused", np.abs(res["0"] - res["1"]).max(), np.abs(res["0"]).max())
