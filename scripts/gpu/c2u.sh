export PYTHONPATH=$PWD
python - <<'PY'
import numpy as np, json
from paper_2502_17217_b200 import cases, solver as sv
z = np.load("tests/golden/full_c2.npz")
case = cases.config("c2"); mesh = case.mesh(); ev = sv.ResidualEvaluator(mesh, case.physics)
f, reps, wall = sv.run_steps_host(ev, case.initial_field(mesh), case.solver(), 1)
u = f[0].reshape(-1, 3)
err = np.abs(u[z["sample_idx"]] - z["u_sample"]).max() / float(z["u_max"])
nrm = abs(np.linalg.norm(f[0]) - float(z["u_norm"])) / float(z["u_norm"])
# one more Newton step from our 9-step iterate: does it move toward the reference's 10-step field?
print(json.dumps({"newton": reps[0].outer_iters, "u_sample_rel_linf": err, "u_norm_rel": nrm, "wall": wall}))
PY
SFV_GMRES_GRAPH=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:arnoldi_kernel -s 10 -c 1 -o gpurun_out/r02_full_arnoldi_kernel python scripts/microbench.py --what gmres --reps 1 > gpurun_out/r02_ncu_arn.log 2>&1; echo arnoldi=$?
