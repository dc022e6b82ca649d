export PYTHONPATH=$PWD
timeout 1200 python - <<'PY'
import numpy as np
from paper_2502_17217_b200 import cases, solver as sv
fx = np.load("tests/golden/full_c3.npz")
case = cases.config("c3"); mesh = case.mesh(); ev = sv.ResidualEvaluator(mesh, case.physics)
f, reps, wall = sv.run_steps_host(ev, case.initial_field(mesh), case.solver(), case.n_steps)
print("newton", [r.outer_iters for r in reps], "ref", fx["newton"].tolist())
for i, r in enumerate(reps):
    k = r.summary()["krylov_per_newton"]; kr = fx["krylov"][i][fx["krylov"][i] >= 0].tolist()
    if k != kr: print("step", i, "krylov", k, "ref", kr)
u = f[0].reshape(-1, 3)
err = np.abs(u[fx["sample_idx"]] - fx["u_sample"]).max() / float(fx["u_max"])
print("sample rel err (of max|u|)", err, "wall", wall)
c = u; edges = np.linspace(0, c.shape[0], 1025).astype(np.int64)
s = np.add.reduceat(c, edges[:-1], axis=0); q = np.add.reduceat(c*c, edges[:-1], axis=0); cnt = np.diff(edges)
rs, rq = fx["u_block_sum"], fx["u_block_sq"]
bound = 1e-8 * np.sqrt(np.maximum(rq, 1e-300) * cnt[:, None])
ratio = np.abs(s - rs) / bound
print("block sum max ratio to bound", ratio.max(), "at", np.unravel_index(ratio.argmax(), ratio.shape))
print("block sq max rel", (np.abs(q - rq) / np.maximum(rq, 1e-300)).max())
print("norm rel", abs(np.linalg.norm(f[0]) - float(fx["u_norm"])) / float(fx["u_norm"]))
PY
