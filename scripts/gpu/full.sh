export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -k run_steps -s 2>&1 | grep -E "newton|passed|failed|assert|Error" | head -30
python - <<'PY'
import numpy as np
from paper_2502_17217_b200 import cases, solver as sv
case = cases.config("c2"); mesh = case.mesh(); ev = sv.ResidualEvaluator(mesh, case.physics)
f, reps, wall = sv.run_steps_host(ev, case.initial_field(mesh), case.solver(), 1)
s = reps[0].summary(); r = np.array(s["r_norms"]); print("ours", (r / r[0]).tolist())
z = np.load("tests/golden/full_c2.npz"); rr = z["r_norms"][0]; print("ref ", (rr / rr[0]).tolist())
PY
