export PYTHONPATH=$PWD
for v in "" fma "" fma; do
  if [ -n "$v" ]; then export SFV_LIB=scripts/probes/variants/libsfv_$v.so; else unset SFV_LIB; fi
  timeout 300 python scripts/microbench.py --config c2 --what jv --reps 300 2>&1 | grep -o '"jv_ms": [0-9.]*' | sed "s/^/${v:-nofma} /"
done
export SFV_LIB=scripts/probes/variants/libsfv_fma.so
timeout 600 python - <<'PY'
import numpy as np
from oracle.bind import OracleCase
from paper_2502_17217_b200 import cases, solver as sv
case = cases.config("c2", n=40); mesh = case.mesh()
ev = sv.ResidualEvaluator(mesh, case.physics); orc = OracleCase(mesh, case.physics)
ev.set_time(1.0); orc.set_time(1.0)
u, v = cases.jv_inputs(mesh)
r_g = ev.residual(u).cpu().numpy(); r_o = orc.residual(u)
print("fma build: R rel Linf", np.abs(r_g - r_o).max() / np.abs(r_o).max())
PY
