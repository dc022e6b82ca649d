:  tests/test_gpu_parity.py -m gpu -x -q -k "ilu" 2>&1 | tail -3
cat > /tmp/ilu_t.py <<'PY'
import time
from paper_2502_17217_b200 import cases, solver as sv
case = cases.config("c2")
mesh = case.mesh()
ev = sv.ResidualEvaluator(mesh, case.physics)
for k in range(2):
    t = time.perf_counter(); pc = sv.make_preconditioner(ev, "ilu1"); print("setup", time.perf_counter() - t, flush=True)
PY
for d in 0 1; do echo "== SFV_DEVICE_ILU=$d"; if [ $d = 1 ]; then export SFV_DEVICE_ILU=1; fi; PYTHONPATH=$PWD SFV_TIMING=1 timeout 300 python /tmp/ilu_t.py 2>&1 | grep -i 'ilu\|setup'; done
