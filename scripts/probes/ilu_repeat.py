"""Repeatability of the streamed ILU(1) apply at C2 against the sync-free sweep (the truth): the
same right-hand sides applied repeatedly with device-built and host-built records."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2502_17217_b200 import cases, solver as sv  # noqa: E402

case = cases.config("c2")
mesh = case.mesh()
ev = sv.ResidualEvaluator(mesh, case.physics)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 2
seeds = tuple(int(x) for x in os.environ.get("ILU_SEEDS", "21,22,23").split(","))
rs = {s: sv.to_device(cases.uniform(s, 3 * mesh.n_cells)) for s in seeds}
os.environ["SFV_HOST_PRECOND"] = "1"
os.environ["SFV_TRI_CLUSTER"] = "0"
pc = sv.make_preconditioner(ev, "ilu1")
assert pc.info()["sweep"] == 0
truth = {s: pc.solve(rs[s]).cpu().numpy() for s in seeds}
del os.environ["SFV_TRI_CLUSTER"]
nbad = ntot = 0
for rnd in range(rounds):
    for host in (0, 1):
        if host:
            os.environ["SFV_HOST_PRECOND"] = "1"
        else:
            os.environ.pop("SFV_HOST_PRECOND", None)
        pc = sv.make_preconditioner(ev, "ilu1")
        assert pc.info()["sweep"] == 200
        for s in seeds:
            for k in range(reps):
                z = pc.solve(rs[s]).cpu().numpy()
                bad = np.nonzero(z != truth[s])[0]
                ntot += 1
                if len(bad):
                    nbad += 1
                    print(f"round {rnd} host={host} seed {s} rep {k}: {len(bad)} entries wrong, first {bad[:3]} (comp {bad[0] % 3}), "
                          f"cells {bad[0] // 3}..{bad[-1] // 3}")
print(f"done: {nbad} wrong of {ntot} applies")
