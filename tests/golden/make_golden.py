"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself
(oracle/_ref/libsolidfv_ref.so, compiled from /root/reference/proj/src by oracle/Makefile).

    python tests/golden/make_golden.py

Each fixture holds the mesh (from the reference's own generate_box_hex/distort_mesh, or
the config-5 tet generator for the tet case), the physics, seeded inputs, and the
reference's outputs: R(u), J.v, stabilisation, ILU(1) and LU applies, and a short
run_steps history.  tests/test_golden.py checks the C oracle (and, on a GPU box, the
CUDA path) against them; nothing at test time needs /root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.bind import RefCase, ref_box_mesh  # noqa: E402
from paper_2502_17217_b200 import cases  # noqa: E402
from paper_2502_17217_b200.abi import (LAW_GUCCIONE, LAW_HOOKE, LAW_J2, LAW_NEO_HOOKEAN, LAW_STVK,  # noqa: E402
                                       PATCH_DISPLACEMENT as D, PATCH_SYMMETRY as S, PATCH_TRACTION as T, Mesh,
                                       Physics, solver_cfg)

CASES = {
    "hex_hooke": dict(mesh=((1.0, 1.2, 0.8), (6, 5, 4), [D, T, T, T, T, T], 0.15, 42), law=LAW_HOOKE),
    "hex_symmetry": dict(mesh=((1.0, 1.0, 1.0), (5, 4, 4), [D, T, S, T, S, T], 0.1, 3), law=LAW_HOOKE),
    "hex_neohookean_tl": dict(mesh=((4.0, 1.0, 1.0), (12, 4, 4), [D, D, T, T, T, T], 0.05, 42),
                              law=LAW_NEO_HOOKEAN, tl=True),
    "hex_transient": dict(mesh=((1.0, 1.0, 1.0), (5, 5, 5), [D, T, T, T, T, T], 0.15, 42), law=LAW_HOOKE,
                          transient=True),
    "tets": dict(tets=4, law=LAW_HOOKE),
    # the remaining hyperelastic laws on the same residual
    "hex_stvk": dict(mesh=((4.0, 1.0, 1.0), (12, 4, 4), [D, D, T, T, T, T], 0.05, 42), law=LAW_STVK, disp=0.3),
    "hex_guccione_tl": dict(mesh=((4.0, 1.0, 1.0), (12, 4, 4), [D, D, T, T, T, T], 0.05, 42), law=LAW_GUCCIONE,
                            tl=True, disp=0.02),
    # J2 plasticity with saturation hardening; the stepped solve commits the plastic state
    # after every increment (nonlinear.cpp:426), so steps 2-3 start from a yielded state
    # the segregated solver (nonlinear.cpp:268-351, IC(0)-CG per component, linalg.cpp:174-421)
    "hex_segregated": dict(mesh=((1.0, 1.0, 1.0), (6, 5, 4), [D, T, T, T, T, T], 0.1, 5), law=LAW_HOOKE,
                           alg="segregated", steps=1),
    "hex_j2": dict(mesh=((4.0, 1.0, 1.0), (12, 4, 4), [D, D, T, T, T, T], 0.05, 42), law=LAW_J2, disp=0.03, steps=3),
}
# steel-like J2: E = 200 GPa, nu = 0.3 (mu, kappa); HardeningCurve::saturation(a, b, c, d)
J2_MU, J2_KAPPA = 200e9 / (2.0 * 1.3), 200e9 / (3.0 * (1.0 - 0.6))
J2_CURVE = (250e6, 1e9, 400e6, 20.0)
# GuccioneParams of the reference's own law test (test_laws.cpp:170-175): f0 = Vec3{1, 2, 2} / 3,
# which types.hpp evaluates as a multiplication by (1.0 / 3.0)
GUCCIONE = (10e3, 8.0, 2.0, 4.0, 50e3, 1.0 * (1.0 / 3.0), 2.0 * (1.0 / 3.0), 2.0 * (1.0 / 3.0))


def physics(spec, npatch):
    bv = np.zeros((npatch, 3))
    bv[1] = (1e6, 2e5, -1e5)
    bv[3] = (0.5e6, 0.0, 0.0)
    if spec["law"] == LAW_HOOKE:
        mu, lam = cases.mu_from(200e9, 0.3), cases.lambda_from(200e9, 0.3)
    elif spec["law"] == LAW_J2:
        mu, lam = J2_MU, J2_KAPPA
        bv[1] = (spec.get("disp", 0.3), 0.0, 0.0)
    else:
        mu, lam = 0.4e6, 2e6
        bv[1] = (spec.get("disp", 0.3), 0.0, 0.0)  # prescribed displacement on xmax (C3 style)
    return Physics(spec["law"], mu, lam, total_lagrangian=spec.get("tl", False),
                   transient=spec.get("transient", False), dt=1e-5, rho=7800.0, bc_value=bv,
                   bc_ramp=np.ones(npatch, dtype=np.int32), guccione=GUCCIONE, j2_curve=J2_CURVE)


def mesh_for(spec) -> Mesh:
    if "tets" in spec:
        from paper_2502_17217_b200.solver import kuhn_tet_mesh
        return kuhn_tet_mesh((1.0, 1.0, 1.0), spec["tets"], [D, T, T, T, T, T], 42, True, True)
    return ref_box_mesh(*spec["mesh"])


def main():
    only = set(sys.argv[1:])
    for name, spec in CASES.items():
        if only and name not in only:
            continue
        m = mesh_for(spec)
        ph = physics(spec, len(m.patch_kind))
        ref = RefCase(m, ph)
        ref.set_time(0.7)
        u, v = cases.jv_inputs(m, seed=13)
        if spec["law"] != LAW_HOOKE:
            u = u * (1e3 if spec["law"] == LAW_J2 else 1e4)
        rng = np.random.default_rng(7)
        hist = np.zeros((4, 3 * m.n_cells))
        if spec.get("transient"):
            hist = rng.uniform(-1e-6, 1e-6, (4, 3 * m.n_cells))
            ref.set_history(*hist)
        r = ref.residual(u)
        jv = ref.jv(u, r, v)
        stab = ref.stabilisation(u)
        out = dict(points=m.points, face_offsets=m.face_offsets, face_points=m.face_points, owner=m.owner,
                   neighbour=m.neighbour, n_cells=m.n_cells, n_internal=m.n_internal, patch_kind=m.patch_kind,
                   patch_start=m.patch_start, patch_count=m.patch_count, law=ph.law, mu=ph.mu, lam=ph.lam,
                   tl=int(ph.total_lagrangian), transient=int(ph.transient), dt=ph.dt, rho=ph.rho,
                   bc_value=ph.bc_value, bc_ramp=ph.bc_ramp, guccione=np.array(ph.guccione),
                   j2_curve=np.array(ph.j2_curve), time=0.7, u=u, v=v, hist=hist, residual=r, jv=jv,
                   stabilisation=stab)
        zin = cases.uniform(21, 3 * m.n_cells)
        if not (m.patch_kind == S).any():
            ref.precond_create(3)
            out["ilu1_in"], out["ilu1_out"] = zin, ref.precond_apply(zin)
        ref.precond_create(5)
        out["lu_out"] = ref.precond_apply(zin)
        out["lu_in"] = zin
        # short run_steps history at r_tol 1e-8 with the automatic preconditioner (LU here)
        f0 = np.zeros((6, 3 * m.n_cells))
        if spec.get("transient"):
            f0[3] = f0[4] = cases.sinusoid_field(cases.cell_centres(m), 1234, 1.0)
        ref2 = RefCase(m, ph)
        cfg = solver_cfg(r_tol=1e-8 if spec.get("alg", "jfnk") == "jfnk" else 1e-6, algorithm=spec.get("alg", "jfnk"))
        steps = spec.get("steps", 2)
        f, reps, _ = ref2.run_steps(f0, cfg, steps)
        out["steps_field0"] = f0
        out["steps_field"] = f
        out["steps_krylov"] = np.array([sum(r.summary()["krylov_per_newton"]) for r in reps])
        out["steps_newton"] = np.array([r.outer_iters for r in reps])
        out["steps_status"] = np.array([r.status for r in reps])
        out["steps_n"] = steps
        out["steps_alg"] = 1 if spec.get("alg") == "segregated" else 0
        out["steps_rtol"] = cfg.r_tol
        if spec["law"] == LAW_J2:  # R after a commit: the residual reads the committed state
            ref3 = RefCase(m, ph)
            ref3.set_time(0.7)
            ref3.commit(u)
            out["residual_after_commit"] = ref3.residual(0.5 * u)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, m.n_cells, "cells", "newton", out["steps_newton"], "krylov", out["steps_krylov"])


if __name__ == "__main__":
    main()
