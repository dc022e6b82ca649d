"""Known-answer tests of the reference's own suites, restated against the GPU path (SURVEY.md
§8c): the GMRES variants (test_linalg.cpp:244-292), the line-search schedule
(test_nonlinear.cpp:184-226), the deformed-area balance under uniform F
(test_discretisation.cpp:316-364) and the approximate-Jacobian coefficients, symmetry dyad and
inertia shift (test_discretisation.cpp:366-503); plus the DiscretisationConfig::body_force and
per-face boundary values (discretisation.cpp:82-85, :160-161) against the C oracle and the
compiled reference.  Every case runs through the C-ABI (libsfv.so) on the device.
"""
import numpy as np
import pytest

from oracle.bind import OracleCase, RefCase, ref_available
from paper_2502_17217_b200 import cases
from paper_2502_17217_b200.abi import (LAW_HOOKE, LAW_NEO_HOOKEAN, PATCH_DISPLACEMENT as D, PATCH_SYMMETRY as S,
                                       PATCH_TRACTION as T, Physics)

pytestmark = pytest.mark.gpu


def _sv():
    from paper_2502_17217_b200 import solver as sv
    return sv


def _hooke(npatch=6, bv=None, mu=3e6, lam=5e6, **kw):
    bvals = np.zeros((npatch, 3)) if bv is None else np.asarray(bv, dtype=float)
    return Physics(LAW_HOOKE, mu, lam, bc_value=bvals, bc_ramp=np.ones(npatch, dtype=np.int32), **kw)


# ---------------------------------------------------------------- GMRES variants
def _gmres_case(n=4):
    """op = J.v of a Hooke box (linear, so J is the system matrix), ILU(0) preconditioner."""
    sv = _sv()
    case = cases.config("c2", n=n)
    mesh = case.mesh()
    ev = sv.ResidualEvaluator(mesh, case.physics)
    orc = OracleCase(mesh, case.physics)
    for x in (ev, orc):
        x.set_time(1.0)
    u = np.zeros(3 * mesh.n_cells)
    r_u = orc.residual(u)
    b = -r_u
    return sv, mesh, ev, orc, u, r_u, b


@pytest.mark.parametrize("right", [False, True])
def test_gmres_left_and_right_preconditioned_vs_oracle(right):
    """test_linalg.cpp:244-271: left and right preconditioning both converge to the solution;
    the device GMRES follows the oracle's gmres_solve iteration for iteration (±1)."""
    sv, mesh, ev, orc, u, r_u, b = _gmres_case()
    sv.make_preconditioner(ev, "ilu0")
    orc.precond_create(2)
    # tolerances stay above the finite-difference noise of J.v (eps ~ 1.5e-8)
    x, it, st, rel = sv.gmres_jv(ev, u, r_u, b, restart=30, rel_reduction=1e-7, max_iters=300,
                                 right_preconditioned=right)
    xo, ito, sto, relo = orc.gmres_jv(u, r_u, b, restart=30, rel_reduction=1e-7, max_iters=300, right=right)
    assert st == "converged" and sto == 0
    assert abs(it - ito) <= 1, (it, ito)
    x = x.cpu().numpy()
    assert np.linalg.norm(x - xo) <= 1e-5 * np.linalg.norm(xo)
    # J x = b: R is affine in u (Hooke, small strain), so R(x) - R(0) = J x
    r_x = orc.residual(x) - r_u
    assert np.linalg.norm(r_x - b) <= 1e-4 * np.linalg.norm(b)


def test_gmres_unpreconditioned_full_space_and_restart_5():
    """test_linalg.cpp:273-286: unpreconditioned GMRES with a large Krylov space converges
    within its budget; restart 5 still converges through outer cycles."""
    sv, mesh, ev, orc, u, r_u, b = _gmres_case(n=3)
    sv.make_preconditioner(ev, "none")
    n = len(b)
    x, it, st, rel = sv.gmres_jv(ev, u, r_u, b, restart=n, rel_reduction=1e-7, max_iters=n)
    assert st == "converged" and it <= n
    sv.make_preconditioner(ev, "ilu0")
    x5, it5, st5, rel5 = sv.gmres_jv(ev, u, r_u, b, restart=5, rel_reduction=1e-7, max_iters=300)
    assert st5 == "converged"
    assert np.linalg.norm(x5.cpu().numpy() - x.cpu().numpy()) <= 1e-5 * np.linalg.norm(x.cpu().numpy())


def test_gmres_exhausts_budget():
    """test_linalg.cpp:288-296: a hopeless tolerance ends as not-converged within the budget."""
    sv, mesh, ev, orc, u, r_u, b = _gmres_case(n=3)
    sv.make_preconditioner(ev, "none")
    x, it, st, rel = sv.gmres_jv(ev, u, r_u, b, restart=5, rel_reduction=1e-16, max_iters=8)
    assert st != "converged" and it <= 8


def test_jfnk_right_preconditioned_matches_oracle():
    """SolverConfig::right_preconditioned through jfnk_solve / run_steps: Newton and Krylov
    counts within ±1 of the oracle, converged u within 1e-8."""
    sv = _sv()
    case = cases.config("c2", n=8)
    mesh = case.mesh()
    ev = sv.ResidualEvaluator(mesh, case.physics)
    orc = OracleCase(mesh, case.physics)
    cfg = case.solver(preconditioner="ilu1", right_preconditioned=True)
    f0 = case.initial_field(mesh)
    f, reps, _ = sv.run_steps_host(ev, f0, cfg, 1)
    fo, repo, _ = orc.run_steps(f0, cfg, 1)
    a, b = reps[0].summary(), repo[0].summary()
    assert a["status"] == "converged" and b["status"] == "converged"
    assert a["outer_iters"] == b["outer_iters"]
    assert all(abs(x - y) <= 1 for x, y in zip(a["krylov_per_newton"], b["krylov_per_newton"]))
    assert np.linalg.norm(f[0] - fo[0]) <= 1e-8 * np.linalg.norm(fo[0])


def test_unbounded_iteration_history():
    """SolveReport::iterations is unbounded (nonlinear.hpp:64): a segregated solve of more than
    64 outer iterations reports every one through the caller's history buffer."""
    sv = _sv()
    import ctypes as C
    from paper_2502_17217_b200.abi import SolveReport
    case = cases.config("c1", n=6)
    mesh = case.mesh()
    ev = sv.ResidualEvaluator(mesh, case.physics)
    cfg = case.solver(algorithm="segregated", max_outer=100)
    f = np.ascontiguousarray(case.initial_field(mesh), dtype=np.float64).reshape(-1).copy()
    reps = (SolveReport * 1)()
    reps[0].attach_history(512)
    nrep, wall = C.c_int(0), C.c_double(0.0)
    ev._check(ev.L.sfv_run_steps_host(ev.h, f.ctypes.data_as(C.POINTER(C.c_double)), C.byref(cfg), 1, reps, 1,
                                      C.byref(nrep), C.byref(wall)))
    rep = reps[0]
    assert rep.outer_iters > 64
    recs = rep.record_list()
    assert len(recs) == rep.n_records == rep.outer_iters + 1
    assert [r.iter for r in recs] == list(range(rep.outer_iters + 1))


# ---------------------------------------------------------------- line search
def test_line_search_schedule():
    """test_nonlinear.cpp:184-226 on the same 3x3x3 Hooke box: along c * (Newton step) the
    affine residual leaves |1 - s c| R0, so c = 1 takes s = 1, c = 3 takes s = 1/2, c = 40
    takes s = 1/32, c = -2 and a zero direction find no strict decrease."""
    sv = _sv()
    mesh = sv.box_mesh((0.3, 0.3, 0.3), (3, 3, 3), [D, T, T, T, T, T])
    ph = _hooke(bv=[(0, 0, 0), (1e4, 0, 0), (0, 0, 0), (0, 0, 0), (0, 0, 0), (0, 0, 0)])
    ev = sv.ResidualEvaluator(mesh, ph)
    orc = OracleCase(mesh, ph)
    for x in (ev, orc):
        x.set_time(1.0)
    n = 3 * mesh.n_cells
    u0 = np.zeros(n)
    r0 = orc.residual(u0)
    r_norm0 = float(np.sqrt(np.dot(r0, r0)))
    # dense Jacobian of the affine residual, then the Newton step J du = -R
    J = np.zeros((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1e-6
        J[:, j] = (orc.residual(e) - r0) / 1e-6
    newton = np.linalg.solve(J, -r0)
    ok, s, rn, res = sv.line_search(ev, u0, newton, r_norm0)
    assert ok and s == 1.0 and rn < 1e-6 * r_norm0
    assert abs(np.linalg.norm(res.cpu().numpy()) - rn) <= 1e-12 * rn
    ok, s, _, _ = sv.line_search(ev, u0, 3.0 * newton, r_norm0)
    assert ok and s == 0.5
    ok, s, _, _ = sv.line_search(ev, u0, 40.0 * newton, r_norm0)
    assert ok and s == 1.0 / 32.0
    ok, _, _, _ = sv.line_search(ev, u0, -2.0 * newton, r_norm0)
    assert not ok
    ok, _, _, _ = sv.line_search(ev, u0, np.zeros(n), r_norm0)
    assert not ok


# ---------------------------------------------------------------- approximate Jacobian
KBAR = 11e6  # 2 mu + lambda with mu = 3e6, lambda = 5e6


def _jac(mesh, ph):
    sv = _sv()
    ev = sv.ResidualEvaluator(mesh, ph)
    rp, col, blk = sv.approximate_jacobian(ev)

    def find(i, j):
        for k in range(rp[i], rp[i + 1]):
            if col[k] == j:
                return blk[k]
        return None
    return ev, rp, col, blk, find


def test_jacobian_hand_computed_coefficients():
    """test_discretisation.cpp:366-386: regular 2x2x2 box, xmin displacement."""
    sv = _sv()
    mesh = sv.box_mesh((1.0, 1.0, 1.0), (2, 2, 2), [D, T, T, T, T, T])
    _, _, _, _, find = _jac(mesh, _hooke())
    ci = 0.5 * KBAR
    cd = KBAR * (1.0 / 0.25) * 0.25
    assert find(0, 1) is not None
    assert find(0, 1)[0, 0] == pytest.approx(ci, rel=1e-13)
    assert find(0, 1)[1, 1] == pytest.approx(ci, rel=1e-13)
    assert find(0, 1)[0, 1] == 0.0
    assert find(0, 0)[0, 0] == pytest.approx(-(3.0 * ci + cd), rel=1e-13)
    assert find(0, 0)[1, 1] == pytest.approx(-(3.0 * ci + cd), rel=1e-13)
    assert find(7, 7)[0, 0] == pytest.approx(-3.0 * ci, rel=1e-13)


def test_jacobian_is_derivative_of_compact_exchange():
    """test_discretisation.cpp:388-431: on a distorted box the assembled J~ equals the
    derivative of the compact two-point exchange kbar |Delta|/|d| |Gamma| (u_N - u_P)."""
    sv = _sv()
    mesh = sv.box_mesh((1.0, 1.0, 1.0), (2, 2, 2), [D, T, T, T, T, T], distort=0.2, seed=6)
    ev, rp, col, blk, find = _jac(mesh, _hooke())
    g = ev.geometry()
    nc = mesh.n_cells
    area = g["area"].reshape(-1, 3)
    delta = g["delta"].reshape(-1, 3)
    dense = np.zeros((3 * nc, 3 * nc))
    for i in range(nc):
        for k in range(rp[i], rp[i + 1]):
            dense[3 * i:3 * i + 3, 3 * col[k]:3 * col[k] + 3] = blk[k]
    comp = np.zeros((3 * nc, 3 * nc))
    kinds = np.repeat(mesh.patch_kind, mesh.patch_count)
    for f in range(mesh.n_faces):
        coeff = KBAR * np.linalg.norm(delta[f]) / g["d_mag"][f] * np.linalg.norm(area[f])
        p = mesh.owner[f]
        for a in range(3):
            if f < mesh.n_internal:
                q = mesh.neighbour[f]
                comp[3 * p + a, 3 * q + a] += coeff
                comp[3 * p + a, 3 * p + a] -= coeff
                comp[3 * q + a, 3 * p + a] += coeff
                comp[3 * q + a, 3 * q + a] -= coeff
            elif kinds[f - mesh.n_internal] == D:
                comp[3 * p + a, 3 * p + a] -= coeff
    assert np.max(np.abs(comp - dense)) <= 1e-13 * KBAR


def test_jacobian_symmetry_dyad_inertia_shift_definiteness():
    """test_discretisation.cpp:433-503: the ymin symmetry face adds -c n n on the adjacent
    diagonals; the BDF2 assembly shifts only the diagonal by -2.25 rho V / dt^2; J~ is
    symmetric and -J~ positive definite; alpha does not reach the matrix."""
    sv = _sv()
    mixed = [D, T, S, T, T, T]
    m = sv.box_mesh((1.0, 1.0, 0.5), (2, 2, 1), mixed)
    m2 = sv.box_mesh((1.0, 1.0, 0.5), (2, 2, 1), [D, T, T, T, T, T])
    _, rp, col, blk, with_sym = _jac(m, _hooke())
    _, _, _, _, without = _jac(m2, _hooke())
    cs = KBAR * (1.0 / 0.5) * 0.25
    for c in (0, 1):
        diff = with_sym(c, c) - without(c, c)
        expect = np.zeros((3, 3))
        expect[1, 1] = -cs
        assert np.linalg.norm(diff - expect) < 1e-13 * cs
    dt, rho = 0.01, 1000.0
    _, _, _, _, trans = _jac(m, _hooke(transient=True, dt=dt, rho=rho))
    shift = -2.25 * rho * 0.125 / (dt * dt)
    for c in range(m.n_cells):
        assert np.linalg.norm(trans(c, c) - with_sym(c, c) - shift * np.eye(3)) < 1e-12 * abs(shift)
        assert np.linalg.norm(trans(c, c ^ 1) - with_sym(c, c ^ 1)) == 0.0
    nn = 3 * m.n_cells
    dense = np.zeros((nn, nn))
    for i in range(m.n_cells):
        for k in range(rp[i], rp[i + 1]):
            dense[3 * i:3 * i + 3, 3 * col[k]:3 * col[k] + 3] = blk[k]
    assert np.max(np.abs(dense - dense.T)) <= 1e-13 * KBAR
    np.linalg.cholesky(-dense)  # raises unless -J~ is positive definite
    _, _, _, _, scaled = _jac(m, _hooke(alpha=0.25))
    assert np.linalg.norm(scaled(0, 0) - with_sym(0, 0)) == 0.0


# ---------------------------------------------------------------- total Lagrangian balance
def _neo_hookean_stress(g, mu, kappa):
    """neo_hookean_stress (laws.cpp:39-47) in numpy."""
    F = np.eye(3) + g.T
    J = np.linalg.det(F)
    b_bar = J ** (-2.0 / 3.0) * (F @ F.T)
    s = (mu / J) * (b_bar - np.trace(b_bar) / 3.0 * np.eye(3))
    return s + 0.5 * kappa * (J * J - 1.0) / J * np.eye(3)


def test_total_lagrangian_uniform_deformation_balances():
    """test_discretisation.cpp:316-364: under a uniform F the transformed internal fluxes
    cancel and the nominal tractions det(F) sigma F^-T n close every cell's balance in the
    total Lagrangian residual; the small-strain residual does not balance."""
    sv = _sv()
    mesh = sv.box_mesh((0.3, 0.2, 0.2), (3, 2, 2), [T] * 6)
    rng = np.random.default_rng(17)
    g = 0.05 * rng.uniform(size=(3, 3))
    F = np.eye(3) + g.T
    mu, kappa = 3e6, 7e6
    sigma = _neo_hookean_stress(g, mu, kappa)
    nominal = np.linalg.det(F) * sigma @ np.linalg.inv(F).T
    normals = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]
    bv = np.array([nominal @ np.array(n, dtype=float) for n in normals])

    def residual(tl):
        ph = Physics(LAW_NEO_HOOKEAN, mu, kappa, total_lagrangian=tl, bc_value=bv,
                     bc_ramp=np.zeros(6, dtype=np.int32))
        ev = sv.ResidualEvaluator(mesh, ph)
        ev.set_time(1.0)
        x = ev.geometry()["centroid"].reshape(-1, 3)
        u = ((F - np.eye(3)) @ x.T).T.reshape(-1)
        return ev.residual(u).cpu().numpy().reshape(-1, 3)

    scale = np.linalg.norm(sigma) * 0.01
    assert np.max(np.linalg.norm(residual(True), axis=1)) < 1e-11 * scale
    assert np.max(np.linalg.norm(residual(False), axis=1)) > 1e-6 * scale


# ---------------------------------------------------------------- body force, per-face BCs
def _bf_case():
    sv = _sv()
    case = cases.config("c2", n=7)
    mesh = case.mesh()
    ev = sv.ResidualEvaluator(mesh, case.physics)
    orc = OracleCase(mesh, case.physics)
    g = ev.geometry()
    x = g["centroid"].reshape(-1, 3)
    # a polynomial body force density evaluated at the centroids (N/m^3)
    f = np.stack([1e6 * x[:, 1] + 2e5, -3e5 * x[:, 2] * x[:, 0], 4e5 + 0.0 * x[:, 0]], axis=1).reshape(-1)
    xf = g["face_centroid"].reshape(-1, 3)[mesh.n_internal:]
    kinds = np.repeat(mesh.patch_kind, mesh.patch_count)

    def face_values(t):
        # traction faces: a position-dependent load; displacement faces: a small prescribed field
        tr = np.stack([1e6 * (1.0 + xf[:, 1]) * t, 2e5 * xf[:, 2] * t, 0.0 * xf[:, 0]], axis=1)
        di = np.stack([1e-4 * xf[:, 1] * t, 0.0 * xf[:, 0], -5e-5 * xf[:, 2] * t], axis=1)
        return np.where((kinds == D)[:, None], di, tr).reshape(-1)
    return sv, case, mesh, ev, orc, f, face_values


def test_body_force_and_face_values_bitwise():
    """R(u) with a body force and per-face boundary values is bit-identical to the oracle,
    and the oracle to the compiled reference (its body_force / BoundaryCondition functions
    return the same samples); J.v at a fixed eps too."""
    sv, case, mesh, ev, orc, f, face_values = _bf_case()
    for x in (ev, orc):
        x.set_time(0.6)
    ev.set_body_force(f)
    orc.set_body_force(f)
    ev.set_boundary_values(face_values(0.6))
    orc.set_face_bc(face_values(0.6))
    u, v = cases.jv_inputs(mesh)
    r = orc.residual(u)
    assert np.array_equal(ev.residual(u).cpu().numpy(), r)
    eps = 4e-8
    jv = sv.jacobian_vector_product(ev, u, r, v, eps=eps).cpu().numpy()
    assert np.array_equal(jv, (orc.residual(u + eps * v) - r) / eps)
    if ref_available():
        ref = RefCase(mesh, case.physics)
        ref.set_time(0.6)
        ref.set_body_force(f)
        ref.set_face_bc(face_values(0.6))
        assert np.array_equal(ref.residual(u), r)


def test_boundary_sampler_in_run_steps():
    """A time-dependent per-face boundary function sampled on every step of run_steps (two
    load increments) gives the oracle's solve when the oracle is fed the same samples step by
    step: Newton counts equal, Krylov ±1, field within 1e-8."""
    sv, case, mesh, ev, orc, f, face_values = _bf_case()
    ev.set_body_force(f)
    orc.set_body_force(f)
    seen = []

    def sampler(t):
        seen.append(t)
        return face_values(t)
    ev.set_boundary_sampler(sampler)
    cfg = case.solver(preconditioner="ilu1")
    f0 = case.initial_field(mesh)
    fg, reps, _ = sv.run_steps_host(ev, f0, cfg, 2)
    assert 0.5 in seen and 1.0 in seen
    # the oracle, one increment at a time with the samples of that increment
    orc.precond_create(3)
    field = f0
    for step, t in ((1, 0.5), (2, 1.0)):
        orc.set_face_bc(face_values(t))
        cur = field.copy()
        orc.set_time(t)
        u, rep = orc.jfnk_solve(cur[0], cfg)
        ref_rep = rep.summary()
        got = reps[step - 1].summary()
        assert got["outer_iters"] == ref_rep["outer_iters"]
        assert all(abs(a - b) <= 1 for a, b in zip(got["krylov_per_newton"], ref_rep["krylov_per_newton"]))
        field = cur
        field[0] = u
    assert np.linalg.norm(fg[0] - field[0]) <= 1e-8 * np.linalg.norm(field[0])
