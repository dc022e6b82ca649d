"""Parity at the BASELINE configurations' full sizes (GPU).

The C oracle (oracle/sfv_oracle.c, itself pinned bit-for-bit against the compiled
reference by test_golden.py) evaluates R(u) on a million cells in well under a second,
so the headline configurations are compared element by element at their real sizes:
C2 (1M cells), C3 (500k, neo-Hookean TL), C4 (1M, BDF2 with history), and C5 at 1.05M
Kuhn tetrahedra (the 24.6M-cell case is compared through size-independent properties).
"""
import numpy as np
import pytest

from oracle.bind import OracleCase
from paper_2502_17217_b200 import cases

pytestmark = pytest.mark.gpu


def _setup(name, n=None, t=1.0):
    from paper_2502_17217_b200 import solver as sv
    case = cases.config(name, n=n)
    mesh = case.mesh()
    ev = sv.ResidualEvaluator(mesh, case.physics)
    orc = OracleCase(mesh, case.physics)
    ev.set_time(t)
    orc.set_time(t)
    return sv, case, mesh, ev, orc


def _rel_linf(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("name,n", [("c2", None), ("c5", 56)])
def test_full_size_residual_and_jv_bitwise(name, n):
    sv, case, mesh, ev, orc = _setup(name, n)
    u, v = cases.jv_inputs(mesh, extent=case.mesh_args.get("extents"))
    r_orc = orc.residual(u)
    r_gpu = ev.residual(u).cpu().numpy()
    assert np.array_equal(r_gpu, r_orc)
    eps = 2.5e-8
    jv_gpu = sv.jacobian_vector_product(ev, u, r_orc, v, eps=eps).cpu().numpy()
    jv_orc = (orc.residual(u + eps * v) - r_orc) / eps
    assert np.array_equal(jv_gpu, jv_orc)


def test_full_size_jv_reference_eps():
    """J.v with the reference's own eps rule (nonlinear.cpp:109-115): eps differs from a
    sequential-sum eps only through the norm reduction order (a few ulps), so J.v agrees
    to finite-difference noise."""
    sv, case, mesh, ev, orc = _setup("c2")
    u, v = cases.jv_inputs(mesh, extent=case.mesh_args.get("extents"))
    r_u = orc.residual(u)
    jv_gpu = sv.jacobian_vector_product(ev, u, r_u, v).cpu().numpy()
    jv_orc = orc.jv(u, r_u, v)
    assert _rel_linf(jv_gpu, jv_orc) < 1e-6


def test_full_size_neo_hookean_tl_residual():
    """C3 at 500k cells, strains O(1e-2): within 1e-12 relative L-inf of the oracle (pow()
    in the neo-Hookean law is not correctly rounded on either side)."""
    sv, case, mesh, ev, orc = _setup("c3", t=0.5)
    u, _ = cases.jv_inputs(mesh, extent=case.mesh_args.get("extents"))
    u = u * 1e4
    r_orc = orc.residual(u)
    assert _rel_linf(ev.residual(u).cpu().numpy(), r_orc) < 1e-12


def test_full_size_transient_residual_bitwise():
    sv, case, mesh, ev, orc = _setup("c4")
    u, _ = cases.jv_inputs(mesh, extent=case.mesh_args.get("extents"))
    hist = [cases.uniform(20 + k, 3 * mesh.n_cells, -1e-6, 1e-6) for k in range(4)]
    ev.set_history(*hist)
    orc.set_history(*hist)
    assert np.array_equal(ev.residual(u).cpu().numpy(), orc.residual(u))


def test_c5_full_size_linearity():
    """C5 at its full 24.6M cells, where the CPU oracle is too slow to compare directly:
    for Hooke the residual is affine in u, so J.v at two eps must agree to FD noise, and
    R(u) - R(0) must be odd in u (R(u) + R(-u) = 2 R(0) up to rounding)."""
    from paper_2502_17217_b200 import solver as sv
    case = cases.config("c5")
    mesh = case.mesh()
    ev = sv.ResidualEvaluator(mesh, case.physics)
    ev.set_time(1.0)
    u, v = cases.jv_inputs(mesh, extent=case.mesh_args.get("extents"))
    r_u = ev.residual(u)
    j1 = sv.jacobian_vector_product(ev, u, r_u, v, eps=1e-7).cpu().numpy()
    j2 = sv.jacobian_vector_product(ev, u, r_u, v, eps=4e-7).cpu().numpy()
    assert _rel_linf(j1, j2) < 1e-5
    r0 = ev.residual(np.zeros_like(u)).cpu().numpy()
    rp = r_u.cpu().numpy()
    rm = ev.residual(-u).cpu().numpy()
    scale = np.max(np.abs(rp - r0))
    assert np.max(np.abs((rp - r0) + (rm - r0))) <= 1e-9 * scale
