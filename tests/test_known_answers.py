"""The reference's own known-answer properties for this path,
restated against both the C oracle (CPU suite) and the GPU path (-m gpu):

  * LS gradients exact on affine fields, regular and distorted box
    (reference: proj/tests/test_discretisation.cpp:66-87, 1e-11 rel)  [GPU: sfv_gradients]
  * Rhie-Chow 5-point pattern on a 9-cell bar, alpha-linearity, zero sum (:97-144)
  * stabilisation vanishes on affine fields on a distorted mesh (:224-241, 1e-12 scale)
  * transient R differs from static R by exactly rho*Omega*a_BDF2 (:259-294, 1e-12 rel)
  * J.v against a dense finite-difference Jacobian on a 3^3 linear box, zero v -> 0
    (proj/tests/test_nonlinear.cpp:130-153, 1e-6 rel-L2)
  * JFNK on a 3^3 linear box with the exact preconditioner converges in 1..5 Newton
    steps; zero load -> zero Newton iterations (:255-296)
"""
import numpy as np
import pytest

from paper_2502_17217_b200 import cases
from paper_2502_17217_b200.abi import (LAW_HOOKE, PATCH_DISPLACEMENT as D, PATCH_SYMMETRY as S,
                                       PATCH_TRACTION as T, Physics, solver_cfg)

BACKENDS = ["oracle", pytest.param("gpu", marks=pytest.mark.gpu)]


class _Gpu:
    def __init__(self, mesh, phys):
        from paper_2502_17217_b200 import solver as sv
        self.sv = sv
        self.ev = sv.ResidualEvaluator(mesh, phys)

    def set_time(self, t):
        self.ev.set_time(t)

    def set_history(self, *h):
        self.ev.set_history(*h)

    def residual(self, u):
        return self.ev.residual(u).cpu().numpy()

    def stabilisation(self, u):
        return self.ev.stabilisation(u).cpu().numpy()

    def jv(self, u, r_u, v):
        return self.sv.jacobian_vector_product(self.ev, u, r_u, v).cpu().numpy()

    def geometry(self):
        return self.ev.geometry()

    def jfnk(self, u, cfg):
        ud, rep = self.sv.jfnk_solve(self.ev, u, cfg)
        return ud.cpu().numpy(), rep


class _Oracle:
    def __init__(self, mesh, phys):
        from oracle.bind import OracleCase
        self.o = OracleCase(mesh, phys)

    def __getattr__(self, k):
        return getattr(self.o, k)

    def jfnk(self, u, cfg):
        return self.o.jfnk_solve(u, cfg)


def _make(backend, mesh, phys):
    return _Gpu(mesh, phys) if backend == "gpu" else _Oracle(mesh, phys)


def _mesh(extents, divisions, kinds, distort=0.0, seed=0):
    from paper_2502_17217_b200.solver import box_mesh
    return box_mesh(extents, divisions, kinds, distort, seed)


def _hooke(npatch=6, alpha=1.0, transient=False, bc=None):
    bv = np.zeros((npatch, 3)) if bc is None else np.asarray(bc, dtype=np.float64)
    return Physics(LAW_HOOKE, cases.mu_from(200e9, 0.3), cases.lambda_from(200e9, 0.3), alpha=alpha,
                   transient=transient, dt=1e-4, rho=7800.0, bc_value=bv, bc_ramp=np.zeros(npatch, dtype=np.int32))


def _centroids(be):
    return be.geometry()["centroid"].reshape(-1, 3)


A = np.array([[1.0e-3, -2.0e-4, 3.0e-4], [5.0e-4, 2.0e-3, -1.0e-4], [-3.0e-4, 4.0e-4, 1.5e-3]])
B = np.array([1e-4, -2e-4, 3e-4])


def _affine(x):  # u_j = sum_i A[i, j] x_i + b_j, so grad(i, j) = du_j/dx_i = A[i, j]
    return (x @ A + B).reshape(-1)


@pytest.mark.gpu
@pytest.mark.parametrize("distort", [0.0, 0.2])
def test_gradients_exact_on_affine_fields(distort):
    mesh = _mesh((1.0, 1.3, 0.7), (6, 5, 4), [T] * 6, distort, 11)
    be = _Gpu(mesh, _hooke())
    G = be.ev.gradients(_affine(_centroids(be))).cpu().numpy()
    assert np.max(np.abs(G - A[None])) <= 1e-11 * np.max(np.abs(A))


@pytest.mark.parametrize("backend", BACKENDS)
def test_stabilisation_vanishes_on_affine_fields(backend):
    mesh = _mesh((1.0, 1.0, 1.0), (6, 6, 6), [T] * 6, 0.2, 5)
    be = _make(backend, mesh, _hooke())
    u = _affine(_centroids(be))
    s = be.stabilisation(u)
    kbar = 2 * cases.mu_from(200e9, 0.3) + cases.lambda_from(200e9, 0.3)
    scale = kbar * np.max(np.abs(A)) * (1.0 / 6) ** 2  # alpha K |Gamma| |grad u| |d|
    assert np.max(np.abs(s)) <= 1e-12 * scale


@pytest.mark.parametrize("backend", BACKENDS)
def test_rhie_chow_bar_pattern(backend):
    """A unit axial spike in a 9-cell bar (unit cross-section, traction ends, symmetry
    planes on the four sides so the stencil is 3-D): the stabilisation is
    alpha K |Gamma| / (4 dx) [-1, 4, -6, 4, -1] around it, linear in alpha, zero sum."""
    n, dx = 9, 0.5
    mesh = _mesh((n * dx, 1.0, 1.0), (n, 1, 1), [T, T, S, S, S, S])
    kbar = 2 * cases.mu_from(200e9, 0.3) + cases.lambda_from(200e9, 0.3)
    u = np.zeros(3 * n)
    u[3 * 4] = 1.0
    out = {}
    for alpha in (1.0, 0.5):
        s = _make(backend, mesh, _hooke(alpha=alpha)).stabilisation(u).reshape(n, 3)
        out[alpha] = s
        expect = alpha * kbar / (4 * dx) * np.array([-1.0, 4.0, -6.0, 4.0, -1.0])
        got = s[2:7, 0]
        assert np.allclose(np.abs(got), np.abs(expect), rtol=1e-12, atol=0)
        assert np.allclose(got / got[2], expect / expect[2], rtol=1e-12)
        assert abs(s[:, 0].sum()) <= 1e-12 * np.max(np.abs(s))
        assert np.all(s[:, 1:] == 0.0)
    assert np.allclose(out[0.5], 0.5 * out[1.0], rtol=1e-14, atol=0)


@pytest.mark.parametrize("backend", BACKENDS)
def test_transient_offset_is_bdf2_inertia(backend):
    mesh = _mesh((1.0, 1.0, 1.0), (5, 4, 3), [D, T, T, T, T, T], 0.1, 2)
    bc = np.zeros((6, 3))
    bc[1] = (1e6, 0.0, 0.0)
    u = cases.uniform(1, 3 * mesh.n_cells, -1e-6, 1e-6)
    hist = [cases.uniform(2 + k, 3 * mesh.n_cells, -1e-6, 1e-6) for k in range(4)]
    st = _make(backend, mesh, _hooke(bc=bc))
    tr = _make(backend, mesh, _hooke(bc=bc, transient=True))
    st.set_time(1.0)
    tr.set_time(1.0)
    tr.set_history(*hist)
    dt, rho = 1e-4, 7800.0
    vol = tr.geometry()["volume"]
    vn = (3.0 * u - 4.0 * hist[0] + hist[1]) / (2.0 * dt)
    acc = (3.0 * vn - 4.0 * hist[2] + hist[3]) / (2.0 * dt)
    expect = -rho * np.repeat(vol, 3) * acc
    diff = tr.residual(u) - st.residual(u)
    assert np.max(np.abs(diff - expect)) <= 1e-12 * np.max(np.abs(expect))


@pytest.mark.parametrize("backend", BACKENDS)
def test_jv_matches_dense_fd_jacobian(backend):
    mesh = _mesh((1.0, 1.0, 1.0), (3, 3, 3), [D, T, T, T, T, T])
    bc = np.zeros((6, 3))
    bc[1] = (1e6, 0.0, 0.0)
    be = _make(backend, mesh, _hooke(bc=bc))
    be.set_time(1.0)
    n = 3 * mesh.n_cells
    rng = np.random.default_rng(3)
    u = rng.uniform(-1e-5, 1e-5, n)
    r_u = be.residual(u)
    h = 1e-7
    J = np.empty((n, n))
    for k in range(n):  # the residual is affine (Hooke, small strain): central differences are exact up to rounding
        e = np.zeros(n)
        e[k] = h
        J[:, k] = (be.residual(u + e) - be.residual(u - e)) / (2 * h)
    v = rng.uniform(-1.0, 1.0, n)
    jv = be.jv(u, r_u, v)
    ref = J @ v
    assert np.linalg.norm(jv - ref) <= 1e-6 * np.linalg.norm(ref)
    assert np.all(be.jv(u, r_u, np.zeros(n)) == 0.0)


@pytest.mark.parametrize("backend", BACKENDS)
def test_jfnk_small_box_converges_and_zero_load(backend):
    mesh = _mesh((1.0, 1.0, 1.0), (3, 3, 3), [D, T, T, T, T, T])
    bc = np.zeros((6, 3))
    bc[1] = (1e6, 0.0, 0.0)
    cfg = solver_cfg(r_tol=1e-8, preconditioner="lu")
    be = _make(backend, mesh, _hooke(bc=bc))
    be.set_time(1.0)
    u, rep = be.jfnk(np.zeros(3 * mesh.n_cells), cfg)
    s = rep.summary()
    assert s["status"] == "converged" and 1 <= s["outer_iters"] <= 5
    assert np.linalg.norm(be.residual(u)) <= 1e-8 * s["initial_residual"] * 1.0001
    be0 = _make(backend, mesh, _hooke())
    be0.set_time(1.0)
    _, rep0 = be0.jfnk(np.zeros(3 * mesh.n_cells), cfg)
    assert rep0.summary()["outer_iters"] == 0


def _hypot_restated(x, y):
    """sfv_hypot (paper_2502_17217_b200/csrc/device.h), line for line: glibc's non-FMA hypot
    (one sqrt, then Borges' correction step), used by the host and the device Givens step."""
    import math
    ax, ay = abs(x), abs(y)
    if ax < ay:
        ax, ay = ay, ax
    if ay == 0.0:
        return ax
    h = math.sqrt(ax * ax + ay * ay)
    if h <= 2.0 * ay:
        delta = h - ay
        t1 = ax * (2.0 * delta - ax)
        t2 = (delta - 2.0 * (ax - ay)) * delta
    else:
        delta = h - ax
        t1 = 2.0 * delta * (ax - 2.0 * ay)
        t2 = (4.0 * delta - ay) * ay + delta * delta
    return h - (t1 + t2) / (2.0 * h)


def test_hypot_matches_the_reference_libm():
    """gmres_solve's Givens rotation calls std::hypot (linalg.cpp:481); the device cycle must
    get the same bits, so sfv_hypot restates the C library's algorithm.  Checked against the
    host libm on random pairs over 16 decades, including near-equal and very unequal pairs."""
    import ctypes
    libm = ctypes.CDLL("libm.so.6")
    libm.hypot.restype = ctypes.c_double
    libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]
    rng = np.random.default_rng(5)
    n = 100000
    a = rng.uniform(-1, 1, n) * 10.0 ** rng.uniform(-8, 8, n)
    b = rng.uniform(-1, 1, n) * 10.0 ** rng.uniform(-8, 8, n)
    b[: n // 3] = a[: n // 3] * rng.uniform(0.3, 3.0, n // 3)
    b[n // 3: n // 2] = a[n // 3: n // 2] * 10.0 ** rng.uniform(-9, -3, n // 2 - n // 3)
    bad = sum(libm.hypot(float(x), float(y)) != _hypot_restated(float(x), float(y)) for x, y in zip(a, b))
    assert bad == 0


def test_division_correction_is_the_division(tmp_path):
    """The U sweep (precond_stream.cu) replaces z / d by q0 = z * RN(1/d), e = fma(-q0, d, z),
    RN(q0 + e * RN(1/d)) — Markstein's correction, which returns the correctly rounded
    quotient.  Checked here against IEEE division on 2e7 random pairs over 120 binades,
    a quarter of them with divisor mantissas next to all-ones."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    src = tmp_path / "mk.c"
    src.write_text(r'''
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <math.h>
static uint64_t s = 88172645463325252ULL;
static uint64_t xr(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static double rnd(int e0, int e1) {
    uint64_t m = xr() & ((1ULL << 52) - 1);
    int e = e0 + (int)(xr() % (uint64_t)(e1 - e0));
    uint64_t b = ((uint64_t)(e + 1023) << 52) | m;
    double d;
    memcpy(&d, &b, 8);
    return (xr() & 1) ? -d : d;
}
int main(void) {
    long bad = 0;
    for (long i = 0; i < 20000000; ++i) {
        double a = rnd(-60, 60), b = rnd(-60, 60);
        if (i % 4 == 0) { uint64_t bb; memcpy(&bb, &b, 8); bb |= ((1ULL << 52) - 1) ^ (xr() & 0xff); memcpy(&b, &bb, 8); }
        double r = 1.0 / b, q0 = a * r, e = fma(-q0, b, a), q = fma(e, r, q0);
        bad += q != a / b;
    }
    printf("%ld\n", bad);
    return 0;
}
''')
    exe = tmp_path / "mk"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", str(exe), str(src), "-lm"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.strip()
    assert out == "0"
