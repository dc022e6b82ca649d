"""BASELINE.json configurations C1-C5 and the seeded synthetic inputs.

There is no public dataset on this path: every input is generated
from a seed — meshes by the reference's own generators (restated in csrc/host_mesh.cpp,
pinned bit-for-bit against the reference), fields by SplitMix64 — and the same bytes
are fed to the GPU path, the C oracle and the compiled reference.

Choices BASELINE leaves open are fixed here once (SURVEY.md findings 6-10):
  * C2 shear direction (0.5e6, 0, 0) on ymax;
  * C3 "normal displacement" as the full vector (0.3 L t, 0, 0) on xmax, mu/kappa direct;
  * C4 uses the reference's BDF2 (it has no backward Euler); v0 = 8 seeded sinusoid modes;
  * C5 is the parity-mirrored Kuhn split with even n, seeded permutation then RCM.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .abi import LAW_HOOKE, LAW_NEO_HOOKEAN, PATCH_DISPLACEMENT as D, PATCH_TRACTION as T, Mesh, Physics, solver_cfg

MASK = np.uint64(0xFFFFFFFFFFFFFFFF)


def mu_from(E, nu):  # laws.hpp:14
    return E / (2.0 * (1.0 + nu))


def lambda_from(E, nu):  # laws.hpp:15
    return E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))


def splitmix64(seed: int, idx: np.ndarray) -> np.ndarray:
    """Counter-based SplitMix64 (mesh.cpp:220-229 mixing), one draw per index."""
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)) ^ ((idx.astype(np.uint64) + np.uint64(1))
                                                                 * np.uint64(0xD1B54A32D192ED03))
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform(seed: int, n: int, lo=-1.0, hi=1.0) -> np.ndarray:
    u01 = (splitmix64(seed, np.arange(n)) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return lo + (hi - lo) * u01


def cell_centres(mesh: Mesh) -> np.ndarray:
    """Vertex-average cell centres (an input generator, not the reference centroid)."""
    nc = mesh.n_cells
    fo = mesh.face_offsets
    npts = np.diff(fo)
    fc = np.add.reduceat(mesh.points[mesh.face_points], fo[:-1], axis=0) / npts[:, None]
    acc = np.zeros((nc, 3))
    cnt = np.zeros(nc)
    np.add.at(acc, mesh.owner, fc)
    np.add.at(cnt, mesh.owner, 1)
    inner = mesh.neighbour >= 0
    np.add.at(acc, mesh.neighbour[inner], fc[inner])
    np.add.at(cnt, mesh.neighbour[inner], 1)
    return acc / cnt[:, None]


def sinusoid_field(x: np.ndarray, seed: int, amplitude: float, modes: int = 8, extent=None) -> np.ndarray:
    """sum_m a_m (.) sin(2 pi k_m . x / L + phi_m), integer k_m in [1,3]^3, scaled so
    max|f| = amplitude at the given points.  Returns interleaved (3 n,)."""
    L = np.asarray(extent if extent is not None else x.max(axis=0) - x.min(axis=0) + 1e-300)
    r = uniform(seed, modes * 10, 0.0, 1.0).reshape(modes, 10)
    f = np.zeros_like(x)
    for m in range(modes):
        k = 1 + np.floor(3 * r[m, 0:3])
        a = 2 * r[m, 3:6] - 1
        phi = 2 * np.pi * r[m, 6]
        f += a[None, :] * np.sin(2 * np.pi * (x / L) @ k + phi)[:, None]
    mag = np.sqrt((f ** 2).sum(axis=1)).max()
    return (amplitude / mag * f).reshape(-1)


def jv_inputs(mesh: Mesh, seed: int = 7, extent=None):
    """Seeded non-equilibrium u (1e-6 L smooth modes) and unit-norm v."""
    x = cell_centres(mesh)
    Lmax = float(np.max(extent)) if extent is not None else float((x.max(0) - x.min(0)).max())
    u = sinusoid_field(x, seed, 1e-6 * Lmax, extent=extent)
    v = uniform(seed + 1, 3 * mesh.n_cells)
    v /= np.linalg.norm(v)
    return u, v


@dataclass
class Case:
    name: str
    mesh_args: dict
    physics: Physics
    n_steps: int = 1
    r_tol: float = 1e-8
    kind: str = "box"  # or "tets"
    transient_v0_seed: int | None = None
    notes: str = ""
    meta: dict = field(default_factory=dict)

    def mesh(self) -> Mesh:
        from .solver import box_mesh, kuhn_tet_mesh
        if self.kind == "tets":
            return kuhn_tet_mesh(**self.mesh_args)
        return box_mesh(**self.mesh_args)

    def solver(self, **kw):
        return solver_cfg(r_tol=self.r_tol, **kw)

    def initial_field(self, mesh: Mesh) -> np.ndarray:
        """VectorField (u, u_old, u_old_old, v_old, v_old_old, a_old) at the start."""
        f = np.zeros((6, 3 * mesh.n_cells))
        if self.transient_v0_seed is not None:
            v0 = sinusoid_field(cell_centres(mesh), self.transient_v0_seed, 1.0,
                                extent=self.mesh_args.get("extents"))
            f[3] = v0
            f[4] = v0
        return f


def _bc(values: dict, n=6, ramp=True):
    bv = np.zeros((n, 3))
    for side, v in values.items():
        bv[side] = v
    return bv, np.full(n, 1 if ramp else 0, dtype=np.int32)


def config(name: str, n: int | None = None) -> Case:
    """BASELINE.json configs.  ``n`` overrides the resolution (parity tests use small n)."""
    if name == "c1":
        n = n or 20
        bv, br = _bc({1: (1e6, 0.0, 0.0)})
        ph = Physics(LAW_HOOKE, mu_from(200e9, 0.3), lambda_from(200e9, 0.3), bc_value=bv, bc_ramp=br)
        return Case("c1", dict(extents=(1.0, 1.0, 1.0), divisions=(n, n, n), kinds=[D, T, T, T, T, T]), ph,
                    notes="20^3 unit cube, xmin clamped, xmax 1 MPa normal traction, E=200GPa nu=0.3")
    if name == "c2":
        n = n or 100
        bv, br = _bc({3: (0.5e6, 0.0, 0.0)})
        ph = Physics(LAW_HOOKE, mu_from(70e9, 0.33), lambda_from(70e9, 0.33), bc_value=bv, bc_ramp=br)
        return Case("c2", dict(extents=(1.0, 1.0, 1.0), divisions=(n, n, n), kinds=[D, T, T, T, T, T],
                               distort=0.15, seed=42), ph,
                    notes="100^3 jittered 0.15 (seed 42), xmin clamped, ymax shear (0.5MPa,0,0), E=70GPa nu=0.33")
    if name == "c3":
        nx = n or 200
        ny = max(2, nx // 4)
        bv, br = _bc({1: (0.3 * 4.0, 0.0, 0.0)})
        ph = Physics(LAW_NEO_HOOKEAN, 0.4e6, 2e6, total_lagrangian=True, bc_value=bv, bc_ramp=br)
        return Case("c3", dict(extents=(4.0, 1.0, 1.0), divisions=(nx, ny, ny), kinds=[D, D, T, T, T, T],
                               distort=0.05, seed=42), ph, n_steps=10,
                    notes="200x50x50 jittered 0.05, neo-Hookean TL mu=0.4MPa kappa=2MPa, xmax u=(1.2 t,0,0), 10 increments")
    if name == "c4":
        n = n or 100
        bv, br = _bc({})
        ph = Physics(LAW_HOOKE, mu_from(200e9, 0.3), lambda_from(200e9, 0.3), transient=True, dt=1e-5, rho=7800.0,
                     bc_value=bv, bc_ramp=br)
        return Case("c4", dict(extents=(1.0, 1.0, 1.0), divisions=(n, n, n), kinds=[D, T, T, T, T, T],
                               distort=0.15, seed=42), ph, n_steps=50, transient_v0_seed=1234,
                    notes="C2 mesh, BDF2 elastodynamics rho=7800 dt=1e-5, 50 steps, v0 = 8 seeded modes (1 m/s)")
    if name == "c5":
        n = n or 160
        bv, br = _bc({1: (1e6, 0.0, 0.0)})
        ph = Physics(LAW_HOOKE, mu_from(200e9, 0.3), lambda_from(200e9, 0.3), bc_value=bv, bc_ramp=br)
        return Case("c5", dict(extents=(1.0, 1.0, 1.0), n=n, kinds=[D, T, T, T, T, T], perm_seed=42,
                               permute=True, rcm=True), ph, kind="tets",
                    notes="mirrored Kuhn tets 6 n^3, permuted (seed 42) then RCM, xmin clamped, xmax 1 MPa")
    raise KeyError(name)
