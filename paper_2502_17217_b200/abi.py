"""ctypes mirrors of include/sfv_case.h — the input/report structs shared by the
product C-ABI (include/sfv.h), the CPU oracle and the reference driver.

Field meanings follow the reference types they restate (see the header):
``MeshDesc`` <- solidfv::Mesh (mesh.hpp:30-49), ``Physics`` <- law +
DiscretisationConfig + config-built BCs (io.cpp:276-279), ``SolverCfg`` <-
SolverConfig (nonlinear.hpp:27-44), ``SolveReport`` <- SolveReport
(nonlinear.hpp:54-65).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

PATCH_DISPLACEMENT, PATCH_TRACTION, PATCH_SYMMETRY = 0, 1, 2
LAW_HOOKE, LAW_NEO_HOOKEAN, LAW_STVK, LAW_GUCCIONE, LAW_J2 = 0, 1, 2, 3, 4
PRECOND = {"auto": 0, "none": 1, "ilu0": 2, "ilu1": 3, "ilu2": 4, "lu": 5}
CONVERGED, DIVERGED, MAX_ITERS = 0, 1, 2
STATUS_NAME = {CONVERGED: "converged", DIVERGED: "diverged", MAX_ITERS: "max-iters"}

ERR = {
    0: "ok",
    1: "InvalidArgument",
    2: "GeometryFailure",
    3: "GradientFailure",
    4: "InvertedElement",
    5: "LawOverflow",
    12: "ReturnMapFailure",
    6: "ResidualNan",
    7: "JvpNan",
    8: "IluBreakdown",
    9: "LuSingular",
    10: "CudaError",
    11: "InternalError",
}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class MeshDesc(C.Structure):
    _fields_ = [
        ("dim", C.c_int),
        ("n_points", C.c_int),
        ("points", _dp),
        ("n_faces", C.c_int),
        ("face_offsets", _ip),
        ("face_points", _ip),
        ("owner", _ip),
        ("neighbour", _ip),
        ("n_cells", C.c_int),
        ("n_internal", C.c_int),
        ("n_patches", C.c_int),
        ("patch_kind", _ip),
        ("patch_start", _ip),
        ("patch_count", _ip),
    ]


class PhysicsDesc(C.Structure):
    _fields_ = [
        ("law", C.c_int),
        ("mu", C.c_double),
        ("lam", C.c_double),
        ("alpha", C.c_double),
        ("total_lagrangian", C.c_int),
        ("transient", C.c_int),
        ("dt", C.c_double),
        ("rho", C.c_double),
        ("bc_value", _dp),
        ("bc_ramp", _ip),
        ("guccione", C.c_double * 8),
        ("j2_curve", C.c_double * 4),
        ("j2_n_table", C.c_int),
        ("j2_table", _dp),
    ]


class SolverCfg(C.Structure):
    _fields_ = [
        ("a_tol", C.c_double),
        ("r_tol", C.c_double),
        ("s_tol", C.c_double),
        ("max_outer", C.c_int),
        ("inner_reduction", C.c_double),
        ("restart", C.c_int),
        ("max_krylov", C.c_int),
        ("preconditioner", C.c_int),
        ("line_search", C.c_int),
        ("algorithm", C.c_int),
        ("relaxation", C.c_double),
        ("right_preconditioned", C.c_int),
    ]


class IterationRecord(C.Structure):
    _fields_ = [
        ("step", C.c_int),
        ("iter", C.c_int),
        ("r_norm", C.c_double),
        ("krylov_iters", C.c_int),
        ("s", C.c_double),
    ]


class SolveReport(C.Structure):
    _fields_ = [
        ("status", C.c_int),
        ("step", C.c_int),
        ("outer_iters", C.c_int),
        ("krylov_iters", C.c_int),
        ("initial_residual", C.c_double),
        ("final_residual", C.c_double),
        ("wall_seconds", C.c_double),
        ("n_records", C.c_int),
        ("records", IterationRecord * 64),
        ("detail", C.c_char * 160),
        ("cg_diag_fallback", C.c_int),
        ("all_records", C.POINTER(IterationRecord)),
        ("all_capacity", C.c_int),
    ]

    def attach_history(self, capacity: int = 4096):
        """Unbounded SolveReport::iterations (nonlinear.hpp:64): the solver writes every
        record into a caller buffer as well as the first 64 into records[]."""
        self._hist = (IterationRecord * capacity)()
        self.all_records = C.cast(self._hist, C.POINTER(IterationRecord))
        self.all_capacity = capacity
        return self

    def record_list(self) -> list:
        if self.all_records and self.all_capacity:
            return [self.all_records[i] for i in range(min(self.n_records, self.all_capacity))]
        return [self.records[i] for i in range(min(self.n_records, 64))]

    def summary(self) -> dict:
        recs = self.record_list()
        n = len(recs)
        return {
            "status": STATUS_NAME.get(self.status, str(self.status)),
            "step": self.step,
            "outer_iters": self.outer_iters,
            "krylov_iters": self.krylov_iters,
            "initial_residual": self.initial_residual,
            "final_residual": self.final_residual,
            "wall_seconds": self.wall_seconds,
            "krylov_per_newton": [recs[i].krylov_iters for i in range(1, n)],
            "r_norms": [recs[i].r_norm for i in range(n)],
            "s": [recs[i].s for i in range(1, n)],
            "cg_diag_fallback": bool(self.cg_diag_fallback),
            "detail": self.detail.decode(errors="replace"),
        }


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def iptr(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_ip)


@dataclass
class Mesh:
    """Face-addressed mesh as flat arrays (the solidfv::Mesh layout, mesh.hpp:30-49)."""

    points: np.ndarray  # (n_points, 3) float64
    face_offsets: np.ndarray  # (n_faces+1,) int32
    face_points: np.ndarray  # int32
    owner: np.ndarray  # int32
    neighbour: np.ndarray  # int32, -1 on boundary
    n_cells: int
    n_internal: int
    patch_kind: np.ndarray  # int32
    patch_start: np.ndarray
    patch_count: np.ndarray
    _keep: list = field(default_factory=list, repr=False)
    on_device: bool = False  # built by a device generator (sfv_mesh_built_on_device)

    @property
    def n_faces(self) -> int:
        return int(self.owner.shape[0])

    def desc(self) -> MeshDesc:
        arrs = [
            np.ascontiguousarray(self.points, dtype=np.float64).reshape(-1),
            np.ascontiguousarray(self.face_offsets, dtype=np.int32),
            np.ascontiguousarray(self.face_points, dtype=np.int32),
            np.ascontiguousarray(self.owner, dtype=np.int32),
            np.ascontiguousarray(self.neighbour, dtype=np.int32),
            np.ascontiguousarray(self.patch_kind, dtype=np.int32),
            np.ascontiguousarray(self.patch_start, dtype=np.int32),
            np.ascontiguousarray(self.patch_count, dtype=np.int32),
        ]
        self._keep = arrs
        d = MeshDesc()
        d.dim = 3
        d.n_points = int(arrs[0].shape[0] // 3)
        d.points = dptr(arrs[0])
        d.n_faces = int(arrs[3].shape[0])
        d.face_offsets = iptr(arrs[1])
        d.face_points = iptr(arrs[2])
        d.owner = iptr(arrs[3])
        d.neighbour = iptr(arrs[4])
        d.n_cells = int(self.n_cells)
        d.n_internal = int(self.n_internal)
        d.n_patches = int(arrs[5].shape[0])
        d.patch_kind = iptr(arrs[5])
        d.patch_start = iptr(arrs[6])
        d.patch_count = iptr(arrs[7])
        return d


@dataclass
class Physics:
    """Law + discretisation + per-patch BC values (value * t when ramped)."""

    law: int = LAW_HOOKE
    mu: float = 0.0
    lam: float = 0.0  # Hooke lambda, or neo-Hookean kappa
    alpha: float = 1.0
    total_lagrangian: bool = False
    transient: bool = False
    dt: float = 0.0
    rho: float = 0.0
    bc_value: np.ndarray = None  # (n_patches, 3)
    bc_ramp: np.ndarray = None  # (n_patches,)
    # GuccioneParams (laws.hpp:38-43): C, c_f, c_t, c_fs, kappa, f0 (3)
    guccione: tuple = (0.0, 0.0, 0.0, 0.0, 0.0, 1.0, 0.0, 0.0)
    # J2 HardeningCurve (laws.hpp:52-64): saturation (a, b, c, d), or a table of (eps_p, sigma_y)
    j2_curve: tuple = (0.0, 0.0, 0.0, 1.0)
    j2_table: np.ndarray = None
    _keep: list = field(default_factory=list, repr=False)

    def desc(self) -> PhysicsDesc:
        bv = np.ascontiguousarray(self.bc_value, dtype=np.float64).reshape(-1)
        br = np.ascontiguousarray(self.bc_ramp, dtype=np.int32)
        tab = np.ascontiguousarray(self.j2_table if self.j2_table is not None else np.zeros((0, 2)),
                                   dtype=np.float64).reshape(-1)
        self._keep = [bv, br, tab]
        p = PhysicsDesc()
        p.law = int(self.law)
        p.mu = float(self.mu)
        p.lam = float(self.lam)
        p.alpha = float(self.alpha)
        p.total_lagrangian = int(bool(self.total_lagrangian))
        p.transient = int(bool(self.transient))
        p.dt = float(self.dt)
        p.rho = float(self.rho)
        p.bc_value = dptr(bv)
        p.bc_ramp = iptr(br)
        for k, x in enumerate(self.guccione):
            p.guccione[k] = float(x)
        for k, x in enumerate(self.j2_curve):
            p.j2_curve[k] = float(x)
        p.j2_n_table = len(tab) // 2
        p.j2_table = dptr(tab) if len(tab) else None
        return p

    @property
    def kbar(self) -> float:
        """law.stabilisation_modulus() (laws.hpp:100, :111, :122, :133)."""
        if self.law in (LAW_NEO_HOOKEAN, LAW_J2):
            return 4.0 / 3.0 * self.mu + self.lam
        if self.law == LAW_GUCCIONE:
            g = self.guccione
            return 4.0 / 3.0 * (g[0] * g[2]) + g[4]
        return 2.0 * self.mu + self.lam


def solver_cfg(r_tol=1e-6, a_tol=1e-50, s_tol=0.0, max_outer=0, inner_reduction=0.0, restart=30,
               max_krylov=300, preconditioner="auto", line_search=True, algorithm="jfnk",
               relaxation=1.0, right_preconditioned=False) -> SolverCfg:
    """SolverConfig defaults (nonlinear.hpp:27-44); algorithm "jfnk" or "segregated"."""
    c = SolverCfg()
    c.algorithm = {"jfnk": 0, "segregated": 1}[algorithm] if isinstance(algorithm, str) else int(algorithm)
    c.relaxation = float(relaxation)
    c.a_tol, c.r_tol, c.s_tol = a_tol, r_tol, s_tol
    c.max_outer, c.inner_reduction = max_outer, inner_reduction
    c.restart, c.max_krylov = restart, max_krylov
    c.preconditioner = PRECOND[preconditioner] if isinstance(preconditioner, str) else int(preconditioner)
    c.line_search = int(bool(line_search))
    c.right_preconditioned = int(bool(right_preconditioned))
    return c
