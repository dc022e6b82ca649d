"""Python mirror of the reference's hot-path interface over libsfv.so (C-ABI, include/sfv.h).

Names, argument meaning and error behaviour follow /root/reference/proj/include/solidfv:

==============================  =========================================================
reference (file:line)            here
==============================  =========================================================
ResidualEvaluator                 ``ResidualEvaluator(mesh, physics)`` (discretisation.hpp:49-91)
  .residual(u)                    ``.residual(u)`` — u, result: (3*n_cells,) interleaved
  .set_time / .set_history        same names
jacobian_vector_product           ``jacobian_vector_product(eval, u, r_u, v)`` (nonlinear.hpp:74)
make_preconditioner               ``make_preconditioner(eval, kind)`` (nonlinear.hpp:122)
Preconditioner::solve             ``Preconditioner.solve(r)`` (linalg.hpp:55-59)
gmres_solve (op = J.v at u)       ``gmres_jv(eval, u, r_u, b, ...)`` (linalg.hpp:94-97)
jfnk_solve                        ``jfnk_solve(eval, u, cfg)`` (nonlinear.hpp:96)
run_steps                         ``run_steps(eval, field, cfg, n_steps)`` (nonlinear.hpp:117)
solidfv::Error subclasses         ``SolidfvError`` with ``.kind`` / ``.cell`` (errors.hpp:8-46)
==============================  =========================================================

Vectors may be numpy arrays (host; copied to the device inside the call) or CUDA
torch tensors (device-resident, zero copy).  The CUDA extension is the only
implementation: if libsfv.so is missing or no GPU is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_SAMPLER = C.CFUNCTYPE(None, C.c_void_p, C.c_double, C.POINTER(C.c_double))

from .abi import ERR, Mesh, MeshDesc, Physics, PhysicsDesc, SolveReport, SolverCfg, dptr, iptr, solver_cfg

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SFV_LIB") or os.path.join(HERE, "libsfv.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p
_lib = None


class SolidfvError(RuntimeError):
    """One solidfv::Error subclass, named by ``kind`` (errors.hpp:8-46)."""

    def __init__(self, code: int, cell: int, msg: str):
        super().__init__(f"{ERR.get(code, code)}: {msg}" + (f" (cell {cell})" if cell >= 0 else ""))
        self.code, self.cell, self.kind = code, cell, ERR.get(code, str(code))


def lib():
    """Load libsfv.so (build it with ``python -m paper_2502_17217_b200.build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is not built: run __graft_entry__.build() or "
                           "python paper_2502_17217_b200/build.py — there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    sig = {
        "sfv_mesh_box": (_vp, [_dp, _ip, _ip, C.c_double, C.c_uint64, C.c_char_p, C.c_int]),
        "sfv_mesh_kuhn_tets": (_vp, [_dp, C.c_int, _ip, C.c_uint64, C.c_int, C.c_int, C.c_char_p, C.c_int]),
        "sfv_mesh_built_on_device": (C.c_int, [_vp]),
        "sfv_mesh_counts": (None, [_vp, _ip]),
        "sfv_mesh_export": (None, [_vp, _dp] + [_ip] * 7),
        "sfv_mesh_free": (None, [_vp]),
        "sfv_create": (_vp, [C.POINTER(MeshDesc), C.POINTER(PhysicsDesc), C.c_char_p, C.c_int]),
        "sfv_destroy": (None, [_vp]),
        "sfv_set_stream": (C.c_int, [_vp, _vp]),
        "sfv_n_cells": (C.c_int, [_vp]),
        "sfv_set_option": (C.c_int, [_vp, C.c_char_p, C.c_int]),
        "sfv_last_error": (C.c_char_p, [_vp]),
        "sfv_launch_count": (C.c_longlong, [_vp]),
        "sfv_device_bytes": (C.c_size_t, [_vp]),
        "sfv_jv_bytes": (C.c_double, [_vp]),
        "sfv_geometry": (C.c_int, [_vp] + [_dp] * 9 + [C.POINTER(C.c_byte), _ip, _ip, _dp]),
        "sfv_set_time": (C.c_int, [_vp, C.c_double]),
        "sfv_set_body_force": (C.c_int, [_vp, _dp]),
        "sfv_set_boundary_values": (C.c_int, [_vp, _dp]),
        "sfv_set_boundary_sampler": (C.c_int, [_vp, _vp, _vp]),
        "sfv_set_history": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
        "sfv_residual": (C.c_int, [_vp, _vp, _vp, _ip]),
        "sfv_stabilisation": (C.c_int, [_vp, _vp, _vp, _ip]),
        "sfv_gradients": (C.c_int, [_vp, _vp, _vp, _ip]),
        "sfv_commit": (C.c_int, [_vp, _vp]),
        "sfv_law_state": (C.c_int, [_vp, _vp]),
        "sfv_jv": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _ip]),
        "sfv_jv_eps": (C.c_int, [_vp, _vp, _vp, _vp, C.c_double, _vp, _ip]),
        "sfv_jv_async": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
        "sfv_check_errors": (C.c_int, [_vp, _ip]),
        "sfv_jv_stage_times": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_int, _dp]),
        "sfv_jv_stage_bytes": (None, [_vp, _dp]),
        "sfv_residual_host": (C.c_int, [_vp, _dp, _dp, _ip]),
        "sfv_jv_host": (C.c_int, [_vp, _dp, _dp, _dp, _dp, _ip]),
        "sfv_precond_create": (C.c_int, [_vp, C.c_int]),
        "sfv_approximate_jacobian": (C.c_int, [_vp, _ip, _ip, _dp]),
        "sfv_line_search": (C.c_int, [_vp, _vp, _vp, C.c_double, _ip, _dp, _dp, _vp]),
        "sfv_precond_apply": (C.c_int, [_vp, _vp, _vp]),
        "sfv_precond_info": (C.c_int, [_vp, _ip]),
        "sfv_precond_sweep": (C.c_int, [_vp]),
        "sfv_gmres_jv": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_int, C.c_double, C.c_int, C.c_int, _ip, _ip, _dp]),
        "sfv_jfnk_solve": (C.c_int, [_vp, _vp, C.POINTER(SolverCfg), C.POINTER(SolveReport)]),
        "sfv_run_steps": (C.c_int, [_vp, _vp, C.POINTER(SolverCfg), C.c_int, C.POINTER(SolveReport), C.c_int,
                                    _ip, _dp]),
        "sfv_run_steps_host": (C.c_int, [_vp, _dp, C.POINTER(SolverCfg), C.c_int, C.POINTER(SolveReport),
                                         C.c_int, _ip, _dp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


# ------------------------------------------------------------------ meshes

def _export_mesh(h) -> Mesh:
    L = lib()
    cnt = np.zeros(6, dtype=np.int32)
    L.sfv_mesh_counts(h, iptr(cnt))
    npnt, nf, nfp, nc, nint, npatch = (int(x) for x in cnt)
    pts = np.zeros(3 * npnt)
    fo = np.zeros(nf + 1, dtype=np.int32)
    fp = np.zeros(nfp, dtype=np.int32)
    own = np.zeros(nf, dtype=np.int32)
    nei = np.zeros(nf, dtype=np.int32)
    pk, ps, pc = (np.zeros(npatch, dtype=np.int32) for _ in range(3))
    L.sfv_mesh_export(h, dptr(pts), iptr(fo), iptr(fp), iptr(own), iptr(nei), iptr(pk), iptr(ps), iptr(pc))
    L.sfv_mesh_free(h)
    return Mesh(pts.reshape(-1, 3), fo, fp, own, nei, nc, nint, pk, ps, pc)


def box_mesh(extents, divisions, kinds, distort: float = 0.0, seed: int = 0) -> Mesh:
    """generate_box_hex + distort_mesh (mesh.cpp:76, :290) on the host; kinds per
    (xmin, xmax, ymin, ymax, zmin, zmax)."""
    e = np.ascontiguousarray(extents, dtype=np.float64)
    d = np.ascontiguousarray(divisions, dtype=np.int32)
    k = np.ascontiguousarray(kinds, dtype=np.int32)
    err = C.create_string_buffer(256)
    h = lib().sfv_mesh_box(dptr(e), iptr(d), iptr(k), float(distort), C.c_uint64(seed), err, 256)
    if not h:
        raise SolidfvError(1, -1, err.value.decode())
    return _export_mesh(h)


def kuhn_tet_mesh(extents, n: int, kinds, perm_seed: int = 0, permute: bool = True, rcm: bool = True) -> Mesh:
    """Config-5 generator: parity-mirrored Kuhn split (6 tets per hex, n even),
    seeded random cell permutation, then reverse Cuthill-McKee renumbering."""
    e = np.ascontiguousarray(extents, dtype=np.float64)
    k = np.ascontiguousarray(kinds, dtype=np.int32)
    err = C.create_string_buffer(256)
    h = lib().sfv_mesh_kuhn_tets(dptr(e), int(n), iptr(k), C.c_uint64(perm_seed), int(permute), int(rcm), err, 256)
    if not h:
        raise SolidfvError(1, -1, err.value.decode())
    on_dev = bool(lib().sfv_mesh_built_on_device(h))
    m = _export_mesh(h)
    m.on_device = on_dev
    return m


# ------------------------------------------------------------------ device arrays

def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2502_17217_b200 needs a CUDA device (B200); there is no CPU fallback")
    return torch


def to_device(a):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1)).to("cuda")


def _ptr(t) -> int:
    return t.data_ptr()


# ------------------------------------------------------------------ evaluator

class ResidualEvaluator:
    """R(u) on the B200 (ResidualEvaluator, discretisation.hpp:49-91)."""

    def __init__(self, mesh: Mesh, physics: Physics):
        self.L = lib()
        _torch()
        self.mesh, self.physics = mesh, physics
        md, pd = mesh.desc(), physics.desc()
        err = C.create_string_buffer(512)
        self.h = self.L.sfv_create(C.byref(md), C.byref(pd), err, 512)
        if not self.h:
            raise SolidfvError(1, -1, err.value.decode())
        self.n_cells = int(self.L.sfv_n_cells(self.h))
        self.n = 3 * self.n_cells
        self._hist = None
        self.set_stream_current()

    def __del__(self):
        if getattr(self, "h", None):
            self.L.sfv_destroy(self.h)
            self.h = None

    # -- plumbing
    def set_stream_current(self):
        torch = _torch()
        self.L.sfv_set_stream(self.h, C.c_void_p(torch.cuda.current_stream().cuda_stream))

    def _check(self, rc: int, cell: int = -1):
        if rc:
            raise SolidfvError(rc, cell, self.L.sfv_last_error(self.h).decode(errors="replace"))

    @property
    def launch_count(self) -> int:
        return int(self.L.sfv_launch_count(self.h))

    @property
    def jv_bytes(self) -> float:
        """Compulsory HBM bytes of one J.v."""
        return float(self.L.sfv_jv_bytes(self.h))

    @property
    def kbar(self) -> float:
        return self.physics.kbar

    def empty(self):
        return _torch().zeros(self.n, dtype=_torch().float64, device="cuda")

    # -- reference API
    def set_option(self, name: str, value: int):
        """Execution switches (sfv_set_option): "gmres_graph" 1/0, "sequential_reductions" 0/1."""
        self._check(self.L.sfv_set_option(self.h, name.encode(), int(value)))

    def set_time(self, t: float):
        self._check(self.L.sfv_set_time(self.h, float(t)))

    def set_body_force(self, f):
        """DiscretisationConfig::body_force sampled at the cell centroids: (3*n_cells,) or None."""
        if f is None:
            self._check(self.L.sfv_set_body_force(self.h, None))
            return
        self._body = np.ascontiguousarray(f, dtype=np.float64).reshape(-1)
        self._check(self.L.sfv_set_body_force(self.h, dptr(self._body)))

    def set_boundary_values(self, values):
        """Per boundary face BC values (3*(n_faces - n_internal),) at the current time, or None."""
        if values is None:
            self._check(self.L.sfv_set_boundary_values(self.h, None))
            return
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        self._check(self.L.sfv_set_boundary_values(self.h, dptr(v)))

    def set_boundary_sampler(self, fn):
        """fn(t) -> (3*(n_faces - n_internal),) per-face BC values; sampled on every set_time and
        every step of run_steps (BoundaryCondition::value at the face centroids).  None clears."""
        if fn is None:
            self._sampler = None
            self._check(self.L.sfv_set_boundary_sampler(self.h, None, None))
            return
        nb = 3 * (self.mesh.n_faces - self.mesh.n_internal)

        def cb(_user, t, out):
            vals = np.ascontiguousarray(fn(t), dtype=np.float64).reshape(-1)
            C.memmove(out, vals.ctypes.data, 8 * nb)

        self._sampler = _SAMPLER(cb)
        self._check(self.L.sfv_set_boundary_sampler(self.h, C.cast(self._sampler, _vp), None))

    def set_history(self, u_old, u_old_old, v_old, v_old_old):
        self._hist = [to_device(a) for a in (u_old, u_old_old, v_old, v_old_old)]
        self._check(self.L.sfv_set_history(self.h, *[_ptr(t) for t in self._hist]))

    def residual(self, u):
        ud = to_device(u)
        r = self.empty()
        cell = C.c_int(-1)
        self._check(self.L.sfv_residual(self.h, _ptr(ud), _ptr(r), C.byref(cell)), cell.value)
        return r

    def stabilisation(self, u):
        """ResidualEvaluator::stabilisation (discretisation.cpp:210-214): the Rhie-Chow sum alone."""
        ud = to_device(u)
        r = self.empty()
        cell = C.c_int(-1)
        self._check(self.L.sfv_stabilisation(self.h, _ptr(ud), _ptr(r), C.byref(cell)), cell.value)
        return r

    def commit(self, u):
        """ResidualEvaluator::commit (discretisation.cpp:91-95): J2's trial state at u becomes the
        committed state (a no-op for the hyperelastic laws)."""
        ud = to_device(u)
        self._check(self.L.sfv_commit(self.h, _ptr(ud)))

    def law_state(self):
        """Committed J2 state, (n_cells, 19): b_bar (row-major), eps_p, F (PlasticCell)."""
        out = np.zeros(19 * self.mesh.n_cells)
        self._check(self.L.sfv_law_state(self.h, out.ctypes.data))
        return out.reshape(-1, 19)

    def gradients(self, u):
        """cell_gradients (discretisation.cpp:10-31) as an (n_cells, 3, 3) array, G[c, i, j] = du_j/dx_i."""
        ud = to_device(u)
        G = _torch().empty(9 * self.mesh.n_cells, dtype=_torch().float64, device="cuda")
        cell = C.c_int(-1)
        self._check(self.L.sfv_gradients(self.h, _ptr(ud), _ptr(G), C.byref(cell)), cell.value)
        return G.reshape(9, self.mesh.n_cells).T.reshape(-1, 3, 3)

    def geometry(self) -> dict:
        m = self.mesh
        nc, nf = m.n_cells, m.n_faces
        nslots = int(2 * m.n_internal + (nf - m.n_internal))
        g = {k: np.zeros(s) for k, s in (("volume", nc), ("centroid", 3 * nc), ("face_centroid", 3 * nf),
                                          ("area", 3 * nf), ("d", 3 * nf), ("d_mag", nf), ("w", nf),
                                          ("delta", 3 * nf), ("g_inv", 9 * nc))}
        sing = np.zeros(nc, dtype=np.int8)
        cfo = np.zeros(nc + 1, dtype=np.int32)
        cff = np.zeros(nslots, dtype=np.int32)
        ls = np.zeros(3 * nslots)
        self.L.sfv_geometry(self.h, *[dptr(g[k]) for k in ("volume", "centroid", "face_centroid", "area", "d",
                                                           "d_mag", "w", "delta", "g_inv")],
                            sing.ctypes.data_as(C.POINTER(C.c_byte)), iptr(cfo), iptr(cff), dptr(ls))
        g.update(g_singular=sing, cf_offsets=cfo, cf_faces=cff, ls_vec=ls)
        return g


def jacobian_vector_product(ev: ResidualEvaluator, u, r_u, v, eps: float | None = None):
    """(R(u + eps v) - R(u)) / eps, eps = sqrt(DBL_EPSILON) sqrt(1+|u|)/|v| (nonlinear.cpp:105-138).
    ``eps`` overrides the step (parity harness only)."""
    ud, rd, vd = to_device(u), to_device(r_u), to_device(v)
    out = ev.empty()
    cell = C.c_int(-1)
    if eps is None:
        rc = ev.L.sfv_jv(ev.h, _ptr(ud), _ptr(rd), _ptr(vd), _ptr(out), C.byref(cell))
    else:
        rc = ev.L.sfv_jv_eps(ev.h, _ptr(ud), _ptr(rd), _ptr(vd), float(eps), _ptr(out), C.byref(cell))
    ev._check(rc, cell.value)
    return out


class Preconditioner:
    """The reference's preconditioner action on the device (linalg.hpp:55-59)."""

    def __init__(self, ev: ResidualEvaluator, kind: str):
        self.ev = ev
        self.kind = kind

    def solve(self, r):
        rd = to_device(r)
        z = self.ev.empty()
        self.ev._check(self.ev.L.sfv_precond_apply(self.ev.h, _ptr(rd), _ptr(z)))
        return z

    def info(self) -> dict:
        i = np.zeros(5, dtype=np.int32)
        self.ev.L.sfv_precond_info(self.ev.h, iptr(i))
        return {"kind": int(i[0]), "levels_fwd": int(i[1]), "levels_bwd": int(i[2]), "nnz_L": int(i[3]),
                "nnz_U": int(i[4]), "sweep": int(self.ev.L.sfv_precond_sweep(self.ev.h))}


def make_preconditioner(ev: ResidualEvaluator, kind: str = "auto") -> Preconditioner:
    """assemble_approximate_jacobian + make_preconditioner (nonlinear.cpp:353-380):
    automatic = LU when 3*n_cells <= 30000, else ILU(1)."""
    from .abi import PRECOND
    ev._check(ev.L.sfv_precond_create(ev.h, PRECOND[kind]))
    return Preconditioner(ev, kind)


def approximate_jacobian(ev: ResidualEvaluator):
    """assemble_approximate_jacobian (discretisation.cpp:216-262): (row_ptr, col, blocks[nnz, 3, 3])."""
    nnz = ev.L.sfv_approximate_jacobian(ev.h, None, None, None)
    if nnz < 0:
        ev._check(nnz)
    rp = np.zeros(ev.n_cells + 1, dtype=np.int32)
    col = np.zeros(nnz, dtype=np.int32)
    blocks = np.zeros(9 * nnz)
    r = ev.L.sfv_approximate_jacobian(ev.h, iptr(rp), iptr(col), dptr(blocks))
    if r < 0:
        ev._check(r)
    return rp, col, blocks.reshape(nnz, 3, 3)


def line_search(ev: ResidualEvaluator, u, du, r_norm0: float):
    """line_search (nonlinear.cpp:140-163): (success, s, r_norm, residual or None)."""
    ud, dd = to_device(u), to_device(du)
    res = ev.empty()
    ok, s, rn = C.c_int(0), C.c_double(0.0), C.c_double(0.0)
    ev._check(ev.L.sfv_line_search(ev.h, _ptr(ud), _ptr(dd), float(r_norm0), C.byref(ok), C.byref(s), C.byref(rn),
                                   _ptr(res)))
    return bool(ok.value), s.value, rn.value, (res if ok.value else None)


def gmres_jv(ev: ResidualEvaluator, u, r_u, b, x0=None, restart=30, rel_reduction=1e-3, max_iters=300,
             right_preconditioned=False):
    """gmres_solve (linalg.cpp:423-538) with op = J.v at u and the context's preconditioner,
    left (default) or right preconditioned."""
    ud, rd, bd = to_device(u), to_device(r_u), to_device(b)
    x = ev.empty() if x0 is None else to_device(x0).clone()
    it, st, rel = C.c_int(0), C.c_int(0), C.c_double(0.0)
    ev._check(ev.L.sfv_gmres_jv(ev.h, _ptr(ud), _ptr(rd), _ptr(bd), _ptr(x), int(restart), float(rel_reduction),
                                int(max_iters), int(bool(right_preconditioned)), C.byref(it), C.byref(st),
                                C.byref(rel)))
    return x, it.value, ["converged", "max-iters", "stagnated"][st.value], rel.value


def jfnk_solve(ev: ResidualEvaluator, u, cfg: SolverCfg | None = None):
    """jfnk_solve (nonlinear.cpp:173-266) fully device-resident; returns (u, SolveReport)."""
    cfg = cfg or solver_cfg()
    ud = to_device(u).clone()
    rep = SolveReport()
    ev._check(ev.L.sfv_jfnk_solve(ev.h, _ptr(ud), C.byref(cfg), C.byref(rep)))
    return ud, rep


def run_steps(ev: ResidualEvaluator, field, cfg: SolverCfg | None = None, n_steps: int = 1):
    """run_steps (nonlinear.cpp:382-446).  field: (6, 3*n_cells) = u, u_old, u_old_old,
    v_old, v_old_old, a_old (VectorField).  Returns (field, [SolveReport], wall_seconds)."""
    cfg = cfg or solver_cfg()
    torch = _torch()
    if isinstance(field, torch.Tensor):
        fd = field.to(device="cuda", dtype=torch.float64).contiguous().clone()
    else:
        fd = torch.from_numpy(np.ascontiguousarray(field, dtype=np.float64)).to("cuda")
    fd = fd.reshape(6, ev.n).contiguous()
    reps = (SolveReport * max(n_steps, 1))()
    nrep, wall = C.c_int(0), C.c_double(0.0)
    ev._check(ev.L.sfv_run_steps(ev.h, _ptr(fd), C.byref(cfg), int(n_steps), reps, max(n_steps, 1), C.byref(nrep),
                                 C.byref(wall)))
    return fd, [reps[i] for i in range(nrep.value)], wall.value


def run_steps_host(ev: ResidualEvaluator, field: np.ndarray, cfg: SolverCfg | None = None, n_steps: int = 1):
    """run_steps through the C-ABI with host buffers (copies inside the call)."""
    cfg = cfg or solver_cfg()
    f = np.ascontiguousarray(field, dtype=np.float64).reshape(-1).copy()
    reps = (SolveReport * max(n_steps, 1))()
    nrep, wall = C.c_int(0), C.c_double(0.0)
    ev._check(ev.L.sfv_run_steps_host(ev.h, dptr(f), C.byref(cfg), int(n_steps), reps, max(n_steps, 1),
                                      C.byref(nrep), C.byref(wall)))
    return f.reshape(6, -1), [reps[i] for i in range(nrep.value)], wall.value
