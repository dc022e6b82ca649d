"""ctypes bindings for the two CPU checkers.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py (cpu_baseline / --impl reference legs) — never by the product package.

* ``OracleCase``  -> oracle/liboracle.so  (plain-C restatement, sfv_oracle.c)
* ``RefCase``     -> oracle/_ref/libsolidfv_ref.so (the reference's own sources,
  compiled where they lie under /root/reference/proj/src by oracle/Makefile;
  present in this container and shipped to the GPU box with gpurun snapshots)
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2502_17217_b200.abi import (ERR, Mesh, MeshDesc, Physics, PhysicsDesc, SolveReport,
                                       SolverCfg, dptr, iptr)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsolidfv_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_libs: dict = {}


class CpuError(RuntimeError):
    def __init__(self, code: int, cell: int, msg: str):
        super().__init__(f"{ERR.get(code, code)}(cell={cell}): {msg}")
        self.code, self.cell, self.kind = code, cell, ERR.get(code, str(code))


def _load(path: str, prefix: str):
    if path in _libs:
        return _libs[path]
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
    lib = C.CDLL(path)
    p = prefix
    f = getattr(lib, p + "create")
    f.restype = C.c_void_p
    f.argtypes = [C.POINTER(MeshDesc), C.POINTER(PhysicsDesc), C.c_char_p, C.c_int]
    getattr(lib, p + "destroy").argtypes = [C.c_void_p]
    getattr(lib, p + "last_error").restype = C.c_char_p
    getattr(lib, p + "last_error").argtypes = [C.c_void_p]
    getattr(lib, p + "geometry").argtypes = [C.c_void_p] + [_dp] * 9 + [C.POINTER(C.c_byte), _ip, _ip, _dp]
    getattr(lib, p + "set_time").argtypes = [C.c_void_p, C.c_double]
    getattr(lib, p + "set_history").argtypes = [C.c_void_p, _dp, _dp, _dp, _dp]
    for name in ("residual", "stabilisation"):
        getattr(lib, p + name).argtypes = [C.c_void_p, _dp, _dp, _ip]
    if prefix == "ref_":
        lib.ref_commit.argtypes = [C.c_void_p, _dp, _ip]
    else:
        lib.orc_commit.argtypes = [C.c_void_p, _dp]
        lib.orc_law_state.argtypes = [C.c_void_p, _dp]
    getattr(lib, p + "set_body_force").argtypes = [C.c_void_p, _dp]
    getattr(lib, p + "set_face_bc").argtypes = [C.c_void_p, _dp]
    getattr(lib, p + "jv").argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _ip]
    getattr(lib, p + "precond_create").argtypes = [C.c_void_p, C.c_int]
    getattr(lib, p + "precond_apply").argtypes = [C.c_void_p, _dp, _dp]
    getattr(lib, p + "jfnk_solve").argtypes = [C.c_void_p, _dp, C.POINTER(SolverCfg), C.POINTER(SolveReport)]
    getattr(lib, p + "run_steps").argtypes = [C.c_void_p, _dp, C.POINTER(SolverCfg), C.c_int,
                                              C.POINTER(SolveReport), C.c_int, _ip, _dp]
    if prefix == "ref_":
        lib.ref_time_jv.restype = C.c_double
        lib.ref_time_jv.argtypes = [C.c_void_p, _dp, _dp, _dp, C.c_int, C.c_int]
        lib.ref_box_mesh.restype = C.c_void_p
        lib.ref_box_mesh.argtypes = [C.c_double] * 3 + [C.c_int] * 3 + [_ip, C.c_double, C.c_uint64]
        lib.ref_mesh_counts.argtypes = [C.c_void_p, _ip]
        lib.ref_mesh_export.argtypes = [C.c_void_p, _dp] + [_ip] * 7
        lib.ref_mesh_free.argtypes = [C.c_void_p]
        lib.ref_jacobian_nnz.argtypes = [C.c_void_p]
        lib.ref_jacobian.argtypes = [C.c_void_p, _ip, _ip, _dp]
    else:
        lib.orc_time_jv.restype = C.c_double
        lib.orc_time_jv.argtypes = [C.c_void_p, _dp, _dp, _dp, C.c_int]
        lib.orc_gmres_jv.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, C.c_int, C.c_double, C.c_int, C.c_int,
                                     _ip, _ip, _dp]
    _libs[path] = lib
    return lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class _CpuCase:
    PREFIX = ""
    PATH = ""

    def __init__(self, mesh: Mesh, phys: Physics):
        self.lib = _load(self.PATH, self.PREFIX)
        self.mesh, self.phys = mesh, phys
        self.n_cells = mesh.n_cells
        md, pd = mesh.desc(), phys.desc()
        err = C.create_string_buffer(256)
        self.h = self._f("create")(C.byref(md), C.byref(pd), err, 256)
        if not self.h:
            raise CpuError(1, -1, err.value.decode())

    def _f(self, name):
        return getattr(self.lib, self.PREFIX + name)

    def __del__(self):
        if getattr(self, "h", None):
            self._f("destroy")(self.h)
            self.h = None

    def _check(self, rc, cell=-1):
        if rc:
            raise CpuError(rc, cell, self._f("last_error")(self.h).decode(errors="replace"))

    def vec(self):
        return np.zeros(3 * self.n_cells)

    def set_time(self, t: float):
        self._f("set_time")(self.h, float(t))

    def set_history(self, u_old, u_old_old, v_old, v_old_old):
        arrs = [np.ascontiguousarray(a, dtype=np.float64).reshape(-1) for a in (u_old, u_old_old, v_old, v_old_old)]
        self._f("set_history")(self.h, *[dptr(a) for a in arrs])

    def set_body_force(self, f):
        """DiscretisationConfig::body_force sampled at the cell centroids (3 nc) or None."""
        arr = None if f is None else np.ascontiguousarray(f, dtype=np.float64).reshape(-1)
        self._check(self._f("set_body_force")(self.h, None if arr is None else dptr(arr)))

    def set_face_bc(self, v):
        """Per boundary face BC values at the current time (3 (nf - nint))."""
        arr = np.ascontiguousarray(v, dtype=np.float64).reshape(-1)
        self._check(self._f("set_face_bc")(self.h, dptr(arr)))

    def residual(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
        r = self.vec()
        cell = C.c_int(-1)
        rc = self._f("residual")(self.h, dptr(u), dptr(r), C.byref(cell))
        self._check(rc, cell.value)
        return r

    def commit(self, u):
        """ResidualEvaluator::commit (discretisation.cpp:91-95): J2's trial state becomes committed."""
        u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
        cell = C.c_int(-1)
        if self.PREFIX == "ref_":
            rc = self.lib.ref_commit(self.h, dptr(u), C.byref(cell))
        else:
            rc = self.lib.orc_commit(self.h, dptr(u))
        self._check(rc, cell.value)

    def law_state(self):
        """Committed J2 state (oracle only): (n_cells, 19) = b_bar, eps_p, F."""
        out = np.zeros(19 * self.n_cells)
        self._check(self.lib.orc_law_state(self.h, dptr(out)))
        return out.reshape(-1, 19)

    def stabilisation(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
        r = self.vec()
        cell = C.c_int(-1)
        rc = self._f("stabilisation")(self.h, dptr(u), dptr(r), C.byref(cell))
        self._check(rc, cell.value)
        return r

    def jv(self, u, r_u, v):
        u, r_u, v = (np.ascontiguousarray(a, dtype=np.float64).reshape(-1) for a in (u, r_u, v))
        out = self.vec()
        cell = C.c_int(-1)
        rc = self._f("jv")(self.h, dptr(u), dptr(r_u), dptr(v), dptr(out), C.byref(cell))
        self._check(rc, cell.value)
        return out

    def geometry(self) -> dict:
        m = self.mesh
        nc, nf = m.n_cells, m.n_faces
        nslots = int(2 * m.n_internal + (nf - m.n_internal))
        g = {
            "volume": np.zeros(nc), "centroid": np.zeros(3 * nc), "face_centroid": np.zeros(3 * nf),
            "area": np.zeros(3 * nf), "d": np.zeros(3 * nf), "d_mag": np.zeros(nf), "w": np.zeros(nf),
            "delta": np.zeros(3 * nf), "g_inv": np.zeros(9 * nc),
        }
        sing = np.zeros(nc, dtype=np.int8)
        cfo = np.zeros(nc + 1, dtype=np.int32)
        cff = np.zeros(nslots, dtype=np.int32)
        ls = np.zeros(3 * nslots)
        self._f("geometry")(self.h, *[dptr(g[k]) for k in ("volume", "centroid", "face_centroid", "area",
                                                           "d", "d_mag", "w", "delta", "g_inv")],
                            sing.ctypes.data_as(C.POINTER(C.c_byte)), iptr(cfo), iptr(cff), dptr(ls))
        g.update(g_singular=sing, cf_offsets=cfo, cf_faces=cff, ls_vec=ls)
        return g

    def precond_create(self, kind: int):
        self._check(self._f("precond_create")(self.h, int(kind)))

    def precond_apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64).reshape(-1)
        z = self.vec()
        self._check(self._f("precond_apply")(self.h, dptr(r), dptr(z)))
        return z

    def jfnk_solve(self, u, cfg: SolverCfg):
        u = np.array(u, dtype=np.float64).reshape(-1)
        rep = SolveReport()
        self._check(self._f("jfnk_solve")(self.h, dptr(u), C.byref(cfg), C.byref(rep)))
        return u, rep

    def run_steps(self, field: np.ndarray, cfg: SolverCfg, n_steps: int):
        """field: (6, 3*n_cells) = u, u_old, u_old_old, v_old, v_old_old, a_old."""
        field = np.array(field, dtype=np.float64).reshape(6, -1).copy()
        reps = (SolveReport * max(n_steps, 1))()
        nrep = C.c_int(0)
        wall = C.c_double(0.0)
        self._check(self._f("run_steps")(self.h, dptr(field.reshape(-1)), C.byref(cfg), int(n_steps), reps,
                                         max(n_steps, 1), C.byref(nrep), C.byref(wall)))
        return field, [reps[i] for i in range(nrep.value)], wall.value


class OracleCase(_CpuCase):
    PREFIX = "orc_"
    PATH = ORACLE_SO

    def time_jv(self, u, r_u, v, reps: int) -> float:
        u, r_u, v = (np.ascontiguousarray(a, dtype=np.float64).reshape(-1) for a in (u, r_u, v))
        return self.lib.orc_time_jv(self.h, dptr(u), dptr(r_u), dptr(v), int(reps))

    def gmres_jv(self, u, r_u, b, restart=30, rel_reduction=1e-3, max_iters=300, right=False):
        u, r_u, b = (np.ascontiguousarray(a, dtype=np.float64).reshape(-1) for a in (u, r_u, b))
        x = self.vec()
        it, st, rel = C.c_int(0), C.c_int(0), C.c_double(0)
        self._check(self.lib.orc_gmres_jv(self.h, dptr(u), dptr(r_u), dptr(b), dptr(x), restart,
                                          rel_reduction, max_iters, int(bool(right)), C.byref(it), C.byref(st),
                                          C.byref(rel)))
        return x, it.value, st.value, rel.value


class RefCase(_CpuCase):
    PREFIX = "ref_"
    PATH = REF_SO

    def time_jv(self, u, r_u, v, reps: int, threads: int = 1) -> float:
        u, r_u, v = (np.ascontiguousarray(a, dtype=np.float64).reshape(-1) for a in (u, r_u, v))
        return self.lib.ref_time_jv(self.h, dptr(u), dptr(r_u), dptr(v), int(reps), int(threads))

    def jacobian(self):
        nnz = self.lib.ref_jacobian_nnz(self.h)
        rp = np.zeros(self.n_cells + 1, dtype=np.int32)
        col = np.zeros(nnz, dtype=np.int32)
        blocks = np.zeros(9 * nnz)
        self.lib.ref_jacobian(self.h, iptr(rp), iptr(col), dptr(blocks))
        return rp, col, blocks.reshape(nnz, 3, 3)


def ref_box_mesh(extents, divisions, kinds, distort=0.0, seed=0) -> Mesh:
    """generate_box_hex + distort_mesh of the reference itself (mesh.cpp:76, :290)."""
    lib = _load(REF_SO, "ref_")
    k = np.ascontiguousarray(kinds, dtype=np.int32)
    h = lib.ref_box_mesh(float(extents[0]), float(extents[1]), float(extents[2]), int(divisions[0]),
                         int(divisions[1]), int(divisions[2]), iptr(k), float(distort), C.c_uint64(seed))
    if not h:
        raise CpuError(1, -1, "ref_box_mesh failed")
    cnt = np.zeros(6, dtype=np.int32)
    lib.ref_mesh_counts(h, iptr(cnt))
    npnt, nf, nfp, nc, nint, npatch = (int(x) for x in cnt)
    pts = np.zeros(3 * npnt)
    fo = np.zeros(nf + 1, dtype=np.int32)
    fp = np.zeros(nfp, dtype=np.int32)
    own = np.zeros(nf, dtype=np.int32)
    nei = np.zeros(nf, dtype=np.int32)
    pk = np.zeros(npatch, dtype=np.int32)
    ps = np.zeros(npatch, dtype=np.int32)
    pc = np.zeros(npatch, dtype=np.int32)
    lib.ref_mesh_export(h, dptr(pts), iptr(fo), iptr(fp), iptr(own), iptr(nei), iptr(pk), iptr(ps), iptr(pc))
    lib.ref_mesh_free(h)
    return Mesh(pts.reshape(-1, 3), fo, fp, own, nei, nc, nint, pk, ps, pc)
