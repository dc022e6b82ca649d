"""CPU-side checks of the boundary: libsfv.so loads without a GPU and exports every
entry point include/*.h declares; the host-side generators and geometry are
bit-identical to the reference's (mesh.cpp) and to the C oracle."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2502_17217_b200 import cases
from paper_2502_17217_b200.abi import PATCH_DISPLACEMENT as D, PATCH_SYMMETRY as S, PATCH_TRACTION as T, dptr, iptr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:sfv|orc)_[a-z0-9_]+)\s*\(", src)))


def test_libsfv_exports_every_declared_symbol():
    from paper_2502_17217_b200.solver import LIB_PATH
    lib = C.CDLL(LIB_PATH)
    names = declared("include/sfv.h")
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_oracle_exports_every_declared_symbol():
    from oracle.bind import ORACLE_SO
    lib = C.CDLL(ORACLE_SO)
    names = declared("oracle/sfv_oracle.h")
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_product_has_no_oracle_dependency():
    """The product library must not link or load anything under oracle/."""
    import subprocess
    from paper_2502_17217_b200.solver import LIB_PATH
    out = subprocess.run(["ldd", LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out and "solidfv_ref" not in out
    for py in ("solver.py", "abi.py", "cases.py", "__init__.py"):
        src = open(os.path.join(ROOT, "paper_2502_17217_b200", py)).read()
        assert "oracle" not in re.sub(r'""".*?"""', "", src, flags=re.S).replace("oracle/", ""), py


@pytest.mark.parametrize("args", [
    ((1.0, 1.2, 0.8), (6, 5, 4), [D, T, S, T, T, T], 0.15, 42),
    ((4.0, 1.0, 1.0), (20, 5, 5), [D, D, T, T, T, T], 0.05, 42),
    ((1.0, 1.0, 1.0), (7, 7, 7), [D, T, T, T, T, T], 0.0, 0),
    ((1.0, 1.0, 1.0), (12, 12, 12), [D, T, T, T, T, T], 0.15, 42),
])
def test_box_generator_matches_reference(args, ref_available):
    if not ref_available:
        pytest.skip("reference build absent")
    from oracle.bind import ref_box_mesh
    from paper_2502_17217_b200.solver import box_mesh
    a, b = box_mesh(*args), ref_box_mesh(*args)
    for k in ("points", "face_offsets", "face_points", "owner", "neighbour", "patch_kind", "patch_start",
              "patch_count"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def _host_geometry(mesh):
    from paper_2502_17217_b200.solver import lib
    L = lib()
    L.sfv_mesh_geometry.restype = C.c_int
    nc, nf = mesh.n_cells, mesh.n_faces
    nslots = int(2 * mesh.n_internal + (nf - mesh.n_internal))
    g = {k: np.zeros(s) for k, s in (("volume", nc), ("centroid", 3 * nc), ("face_centroid", 3 * nf),
                                      ("area", 3 * nf), ("d", 3 * nf), ("d_mag", nf), ("w", nf), ("delta", 3 * nf),
                                      ("g_inv", 9 * nc))}
    sing = np.zeros(nc, dtype=np.int8)
    cfo, cff, ls = np.zeros(nc + 1, dtype=np.int32), np.zeros(nslots, dtype=np.int32), np.zeros(3 * nslots)
    err = C.create_string_buffer(256)
    md = mesh.desc()
    rc = L.sfv_mesh_geometry(C.byref(md), *[dptr(g[k]) for k in ("volume", "centroid", "face_centroid", "area",
                                                                 "d", "d_mag", "w", "delta", "g_inv")],
                             sing.ctypes.data_as(C.POINTER(C.c_byte)), iptr(cfo), iptr(cff), dptr(ls), err, 256)
    assert rc == 0, err.value
    g.update(g_singular=sing, cf_offsets=cfo, cf_faces=cff, ls_vec=ls)
    return g


@pytest.mark.parametrize("name,n", [("c1", 6), ("c2", 8), ("c2", 24), ("c3", 12), ("c5", 4), ("c5", 12)])
def test_product_geometry_matches_oracle(name, n):
    from oracle.bind import OracleCase
    case = cases.config(name, n=n)
    mesh = case.mesh()
    g1 = _host_geometry(mesh)
    g2 = OracleCase(mesh, case.physics).geometry()
    for k in g1:
        assert np.array_equal(g1[k], g2[k]), k


def test_tet_generator_properties():
    from oracle.bind import OracleCase
    for n, singular in ((4, 0), (6, 0), (5, 30)):  # even n: conforming and regular (SURVEY finding 7)
        case = cases.config("c5", n=n)
        mesh = case.mesh()
        assert mesh.n_cells == 6 * n ** 3
        assert mesh.n_faces - mesh.n_internal == 12 * n * n  # conforming boundary
        assert int(mesh.owner[: mesh.n_internal].max()) < mesh.n_cells
        assert np.all(mesh.owner[: mesh.n_internal] < mesh.neighbour[: mesh.n_internal])
        g = OracleCase(mesh, case.physics).geometry()
        assert int(g["g_singular"].sum()) == singular
        assert (g["volume"] > 0).all()


def test_seeded_inputs_deterministic():
    case = cases.config("c2", n=6)
    m = case.mesh()
    u1, v1 = cases.jv_inputs(m)
    u2, v2 = cases.jv_inputs(m)
    assert np.array_equal(u1, u2) and np.array_equal(v1, v2)
    assert abs(np.linalg.norm(v1) - 1.0) < 1e-14
    assert np.abs(u1).max() <= 1e-6 * 1.0 + 1e-18


def test_gpu_path_fails_loudly_without_device(monkeypatch):
    import paper_2502_17217_b200.solver as sv
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    case = cases.config("c1", n=4)
    with pytest.raises(RuntimeError):
        sv.ResidualEvaluator(case.mesh(), case.physics)


def test_report_csv_writers(tmp_path):
    """metrics.csv / iterations.csv in the reference's format (io.cpp:458-488)."""
    from paper_2502_17217_b200.abi import SolveReport
    from paper_2502_17217_b200.reports import write_iterations_csv, write_metrics_csv
    r = SolveReport()
    r.status, r.step, r.outer_iters, r.krylov_iters = 0, 1, 2, 17
    r.initial_residual, r.final_residual, r.wall_seconds = 1234.5, 1.0 / 3.0, 0.25
    r.n_records = 2
    r.records[0].step, r.records[0].iter, r.records[0].r_norm = 1, 0, 1234.5
    r.records[1].step, r.records[1].iter, r.records[1].r_norm = 1, 1, 2.0 / 3.0
    r.records[1].krylov_iters, r.records[1].s = 17, 0.5
    write_metrics_csv([r], str(tmp_path / "m.csv"))
    write_iterations_csv([r], str(tmp_path / "i.csv"))
    m = (tmp_path / "m.csv").read_text().splitlines()
    assert m[0] == "step,status,outer_iters,krylov_iters,initial_residual,final_residual,wall_seconds,detail"
    assert m[1] == "1,converged,2,17,1234.5,0.333333333333,0.25,"
    assert m[2] == "total,,2,17,,,0.25,"
    i = (tmp_path / "i.csv").read_text().splitlines()
    assert i == ["step,iter,r_norm,krylov_iters,s", "1,0,1234.5,0,0", "1,1,0.666666666667,17,0.5"]
