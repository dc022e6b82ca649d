// ref_driver.cpp — extern "C" shim around the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled (by oracle/Makefile) together with the
// reference sources where they lie under /root/reference/proj/src into
// oracle/_ref/libsolidfv_ref.so, with the reference's own flags (-std=c++20 -O2,
// /root/reference/proj/CMakeLists.txt:3,11).  Used by tests/ to pin the C
// restatement oracle (oracle/sfv_oracle.c) and by bench.py --impl reference as
// the CPU baseline.  Nothing here is on the product path.
//
// Every entry point drives the reference through its public C++ API:
//   generate_box_hex / distort_mesh / compute_geometry (mesh.hpp:77-89),
//   ResidualEvaluator::residual (discretisation.hpp:55),
//   jacobian_vector_product (nonlinear.hpp:74), jfnk_solve / run_steps
//   (nonlinear.hpp:96-118), make_preconditioner (nonlinear.hpp:122).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <array>
#include <map>
#include <memory>
#include <thread>
#include <vector>

#include "sfv_case.h"
#include "solidfv/discretisation.hpp"
#include "solidfv/errors.hpp"
#include "solidfv/laws.hpp"
#include "solidfv/mesh.hpp"
#include "solidfv/nonlinear.hpp"

using namespace solidfv;

namespace {

struct RefCase {
    Mesh mesh;
    MeshGeometry geom;
    // what the evaluator was built from (rebuilt when the body force or the BC values change)
    std::shared_ptr<MechanicalLaw> law;
    BoundaryConditions bcs;
    DiscretisationConfig dc;
    std::unique_ptr<ResidualEvaluator> eval;
    std::unique_ptr<Preconditioner> precond;
    std::string last_error;
};

PatchKind kind_of(int k) {
    return k == SFV_PATCH_DISPLACEMENT ? PatchKind::displacement
           : k == SFV_PATCH_SYMMETRY   ? PatchKind::symmetry
                                       : PatchKind::traction;
}

int kind_code(PatchKind k) {
    return k == PatchKind::displacement ? SFV_PATCH_DISPLACEMENT
           : k == PatchKind::symmetry   ? SFV_PATCH_SYMMETRY
                                        : SFV_PATCH_TRACTION;
}

Mesh mesh_from_desc(const sfv_mesh_desc* d) {
    Mesh m;
    m.dim = d->dim;
    m.points.resize(d->n_points);
    for (int i = 0; i < d->n_points; ++i)
        m.points[i] = {d->points[3 * i], d->points[3 * i + 1], d->points[3 * i + 2]};
    m.faces.resize(d->n_faces);
    for (int f = 0; f < d->n_faces; ++f)
        m.faces[f].assign(d->face_points + d->face_offsets[f], d->face_points + d->face_offsets[f + 1]);
    m.owner.assign(d->owner, d->owner + d->n_faces);
    m.neighbour.assign(d->neighbour, d->neighbour + d->n_faces);
    static const char* names[6] = {"xmin", "xmax", "ymin", "ymax", "zmin", "zmax"};
    for (int p = 0; p < d->n_patches; ++p)
        m.patches.push_back({p < 6 ? names[p] : "patch" + std::to_string(p), kind_of(d->patch_kind[p]),
                             d->patch_start[p], d->patch_count[p]});
    m.n_cells = d->n_cells;
    m.n_internal = d->n_internal;
    m.finalise();
    return m;
}

std::vector<Vec3> cells_of(const double* flat, int n) {
    std::vector<Vec3> v(n);
    for (int c = 0; c < n; ++c) v[c] = {flat[3 * c], flat[3 * c + 1], flat[3 * c + 2]};
    return v;
}

void store(const std::vector<Vec3>& v, double* flat) {
    for (std::size_t c = 0; c < v.size(); ++c) {
        flat[3 * c] = v[c].x;
        flat[3 * c + 1] = v[c].y;
        flat[3 * c + 2] = v[c].z;
    }
}

template <typename F>
int guarded(RefCase* rc, int* cell, F&& body) {
    if (cell) *cell = -1;
    try {
        body();
        return SFV_OK;
    } catch (const GradientFailure& e) {
        if (cell) *cell = e.cell;
        rc->last_error = e.what();
        return SFV_ERR_GRADIENT_FAILURE;
    } catch (const InvertedElement& e) {
        if (cell) *cell = e.cell;
        rc->last_error = e.what();
        return SFV_ERR_INVERTED_ELEMENT;
    } catch (const LawOverflow& e) {
        if (cell) *cell = e.cell;
        rc->last_error = e.what();
        return SFV_ERR_LAW_OVERFLOW;
    } catch (const ReturnMapFailure& e) {
        if (cell) *cell = e.cell;
        rc->last_error = e.what();
        return SFV_ERR_RETURN_MAP;
    } catch (const ResidualNan& e) {
        if (cell) *cell = e.cell;
        rc->last_error = e.what();
        return SFV_ERR_RESIDUAL_NAN;
    } catch (const JvpNan& e) {
        rc->last_error = e.what();
        return SFV_ERR_JVP_NAN;
    } catch (const IluBreakdown& e) {
        rc->last_error = e.what();
        return SFV_ERR_ILU_BREAKDOWN;
    } catch (const LuSingular& e) {
        rc->last_error = e.what();
        return SFV_ERR_LU_SINGULAR;
    } catch (const GeometryFailure& e) {
        rc->last_error = e.what();
        return SFV_ERR_GEOMETRY;
    } catch (const std::exception& e) {
        rc->last_error = e.what();
        return SFV_ERR_INVALID_ARGUMENT;
    }
}

SolverConfig solver_of(const sfv_solver_cfg* c) {
    SolverConfig s;
    s.algorithm = Algorithm::jfnk;
    s.a_tol = c->a_tol;
    s.r_tol = c->r_tol;
    s.s_tol = c->s_tol;
    s.max_outer = c->max_outer;
    s.inner_reduction = c->inner_reduction;
    s.restart = c->restart;
    s.max_krylov = c->max_krylov;
    static const PreconditionerKind kinds[6] = {
        PreconditionerKind::automatic, PreconditionerKind::none, PreconditionerKind::ilu0,
        PreconditionerKind::ilu1,      PreconditionerKind::ilu2, PreconditionerKind::lu};
    s.preconditioner = kinds[c->preconditioner];
    s.line_search = c->line_search != 0;
    s.algorithm = c->algorithm == SFV_ALG_SEGREGATED ? Algorithm::segregated : Algorithm::jfnk;
    s.relaxation = c->relaxation > 0.0 ? c->relaxation : 1.0;
    s.right_preconditioned = c->right_preconditioned != 0;
    return s;
}

void report_of(const SolveReport& r, sfv_solve_report* out) {
    std::memset(out, 0, sizeof(*out));
    out->status = r.status == SolveStatus::converged  ? SFV_CONVERGED
                  : r.status == SolveStatus::diverged ? SFV_DIVERGED
                                                      : SFV_MAX_ITERS;
    out->step = r.step;
    out->outer_iters = r.outer_iters;
    out->krylov_iters = r.krylov_iters;
    out->initial_residual = r.initial_residual;
    out->final_residual = r.final_residual;
    out->wall_seconds = r.wall_seconds;
    const int cap = static_cast<int>(sizeof(out->records) / sizeof(out->records[0]));
    out->n_records = std::min<int>(cap, static_cast<int>(r.iterations.size()));
    for (int i = 0; i < out->n_records; ++i) {
        out->records[i] = {r.iterations[i].step, r.iterations[i].iter, r.iterations[i].r_norm,
                           r.iterations[i].krylov_iters, r.iterations[i].s};
    }
    std::snprintf(out->detail, SFV_DETAIL_LEN, "%s", r.detail.c_str());
    out->cg_diag_fallback = r.cg_diag_fallback ? 1 : 0;
}

}  // namespace

extern "C" {

// ---- mesh generation through the reference generators (pins the product's generator) ----

void* ref_box_mesh(double lx, double ly, double lz, int nx, int ny, int nz, const int* kinds,
                   double distort, uint64_t seed) {
    try {
        BoxPatchSpec spec;
        for (int s = 0; s < 6; ++s) spec[s] = kind_of(kinds[s]);
        auto* m = new Mesh(generate_box_hex({lx, ly, lz}, {nx, ny, nz}, spec));
        if (distort > 0.0) *m = distort_mesh(*m, distort, seed);
        return m;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ref_box_mesh: %s\n", e.what());
        return nullptr;
    }
}

void ref_mesh_counts(void* h, int* counts) {
    const Mesh& m = *static_cast<Mesh*>(h);
    int fp = 0;
    for (const auto& f : m.faces) fp += static_cast<int>(f.size());
    counts[0] = static_cast<int>(m.points.size());
    counts[1] = m.n_faces();
    counts[2] = fp;
    counts[3] = m.n_cells;
    counts[4] = m.n_internal;
    counts[5] = static_cast<int>(m.patches.size());
}

void ref_mesh_export(void* h, double* points, int* face_offsets, int* face_points, int* owner,
                     int* neighbour, int* patch_kind, int* patch_start, int* patch_count) {
    const Mesh& m = *static_cast<Mesh*>(h);
    for (std::size_t i = 0; i < m.points.size(); ++i) {
        points[3 * i] = m.points[i].x;
        points[3 * i + 1] = m.points[i].y;
        points[3 * i + 2] = m.points[i].z;
    }
    int q = 0;
    for (int f = 0; f < m.n_faces(); ++f) {
        face_offsets[f] = q;
        for (int p : m.faces[f]) face_points[q++] = p;
        owner[f] = m.owner[f];
        neighbour[f] = m.neighbour[f];
    }
    face_offsets[m.n_faces()] = q;
    for (std::size_t p = 0; p < m.patches.size(); ++p) {
        patch_kind[p] = kind_code(m.patches[p].kind);
        patch_start[p] = m.patches[p].start;
        patch_count[p] = m.patches[p].count;
    }
}

void ref_mesh_free(void* h) { delete static_cast<Mesh*>(h); }

// ---- one evaluator ----

void* ref_create(const sfv_mesh_desc* md, const sfv_physics* ph, char* err, int errlen) {
    auto rc = std::make_unique<RefCase>();
    try {
        rc->mesh = mesh_from_desc(md);
        rc->geom = compute_geometry(rc->mesh);
        std::shared_ptr<MechanicalLaw> law;
        if (ph->law == SFV_LAW_NEO_HOOKEAN) {
            law = std::make_shared<NeoHookeanLaw>(ph->mu, ph->lambda);
        } else if (ph->law == SFV_LAW_STVK) {
            law = std::make_shared<StVenantKirchhoffLaw>(ph->mu, ph->lambda);
        } else if (ph->law == SFV_LAW_J2) {
            HardeningCurve curve = HardeningCurve::saturation(ph->j2_curve[0], ph->j2_curve[1], ph->j2_curve[2],
                                                              ph->j2_curve[3]);
            for (int k = 0; k < ph->j2_n_table; ++k)
                curve.table.emplace_back(ph->j2_table[2 * k], ph->j2_table[2 * k + 1]);
            law = std::make_shared<J2PlasticLaw>(ph->mu, ph->lambda, curve);
        } else if (ph->law == SFV_LAW_GUCCIONE) {
            const double* q = ph->guccione;
            GuccioneParams gp{q[0], q[1], q[2], q[3], q[4], Vec3{q[5], q[6], q[7]}};
            law = std::make_shared<GuccioneLaw>(gp);
        } else {
            law = std::make_shared<HookeLaw>(ph->mu, ph->lambda);
        }
        BoundaryConditions bcs;
        for (int p = 0; p < md->n_patches; ++p) {
            const Vec3 v{ph->bc_value[3 * p], ph->bc_value[3 * p + 1], ph->bc_value[3 * p + 2]};
            const bool ramp = ph->bc_ramp[p] != 0;
            BoundaryCondition bc;
            bc.kind = kind_of(md->patch_kind[p]);
            if (bc.kind != PatchKind::symmetry)
                bc.value = [v, ramp](const Vec3&, double t) { return ramp ? v * t : v; };
            bcs.push_back(bc);
        }
        DiscretisationConfig dc;
        dc.alpha = ph->alpha;
        dc.total_lagrangian = ph->total_lagrangian != 0;
        dc.transient = ph->transient != 0;
        dc.dt = ph->dt;
        dc.rho = ph->rho;
        rc->law = law;
        rc->bcs = bcs;
        rc->dc = dc;
        rc->eval = std::make_unique<ResidualEvaluator>(rc->mesh, rc->geom, bcs, law, dc);
    } catch (const std::exception& e) {
        if (err) std::snprintf(err, errlen, "%s", e.what());
        return nullptr;
    }
    return rc.release();
}

using PointMap = std::map<std::array<double, 3>, Vec3>;
static std::array<double, 3> key_of(const Vec3& x) { return {x.x, x.y, x.z}; }

// DiscretisationConfig::body_force (discretisation.hpp:24) as a function of position that
// returns the given per-cell values at the cell centroids (where the residual samples it,
// discretisation.cpp:160-161); f NULL clears it.  The evaluator is rebuilt.
int ref_set_body_force(void* h, const double* f) {
    RefCase* rc = static_cast<RefCase*>(h);
    return guarded(rc, nullptr, [&] {
        if (!f) {
            rc->dc.body_force = nullptr;
        } else {
            auto map = std::make_shared<PointMap>();
            for (int c = 0; c < rc->mesh.n_cells; ++c)
                (*map)[key_of(rc->geom.centroid[c])] = Vec3{f[3 * c], f[3 * c + 1], f[3 * c + 2]};
            rc->dc.body_force = [map](const Vec3& x) { return map->at(key_of(x)); };
        }
        const double t = rc->eval->time();
        rc->eval = std::make_unique<ResidualEvaluator>(rc->mesh, rc->geom, rc->bcs, rc->law, rc->dc);
        rc->eval->set_time(t);
    });
}

// BoundaryCondition::value (fields.hpp:16-19) as a function of position returning the given
// per-boundary-face values (3 (n_faces - n_internal)) at the face centroids, where
// ResidualEvaluator::bc_value samples it (discretisation.cpp:82-85).  The evaluator is rebuilt.
int ref_set_face_bc(void* h, const double* v) {
    RefCase* rc = static_cast<RefCase*>(h);
    return guarded(rc, nullptr, [&] {
        auto map = std::make_shared<PointMap>();
        for (int f = rc->mesh.n_internal; f < rc->mesh.n_faces(); ++f) {
            const int i = f - rc->mesh.n_internal;
            (*map)[key_of(rc->geom.face_centroid[f])] = Vec3{v[3 * i], v[3 * i + 1], v[3 * i + 2]};
        }
        for (BoundaryCondition& bc : rc->bcs)
            if (bc.kind != PatchKind::symmetry) bc.value = [map](const Vec3& x, double) { return map->at(key_of(x)); };
        const double t = rc->eval->time();
        rc->eval = std::make_unique<ResidualEvaluator>(rc->mesh, rc->geom, rc->bcs, rc->law, rc->dc);
        rc->eval->set_time(t);
    });
}

void ref_destroy(void* h) { delete static_cast<RefCase*>(h); }

const char* ref_last_error(void* h) { return static_cast<RefCase*>(h)->last_error.c_str(); }

// Geometry export, for pinning the restatement bit for bit.  Per-cell LS vectors
// are returned in Mesh::cell_faces order (CSR offsets in cf_offsets).
void ref_geometry(void* h, double* volume, double* centroid, double* face_centroid, double* area,
                  double* d, double* d_mag, double* w, double* delta, double* g_inv,
                  signed char* g_singular, int* cf_offsets, int* cf_faces, double* ls_vec) {
    const RefCase& rc = *static_cast<RefCase*>(h);
    const Mesh& m = rc.mesh;
    const MeshGeometry& g = rc.geom;
    for (int c = 0; c < m.n_cells; ++c) {
        volume[c] = g.volume[c];
        for (int k = 0; k < 3; ++k) centroid[3 * c + k] = g.centroid[c][k];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) g_inv[9 * c + 3 * i + j] = g.g_inv[c](i, j);
        g_singular[c] = g.g_singular[c];
    }
    for (int f = 0; f < m.n_faces(); ++f) {
        for (int k = 0; k < 3; ++k) {
            face_centroid[3 * f + k] = g.face_centroid[f][k];
            area[3 * f + k] = g.area[f][k];
            d[3 * f + k] = g.d[f][k];
            delta[3 * f + k] = g.delta[f][k];
        }
        d_mag[f] = g.d_mag[f];
        w[f] = g.w[f];
    }
    int q = 0;
    for (int c = 0; c < m.n_cells; ++c) {
        cf_offsets[c] = q;
        for (std::size_t i = 0; i < m.cell_faces[c].size(); ++i, ++q) {
            cf_faces[q] = m.cell_faces[c][i];
            for (int k = 0; k < 3; ++k) ls_vec[3 * q + k] = g.ls_vec[c][i][k];
        }
    }
    cf_offsets[m.n_cells] = q;
}

void ref_set_time(void* h, double t) { static_cast<RefCase*>(h)->eval->set_time(t); }

void ref_set_history(void* h, const double* u_old, const double* u_old_old, const double* v_old,
                     const double* v_old_old) {
    RefCase& rc = *static_cast<RefCase*>(h);
    VectorField f(rc.mesh.n_cells);
    f.u_old = cells_of(u_old, rc.mesh.n_cells);
    f.u_old_old = cells_of(u_old_old, rc.mesh.n_cells);
    f.v_old = cells_of(v_old, rc.mesh.n_cells);
    f.v_old_old = cells_of(v_old_old, rc.mesh.n_cells);
    rc.eval->set_history(f);
}

int ref_residual(void* h, const double* u, double* r, int* cell) {
    RefCase* rc = static_cast<RefCase*>(h);
    return guarded(rc, cell, [&] { store(rc->eval->residual(cells_of(u, rc->mesh.n_cells)), r); });
}

// ResidualEvaluator::commit (discretisation.cpp:91-95)
int ref_commit(void* h, const double* u, int* cell) {
    RefCase* rc = static_cast<RefCase*>(h);
    return guarded(rc, cell, [&] { rc->eval->commit(cells_of(u, rc->mesh.n_cells)); });
}

int ref_stabilisation(void* h, const double* u, double* r, int* cell) {
    RefCase* rc = static_cast<RefCase*>(h);
    return guarded(rc, cell,
                   [&] { store(rc->eval->stabilisation(cells_of(u, rc->mesh.n_cells)), r); });
}

int ref_jv(void* h, const double* u, const double* r_u, const double* v, double* out, int* cell) {
    RefCase* rc = static_cast<RefCase*>(h);
    const int n = 3 * rc->mesh.n_cells;
    return guarded(rc, cell, [&] {
        const std::vector<double> jv = jacobian_vector_product(
            *rc->eval, cells_of(u, rc->mesh.n_cells), std::vector<double>(r_u, r_u + n),
            std::vector<double>(v, v + n));
        std::memcpy(out, jv.data(), sizeof(double) * n);
    });
}

// Aggregate J.v throughput of the reference on `threads` host threads, each
// calling jacobian_vector_product `reps` times on the same (const) evaluator.
// Hooke/neo-Hookean stress() holds no state, so concurrent calls are safe.
double ref_time_jv(void* h, const double* u, const double* r_u, const double* v, int reps,
                   int threads) {
    RefCase* rc = static_cast<RefCase*>(h);
    const int n = 3 * rc->mesh.n_cells;
    const std::vector<Vec3> uc = cells_of(u, rc->mesh.n_cells);
    const std::vector<double> ru(r_u, r_u + n), vv(v, v + n);
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&] {
            for (int r = 0; r < reps; ++r) (void)jacobian_vector_product(*rc->eval, uc, ru, vv);
        });
    for (auto& th : pool) th.join();
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return s;
}

// Approximate-Jacobian preconditioner exactly as run_steps builds it
// (nonlinear.cpp:390-400): expand_scalar of the block matrix, then make_preconditioner.
int ref_precond_create(void* h, int kind) {
    RefCase* rc = static_cast<RefCase*>(h);
    return guarded(rc, nullptr, [&] {
        sfv_solver_cfg c{};
        c.preconditioner = kind;
        const BlockSparseMatrix jac = assemble_approximate_jacobian(
            rc->mesh, rc->geom, rc->eval->kbar(), rc->eval->config());
        rc->precond = make_preconditioner(jac.expand_scalar(), solver_of(&c).preconditioner);
    });
}

int ref_precond_apply(void* h, const double* r, double* z) {
    RefCase* rc = static_cast<RefCase*>(h);
    const int n = 3 * rc->mesh.n_cells;
    return guarded(rc, nullptr, [&] {
        std::vector<double> in(r, r + n);
        const std::vector<double> out = rc->precond ? rc->precond->solve(in) : in;
        std::memcpy(z, out.data(), sizeof(double) * n);
    });
}

// Approximate Jacobian in block-CSR form (cell graph, diagonal of each 3x3 block).
int ref_jacobian_nnz(void* h) {
    RefCase* rc = static_cast<RefCase*>(h);
    const BlockSparseMatrix jac =
        assemble_approximate_jacobian(rc->mesh, rc->geom, rc->eval->kbar(), rc->eval->config());
    return static_cast<int>(jac.col.size());
}

void ref_jacobian(void* h, int* row_ptr, int* col, double* blocks) {
    RefCase* rc = static_cast<RefCase*>(h);
    const BlockSparseMatrix jac =
        assemble_approximate_jacobian(rc->mesh, rc->geom, rc->eval->kbar(), rc->eval->config());
    std::memcpy(row_ptr, jac.row_ptr.data(), sizeof(int) * jac.row_ptr.size());
    std::memcpy(col, jac.col.data(), sizeof(int) * jac.col.size());
    for (std::size_t p = 0; p < jac.blocks.size(); ++p)
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) blocks[9 * p + 3 * i + j] = jac.blocks[p](i, j);
}

// One JFNK solve at the evaluator's current time with the preconditioner built by
// ref_precond_create (null => identity).  u is the initial guess in, iterate out.
int ref_jfnk_solve(void* h, double* u, const sfv_solver_cfg* cfg, sfv_solve_report* rep) {
    RefCase* rc = static_cast<RefCase*>(h);
    return guarded(rc, nullptr, [&] {
        std::vector<Vec3> uc = cells_of(u, rc->mesh.n_cells);
        const SolveReport r = jfnk_solve(*rc->eval, uc, solver_of(cfg), rc->precond.get());
        store(uc, u);
        report_of(r, rep);
    });
}

// run_steps (nonlinear.cpp:382-446).  field holds 6 interleaved arrays of 3*n_cells:
// u, u_old, u_old_old, v_old, v_old_old, a_old (VectorField, fields.hpp:29-42).
int ref_run_steps(void* h, double* field, const sfv_solver_cfg* cfg, int n_steps,
                  sfv_solve_report* reports, int cap, int* n_reports, double* wall) {
    RefCase* rc = static_cast<RefCase*>(h);
    const int nc = rc->mesh.n_cells;
    return guarded(rc, nullptr, [&] {
        VectorField f(nc);
        f.u = cells_of(field, nc);
        f.u_old = cells_of(field + 3 * nc, nc);
        f.u_old_old = cells_of(field + 6 * nc, nc);
        f.v_old = cells_of(field + 9 * nc, nc);
        f.v_old_old = cells_of(field + 12 * nc, nc);
        f.a_old = cells_of(field + 15 * nc, nc);
        const SteppingResult res = run_steps(*rc->eval, f, solver_of(cfg), n_steps);
        store(f.u, field);
        store(f.u_old, field + 3 * nc);
        store(f.u_old_old, field + 6 * nc);
        store(f.v_old, field + 9 * nc);
        store(f.v_old_old, field + 12 * nc);
        store(f.a_old, field + 15 * nc);
        *n_reports = std::min<int>(cap, static_cast<int>(res.steps.size()));
        for (int i = 0; i < *n_reports; ++i) report_of(res.steps[i], &reports[i]);
        *wall = res.wall_seconds;
    });
}

}  // extern "C"
