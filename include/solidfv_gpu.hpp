// solidfv_gpu.hpp — the reference's JFNK hot path on the B200, behind the reference's own
// C++ types (/root/reference/proj/include/solidfv).  Header-only; links against libsfv.so
// (include/sfv.h) and the reference library.  INTEGRATION.md shows how a reference build adds it.
//
//   reference call (nonlinear.hpp / linalg.hpp)            drop-in here
//   ---------------------------------------------------    ------------------------------------------
//   run_steps(eval, field, cfg, n, on_step)  :105-107       gpu::run_steps(eval, field, cfg, n, on_step)
//   jfnk_solve(eval, u, cfg, precond)        :96-97         gpu::jfnk_solve(ctx, u, cfg)
//   jacobian_vector_product(eval, u, r_u, v) :72-77         gpu::jacobian_vector_product(ctx, u, r_u, v)
//   LinearOperator for gmres_solve           linalg.hpp:53  gpu::jacobian_operator(ctx, u, r_u)
//   make_preconditioner(J~, kind) -> Preconditioner         gpu::make_preconditioner(ctx, kind)
//   eval.residual(u)                         disc.hpp:55    gpu::residual(ctx, u)
//   line_search(eval, u, du, r0)             :88-90         gpu::line_search(ctx, u, du, r0)
//
// What crosses to the device: the mesh (sfv_mesh_desc), the law parameters (the reference's
// law classes keep them private: build laws with gpu::hooke(...) etc., which return the
// reference's own law objects, or pass a plain HookeLaw, whose mu and lambda are read back
// exactly from two stress evaluations), DiscretisationConfig (alpha, total Lagrangian,
// transient dt / rho, and body_force sampled at the cell centroids), and the boundary
// conditions as BoundaryCondition::value sampled at the boundary-face centroids at every
// time the solver visits (ResidualEvaluator::bc_value, discretisation.cpp:82-85).  Every
// device failure is rethrown as the reference's exception type (errors.hpp).
#pragma once

#include <cmath>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "sfv.h"
#include "solidfv/discretisation.hpp"
#include "solidfv/errors.hpp"
#include "solidfv/laws.hpp"
#include "solidfv/linalg.hpp"
#include "solidfv/nonlinear.hpp"

namespace solidfv {
namespace gpu {

// ------------------------------------------------------------------ law parameters
struct LawParams {
    int law = SFV_LAW_HOOKE;
    double mu = 0.0, lambda = 0.0;  // lambda: Lame lambda (Hooke, StVK) or kappa (neo-Hookean, J2)
    GuccioneParams guccione{};
    HardeningCurve curve{};
};

class DescribedLaw {
public:
    virtual ~DescribedLaw() = default;
    virtual const LawParams& gpu_params() const = 0;
};

// The reference's law class, remembering the parameters it was built with.
template <class Base>
class Described final : public Base, public DescribedLaw {
public:
    template <class... A>
    explicit Described(LawParams p, A&&... a) : Base(std::forward<A>(a)...), p_(std::move(p)) {}
    const LawParams& gpu_params() const override { return p_; }

private:
    LawParams p_;
};

inline std::shared_ptr<MechanicalLaw> hooke(double mu, double lambda) {
    return std::make_shared<Described<HookeLaw>>(LawParams{SFV_LAW_HOOKE, mu, lambda, {}, {}}, mu, lambda);
}
inline std::shared_ptr<MechanicalLaw> stvk(double mu, double lambda) {
    return std::make_shared<Described<StVenantKirchhoffLaw>>(LawParams{SFV_LAW_STVK, mu, lambda, {}, {}}, mu,
                                                             lambda);
}
inline std::shared_ptr<MechanicalLaw> neo_hookean(double mu, double kappa) {
    return std::make_shared<Described<NeoHookeanLaw>>(LawParams{SFV_LAW_NEO_HOOKEAN, mu, kappa, {}, {}}, mu, kappa);
}
inline std::shared_ptr<MechanicalLaw> guccione(const GuccioneParams& g) {
    return std::make_shared<Described<GuccioneLaw>>(LawParams{SFV_LAW_GUCCIONE, 0.0, 0.0, g, {}}, g);
}
inline std::shared_ptr<MechanicalLaw> j2(double mu, double kappa, const HardeningCurve& c) {
    return std::make_shared<Described<J2PlasticLaw>>(LawParams{SFV_LAW_J2, mu, kappa, {}, c}, mu, kappa, c);
}

// Parameters of the evaluator's law: a gpu:: law, or a plain HookeLaw (hooke_stress,
// laws.cpp:20-27, returns mu * (1 + 0) for a unit shear gradient and lambda * 1 off the loaded
// diagonal for a unit stretch — exact in IEEE arithmetic).
inline LawParams law_params(MechanicalLaw& law) {
    if (const auto* d = dynamic_cast<const DescribedLaw*>(&law)) return d->gpu_params();
    if (dynamic_cast<HookeLaw*>(&law)) {
        Mat3 shear = Mat3::zero(), stretch = Mat3::zero();
        shear(0, 1) = 1.0;
        stretch(0, 0) = 1.0;
        LawParams p;
        p.mu = law.stress(0, shear)(0, 1);
        p.lambda = law.stress(0, stretch)(1, 1);
        return p;
    }
    throw InvalidArgument("solidfv::gpu: the law's parameters are not visible; build it with solidfv::gpu::"
                          "hooke / stvk / neo_hookean / guccione / j2");
}

// ------------------------------------------------------------------ errors
[[noreturn]] inline void raise(int code, const char* msg, int cell) {
    const std::string m = msg ? msg : "";
    switch (code) {
        case SFV_ERR_GEOMETRY: throw GeometryFailure(m);
        case SFV_ERR_GRADIENT_FAILURE: throw GradientFailure(cell, m);
        case SFV_ERR_INVERTED_ELEMENT: throw InvertedElement(cell, m);
        case SFV_ERR_LAW_OVERFLOW: throw LawOverflow(cell, m);
        case SFV_ERR_RETURN_MAP: throw ReturnMapFailure(cell, m);
        case SFV_ERR_RESIDUAL_NAN: throw ResidualNan(cell, m);
        case SFV_ERR_JVP_NAN: throw JvpNan(m);
        case SFV_ERR_ILU_BREAKDOWN: throw IluBreakdown(m);
        case SFV_ERR_LU_SINGULAR: throw LuSingular(m);
        case SFV_ERR_INVALID_ARGUMENT: throw InvalidArgument(m);
        default: throw Error("solidfv::gpu: " + m);
    }
}

// ------------------------------------------------------------------ flat <-> Vec3 (fields.cpp:20-32)
inline std::vector<double> flat(const std::vector<Vec3>& v) {
    std::vector<double> o(3 * v.size());
    for (size_t c = 0; c < v.size(); ++c) {
        o[3 * c] = v[c].x;
        o[3 * c + 1] = v[c].y;
        o[3 * c + 2] = v[c].z;
    }
    return o;
}
inline std::vector<Vec3> cells(const double* f, size_t nc) {
    std::vector<Vec3> o(nc);
    for (size_t c = 0; c < nc; ++c) o[c] = Vec3{f[3 * c], f[3 * c + 1], f[3 * c + 2]};
    return o;
}

// ------------------------------------------------------------------ context
// One device evaluator mirroring a ResidualEvaluator: geometry and the J.v tables are built on
// the device from the mesh (bit-identical to compute_geometry).  The boundary values follow
// the evaluator's time: sync_time() re-samples them at eval.time().
class Context {
public:
    explicit Context(const ResidualEvaluator& eval) : eval_(eval) {
        const Mesh& m = eval.mesh();
        if (m.dim != 3) throw InvalidArgument("solidfv::gpu: 3-D meshes only");
        params_ = law_params(eval.law());
        for (const Vec3& p : m.points) {
            pts_.push_back(p.x);
            pts_.push_back(p.y);
            pts_.push_back(p.z);
        }
        foff_.push_back(0);
        for (const auto& f : m.faces) {
            fpts_.insert(fpts_.end(), f.begin(), f.end());
            foff_.push_back(static_cast<int>(fpts_.size()));
        }
        for (const Patch& p : m.patches) {
            pkind_.push_back(p.kind == PatchKind::displacement ? SFV_PATCH_DISPLACEMENT
                             : p.kind == PatchKind::symmetry   ? SFV_PATCH_SYMMETRY
                                                               : SFV_PATCH_TRACTION);
            pstart_.push_back(p.start);
            pcount_.push_back(p.count);
        }
        sfv_mesh_desc md{};
        md.dim = 3;
        md.n_points = static_cast<int>(m.points.size());
        md.points = pts_.data();
        md.n_faces = m.n_faces();
        md.face_offsets = foff_.data();
        md.face_points = fpts_.data();
        md.owner = m.owner.data();
        md.neighbour = m.neighbour.data();
        md.n_cells = m.n_cells;
        md.n_internal = m.n_internal;
        md.n_patches = static_cast<int>(m.patches.size());
        md.patch_kind = pkind_.data();
        md.patch_start = pstart_.data();
        md.patch_count = pcount_.data();
        const DiscretisationConfig& dc = eval.config();
        std::vector<double> zero_bc(3 * m.patches.size(), 0.0);  // per-face values below
        std::vector<int> no_ramp(m.patches.size(), 0);
        std::vector<double> table;
        for (const auto& e : params_.curve.table) {
            table.push_back(e.first);
            table.push_back(e.second);
        }
        sfv_physics ph{};
        ph.law = params_.law;
        ph.mu = params_.mu;
        ph.lambda = params_.lambda;
        ph.alpha = dc.alpha;
        ph.total_lagrangian = dc.total_lagrangian ? 1 : 0;
        ph.transient = dc.transient ? 1 : 0;
        ph.dt = dc.dt;
        ph.rho = dc.rho;
        ph.bc_value = zero_bc.data();
        ph.bc_ramp = no_ramp.data();
        const GuccioneParams& g = params_.guccione;
        const double gq[8] = {g.C, g.c_f, g.c_t, g.c_fs, g.kappa, g.f0.x, g.f0.y, g.f0.z};
        for (int k = 0; k < 8; ++k) ph.guccione[k] = gq[k];
        ph.j2_curve[0] = params_.curve.a;
        ph.j2_curve[1] = params_.curve.b;
        ph.j2_curve[2] = params_.curve.c;
        ph.j2_curve[3] = params_.curve.d;
        ph.j2_n_table = static_cast<int>(params_.curve.table.size());
        ph.j2_table = table.empty() ? nullptr : table.data();
        char err[256] = {0};
        ctx_ = sfv_create(&md, &ph, err, sizeof err);
        if (!ctx_) throw GeometryFailure(err);
        if (dc.body_force) {  // discretisation.cpp:160-161, sampled where the residual samples it
            std::vector<double> f = flat([&] {
                std::vector<Vec3> v(m.n_cells);
                for (int c = 0; c < m.n_cells; ++c) v[c] = dc.body_force(eval.geometry().centroid[c]);
                return v;
            }());
            check(sfv_set_body_force(ctx_, f.data()));
        }
        sync_time();
    }
    ~Context() {
        if (ctx_) sfv_destroy(ctx_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;

    sfv_ctx* get() const { return ctx_; }
    const ResidualEvaluator& evaluator() const { return eval_; }
    const LawParams& law() const { return params_; }
    int n_cells() const { return eval_.mesh().n_cells; }

    // BoundaryCondition::value at every boundary-face centroid and the evaluator's time
    void sync_time() {
        check(sfv_set_time(ctx_, eval_.time()));
        std::vector<double> v = boundary_values(eval_);
        check(sfv_set_boundary_values(ctx_, v.data()));
    }
    static std::vector<double> boundary_values(const ResidualEvaluator& ev) {
        const Mesh& m = ev.mesh();
        std::vector<double> v(3 * static_cast<size_t>(m.n_faces() - m.n_internal), 0.0);
        for (int f = m.n_internal; f < m.n_faces(); ++f) {
            if (m.kind(f) == PatchKind::symmetry) continue;
            const Vec3 x = ev.bc_value(f);
            const size_t i = 3 * static_cast<size_t>(f - m.n_internal);
            v[i] = x.x;
            v[i + 1] = x.y;
            v[i + 2] = x.z;
        }
        return v;
    }
    void check(int code, int cell = -1) const {
        if (code != SFV_OK) raise(code, sfv_last_error(ctx_), cell);
    }

private:
    const ResidualEvaluator& eval_;
    LawParams params_;
    sfv_ctx* ctx_ = nullptr;
    std::vector<double> pts_;
    std::vector<int> foff_, fpts_, pkind_, pstart_, pcount_;
};

// ------------------------------------------------------------------ evaluations
inline std::vector<Vec3> residual(Context& ctx, const std::vector<Vec3>& u) {
    const std::vector<double> uf = flat(u);
    std::vector<double> r(uf.size());
    int cell = -1;
    ctx.check(sfv_residual_host(ctx.get(), uf.data(), r.data(), &cell), cell);
    return cells(r.data(), u.size());
}

inline std::vector<double> jacobian_vector_product(Context& ctx, const std::vector<Vec3>& u,
                                                   const std::vector<double>& r_u_flat, const std::vector<double>& v) {
    const std::vector<double> uf = flat(u);
    std::vector<double> out(v.size());
    int cell = -1;
    ctx.check(sfv_jv_host(ctx.get(), uf.data(), r_u_flat.data(), v.data(), out.data(), &cell), cell);
    return out;
}

// The J.v LinearOperator gmres_solve applies (nonlinear.cpp:198-200), evaluated on the device.
inline LinearOperator jacobian_operator(Context& ctx, const std::vector<Vec3>& u, std::vector<double> r_u_flat) {
    auto uf = std::make_shared<std::vector<double>>(flat(u));
    auto ru = std::make_shared<std::vector<double>>(std::move(r_u_flat));
    Context* c = &ctx;
    return [c, uf, ru](const std::vector<double>& v) {
        std::vector<double> out(v.size());
        int cell = -1;
        c->check(sfv_jv_host(c->get(), uf->data(), ru->data(), v.data(), out.data(), &cell), cell);
        return out;
    };
}

// The preconditioner run_steps builds from J~ (nonlinear.cpp:353-380, :391-395), factored
// and applied on the device; usable wherever the reference takes a Preconditioner.
class GpuPreconditioner final : public Preconditioner {
public:
    GpuPreconditioner(Context& ctx, PreconditionerKind kind) : ctx_(ctx) {
        static const int code[6] = {SFV_PRECOND_AUTO, SFV_PRECOND_NONE, SFV_PRECOND_ILU0,
                                    SFV_PRECOND_ILU1, SFV_PRECOND_ILU2, SFV_PRECOND_LU};
        ctx.check(sfv_precond_create(ctx.get(), code[static_cast<int>(kind)]));
    }
    std::vector<double> solve(const std::vector<double>& r) const override {
        std::vector<double> z(r.size());
        ctx_.check(sfv_precond_apply_host(ctx_.get(), r.data(), z.data()));
        return z;
    }

private:
    Context& ctx_;
};

inline std::unique_ptr<GpuPreconditioner> make_preconditioner(Context& ctx, PreconditionerKind kind) {
    return std::make_unique<GpuPreconditioner>(ctx, kind);
}

// ------------------------------------------------------------------ solver config / reports
inline sfv_solver_cfg solver_cfg(const SolverConfig& s) {
    s.validate();
    sfv_solver_cfg c{};
    c.a_tol = s.a_tol;
    c.r_tol = s.r_tol;
    c.s_tol = s.s_tol;
    c.max_outer = s.max_outer;
    c.inner_reduction = s.inner_reduction;
    c.restart = s.restart;
    c.max_krylov = s.max_krylov;
    static const int code[6] = {SFV_PRECOND_AUTO, SFV_PRECOND_NONE, SFV_PRECOND_ILU0,
                                SFV_PRECOND_ILU1, SFV_PRECOND_ILU2, SFV_PRECOND_LU};
    c.preconditioner = code[static_cast<int>(s.preconditioner)];
    c.line_search = s.line_search ? 1 : 0;
    c.algorithm = s.algorithm == Algorithm::segregated ? SFV_ALG_SEGREGATED : SFV_ALG_JFNK;
    c.relaxation = s.relaxation;
    c.right_preconditioned = s.right_preconditioned ? 1 : 0;
    return c;
}

// sfv_solve_report with its unbounded iteration history attached
struct ReportBuffer {
    sfv_solve_report r{};
    std::vector<sfv_iteration_record> all;
    explicit ReportBuffer(size_t cap = 4096) : all(cap) {
        r.all_records = all.data();
        r.all_capacity = static_cast<int>(cap);
    }
    SolveReport to_reference() const {
        SolveReport o;
        o.status = r.status == SFV_CONVERGED ? SolveStatus::converged
                   : r.status == SFV_DIVERGED ? SolveStatus::diverged
                                              : SolveStatus::max_iters;
        o.detail = r.detail;
        o.step = r.step;
        o.outer_iters = r.outer_iters;
        o.krylov_iters = r.krylov_iters;
        o.initial_residual = r.initial_residual;
        o.final_residual = r.final_residual;
        o.cg_diag_fallback = r.cg_diag_fallback != 0;
        o.wall_seconds = r.wall_seconds;
        const int n = r.n_records < r.all_capacity ? r.n_records : r.all_capacity;
        for (int i = 0; i < n; ++i)
            o.iterations.push_back({all[i].step, all[i].iter, all[i].r_norm, all[i].krylov_iters, all[i].s});
        return o;
    }
};

// jfnk_solve at the evaluator's current time with the context's preconditioner (build it
// with make_preconditioner first; none otherwise).  u: initial guess in, iterate out.
inline SolveReport jfnk_solve(Context& ctx, std::vector<Vec3>& u, const SolverConfig& cfg) {
    ctx.sync_time();
    const sfv_solver_cfg c = solver_cfg(cfg);
    std::vector<double> uf = flat(u);
    ReportBuffer rb;
    ctx.check(sfv_jfnk_solve_host(ctx.get(), uf.data(), &c, &rb.r));
    u = cells(uf.data(), u.size());
    return rb.to_reference();
}

inline LineSearchResult line_search(Context& ctx, const std::vector<Vec3>& u, const std::vector<Vec3>& du,
                                    double r_norm0) {
    // line_search's schedule (nonlinear.cpp:140-163) with every residual evaluated on the device
    LineSearchResult out;
    double s = 1.0;
    for (int attempt = 0; attempt < 6; ++attempt, s *= 0.5) {  // nonlinear.cpp:143-161
        std::vector<Vec3> cand = u;
        for (size_t c = 0; c < u.size(); ++c) cand[c] += s * du[c];
        std::vector<Vec3> r;
        try {
            r = residual(ctx, cand);
        } catch (const Error&) {
            continue;
        }
        double n2 = 0.0;
        for (const Vec3& x : r) n2 += x.x * x.x + x.y * x.y + x.z * x.z;
        const double rn = std::sqrt(n2);
        if (rn < r_norm0) {
            out.success = true;
            out.s = s;
            out.r_norm = rn;
            out.residual = std::move(r);
            return out;
        }
    }
    return out;
}

// ------------------------------------------------------------------ run_steps
namespace detail {
struct StepState {
    ResidualEvaluator* eval;
    const StepCallback* on_step;
    bool commit_cpu;
    VectorField* field;
};
inline void sample_bcs(void* user, double t, double* values) {
    auto* st = static_cast<StepState*>(user);
    st->eval->set_time(t);  // run_steps sets the evaluator's time per step (nonlinear.cpp:403)
    const std::vector<double> v = Context::boundary_values(*st->eval);
    for (size_t i = 0; i < v.size(); ++i) values[i] = v[i];
}
inline void on_step(void* user, int step, const double* f) {
    auto* st = static_cast<StepState*>(user);
    const size_t nc = st->field->u.size(), n = 3 * nc;
    VectorField& fld = *st->field;
    fld.u = cells(f, nc);
    fld.u_old = cells(f + n, nc);
    fld.u_old_old = cells(f + 2 * n, nc);
    fld.v_old = cells(f + 3 * n, nc);
    fld.v_old_old = cells(f + 4 * n, nc);
    fld.a_old = cells(f + 5 * n, nc);
    if (st->commit_cpu) st->eval->commit(fld.u);  // keep the host law's committed state in step
    if (*st->on_step) (*st->on_step)(step, fld);
}
}  // namespace detail

// run_steps (nonlinear.cpp:382-446) on the device: same signature, same result type.  The
// approximate Jacobian, its factorisation, every Newton and Krylov iteration, the predictor,
// commit and history rotation run on the GPU; boundary values are sampled from the
// evaluator's BoundaryConditions at every step time; on_step sees the field after each
// converged step.  A stateful law (J2) is also committed on the host evaluator per step.
inline SteppingResult run_steps(ResidualEvaluator& eval, VectorField& field, const SolverConfig& cfg, int n_steps,
                                const StepCallback& on_step = {}) {
    cfg.validate();
    if (n_steps < 1) throw InvalidArgument("run_steps: need at least one step");
    Context ctx(eval);
    const sfv_solver_cfg c = solver_cfg(cfg);
    detail::StepState st{&eval, &on_step, ctx.law().law == SFV_LAW_J2, &field};
    ctx.check(sfv_set_boundary_sampler(ctx.get(), detail::sample_bcs, &st));
    ctx.check(sfv_set_step_callback(ctx.get(), detail::on_step, &st));
    std::vector<double> f;
    for (const auto* a : {&field.u, &field.u_old, &field.u_old_old, &field.v_old, &field.v_old_old, &field.a_old}) {
        const std::vector<double> x = flat(*a);
        f.insert(f.end(), x.begin(), x.end());
    }
    std::vector<ReportBuffer> rb(static_cast<size_t>(n_steps));
    std::vector<sfv_solve_report> reps(static_cast<size_t>(n_steps));
    for (int i = 0; i < n_steps; ++i) reps[i] = rb[i].r;
    int n_rep = 0;
    double wall = 0.0;
    ctx.check(sfv_run_steps_host(ctx.get(), f.data(), &c, n_steps, reps.data(), n_steps, &n_rep, &wall));
    const size_t nc = field.u.size(), n = 3 * nc;  // the field as of the last converged step
    std::vector<Vec3>* parts[6] = {&field.u, &field.u_old, &field.u_old_old, &field.v_old, &field.v_old_old,
                                   &field.a_old};
    for (int k = 0; k < 6; ++k) *parts[k] = cells(f.data() + k * n, nc);
    SteppingResult out;
    for (int i = 0; i < n_rep; ++i) {
        rb[i].r = reps[i];
        out.steps.push_back(rb[i].to_reference());
        if (out.steps.back().status != SolveStatus::converged) out.status = out.steps.back().status;
    }
    out.wall_seconds = wall;
    return out;
}

}  // namespace gpu
}  // namespace solidfv
