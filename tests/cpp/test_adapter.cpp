// The drop-in adapter (include/solidfv_gpu.hpp) compiled against the reference's own headers
// and sources (/root/reference/proj, built by tests/cpp/Makefile) and run on the GPU by
// tests/test_gpu_adapter.py.  Each check puts the GPU path where the reference's API expects
// its CPU counterpart and compares with the reference itself:
//   A. gpu::residual == ResidualEvaluator::residual, bit for bit — a distorted mesh with
//      position-dependent boundary functions and a body force (a plain HookeLaw);
//   B. the GPU preconditioner's solve == the reference's IlukPrecond::solve, bit for bit;
//   C. the reference's own gmres_solve with the GPU J.v operator and GPU preconditioner,
//      left and right preconditioned, against the same call with the CPU operator and
//      preconditioner (iterations +-1, solution 1e-6);
//   D. gpu::run_steps against run_steps: statuses, Newton counts, Krylov +-1 per Newton,
//      field 1e-8, on_step called for every step — a Hooke case (automatic LU) and a
//      neo-Hookean total-Lagrangian case built with gpu::neo_hookean (ILU(1)).
// Exit status 0 when every check holds; one line per check on stdout.
#include <cmath>
#include <cstdio>
#include <memory>
#include <vector>

#include "solidfv/discretisation.hpp"
#include "solidfv/linalg.hpp"
#include "solidfv/mesh.hpp"
#include "solidfv/nonlinear.hpp"
#include "solidfv_gpu.hpp"

using namespace solidfv;

namespace {

int failures = 0;
void check(bool ok, const char* what, double a = 0.0, double b = 0.0) {
    std::printf("%s %s (%.6g, %.6g)\n", ok ? "PASS" : "FAIL", what, a, b);
    if (!ok) ++failures;
}

double rel(const std::vector<double>& a, const std::vector<double>& b) {
    double d = 0.0, n = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
        d += (a[i] - b[i]) * (a[i] - b[i]);
        n += b[i] * b[i];
    }
    return std::sqrt(d) / std::max(std::sqrt(n), 1e-300);
}

struct Case {
    Mesh mesh;
    MeshGeometry geom;
    std::unique_ptr<ResidualEvaluator> eval;
};

std::unique_ptr<Case> hooke_case() {
    auto c = std::make_unique<Case>();
    BoxPatchSpec spec;
    spec.fill(PatchKind::traction);
    spec[0] = PatchKind::displacement;
    c->mesh = distort_mesh(generate_box_hex({1.0, 1.0, 1.0}, {12, 12, 12}, spec), 0.15, 42);
    c->geom = compute_geometry(c->mesh);
    BoundaryConditions bcs;
    for (const Patch& p : c->mesh.patches) {
        BoundaryCondition bc;
        bc.kind = p.kind;
        if (p.kind == PatchKind::displacement)
            bc.value = [](const Vec3& x, double t) { return Vec3{1e-5 * x.y * t, 0.0, -2e-6 * x.z * t}; };
        else if (p.name == "ymax")
            bc.value = [](const Vec3& x, double t) { return Vec3{0.5e6 * (1.0 + x.x) * t, 0.0, 0.0}; };
        else
            bc.value = [](const Vec3&, double) { return Vec3{}; };
        bcs.push_back(bc);
    }
    DiscretisationConfig dc;
    dc.body_force = [](const Vec3& x) { return Vec3{0.0, -7800.0 * 9.81 * (1.0 + x.x), 0.0}; };
    const double E = 70e9, nu = 0.33;
    c->eval = std::make_unique<ResidualEvaluator>(c->mesh, c->geom, bcs,
                                                  std::make_shared<HookeLaw>(mu_from(E, nu), lambda_from(E, nu)), dc);
    return c;
}

std::unique_ptr<Case> tl_case(bool gpu_law) {
    auto c = std::make_unique<Case>();
    BoxPatchSpec spec;
    spec.fill(PatchKind::traction);
    spec[0] = PatchKind::displacement;
    spec[1] = PatchKind::displacement;
    c->mesh = distort_mesh(generate_box_hex({4.0, 1.0, 1.0}, {16, 4, 4}, spec), 0.05, 42);
    c->geom = compute_geometry(c->mesh);
    BoundaryConditions bcs;
    for (const Patch& p : c->mesh.patches) {
        BoundaryCondition bc;
        bc.kind = p.kind;
        if (p.name == "xmax")
            bc.value = [](const Vec3&, double t) { return Vec3{0.3 * t, 0.0, 0.0}; };
        else
            bc.value = [](const Vec3&, double) { return Vec3{}; };
        bcs.push_back(bc);
    }
    DiscretisationConfig dc;
    dc.total_lagrangian = true;
    std::shared_ptr<MechanicalLaw> law =
        gpu_law ? gpu::neo_hookean(0.4e6, 2e6) : std::make_shared<NeoHookeanLaw>(0.4e6, 2e6);
    c->eval = std::make_unique<ResidualEvaluator>(c->mesh, c->geom, bcs, law, dc);
    return c;
}

void compare_steps(const char* name, const SteppingResult& cpu, const SteppingResult& gpu, const VectorField& fc,
                   const VectorField& fg, int cpu_cb, int gpu_cb) {
    bool same = cpu.steps.size() == gpu.steps.size() && cpu.status == gpu.status;
    bool kry = same;
    for (size_t i = 0; same && i < cpu.steps.size(); ++i) {
        same = cpu.steps[i].status == gpu.steps[i].status && cpu.steps[i].outer_iters == gpu.steps[i].outer_iters;
        for (size_t k = 1; kry && k < cpu.steps[i].iterations.size() && k < gpu.steps[i].iterations.size(); ++k)
            kry = std::abs(cpu.steps[i].iterations[k].krylov_iters - gpu.steps[i].iterations[k].krylov_iters) <= 1;
    }
    char buf[160];
    std::snprintf(buf, sizeof buf, "%s: run_steps statuses and Newton counts", name);
    check(same, buf, cpu.steps.empty() ? 0 : cpu.steps.back().outer_iters,
          gpu.steps.empty() ? 0 : gpu.steps.back().outer_iters);
    std::snprintf(buf, sizeof buf, "%s: Krylov iterations per Newton step within 1", name);
    check(kry, buf);
    const double e = rel(gpu::flat(fg.u), gpu::flat(fc.u));
    std::snprintf(buf, sizeof buf, "%s: field within 1e-8", name);
    check(e <= 1e-8, buf, e, 1e-8);
    std::snprintf(buf, sizeof buf, "%s: on_step after every step", name);
    check(cpu_cb == gpu_cb && gpu_cb == static_cast<int>(gpu.steps.size()), buf, cpu_cb, gpu_cb);
}

}  // namespace

int main() {
    try {
        // ---------------------------------------------------------------- A, B, C
        auto hc = hooke_case();
        ResidualEvaluator& ev = *hc->eval;
        ev.set_time(1.0);
        const int nc = hc->mesh.n_cells;
        std::vector<Vec3> u(nc);
        for (int c = 0; c < nc; ++c) {
            const Vec3& x = hc->geom.centroid[c];
            u[c] = Vec3{1e-6 * std::sin(3.0 * x.x + x.y), 2e-7 * std::cos(2.0 * x.z), -1e-6 * x.x * x.y};
        }
        gpu::Context ctx(ev);
        const std::vector<Vec3> r_cpu = ev.residual(u);
        const std::vector<Vec3> r_gpu = gpu::residual(ctx, u);
        check(gpu::flat(r_cpu) == gpu::flat(r_gpu), "A: residual bit-identical (boundary functions, body force)");

        const std::vector<double> r_flat = flatten(r_cpu, 3);
        const BlockSparseMatrix jac = assemble_approximate_jacobian(hc->mesh, hc->geom, ev.kbar(), ev.config());
        const auto pc_cpu = make_preconditioner(jac.expand_scalar(), PreconditionerKind::ilu1);
        const auto pc_gpu = gpu::make_preconditioner(ctx, PreconditionerKind::ilu1);
        std::vector<double> probe(r_flat.size());
        for (size_t i = 0; i < probe.size(); ++i) probe[i] = std::sin(0.37 * static_cast<double>(i));
        check(pc_cpu->solve(probe) == pc_gpu->solve(probe), "B: ILU(1) preconditioner solve bit-identical");

        std::vector<double> b(r_flat.size());
        for (size_t i = 0; i < b.size(); ++i) b[i] = -r_flat[i];
        const LinearOperator op_cpu = [&](const std::vector<double>& v) {
            return jacobian_vector_product(ev, u, r_flat, v);
        };
        const LinearOperator op_gpu = gpu::jacobian_operator(ctx, u, r_flat);
        for (bool right : {false, true}) {
            const GmresResult gc = gmres_solve(op_cpu, b, std::vector<double>(b.size(), 0.0), pc_cpu.get(), 30, 1e-6,
                                               300, right);
            const GmresResult gg = gmres_solve(op_gpu, b, std::vector<double>(b.size(), 0.0), pc_gpu.get(), 30, 1e-6,
                                               300, right);
            check(gc.status == gg.status && std::abs(gc.iters - gg.iters) <= 1,
                  right ? "C: gmres_solve (right) with the GPU operator: status, iterations +-1"
                        : "C: gmres_solve (left) with the GPU operator: status, iterations +-1",
                  gc.iters, gg.iters);
            const double e = rel(gg.x, gc.x);
            check(e <= 1e-6, right ? "C: gmres_solve (right) solutions agree" : "C: gmres_solve (left) solutions agree",
                  e, 1e-6);
        }

        // ---------------------------------------------------------------- D
        SolverConfig cfg;
        cfg.r_tol = 1e-8;
        {
            auto a = hooke_case(), g = hooke_case();
            VectorField fa(a->mesh.n_cells), fg(g->mesh.n_cells);
            int na = 0, ng = 0;
            const SteppingResult ra = run_steps(*a->eval, fa, cfg, 2, [&](int, const VectorField&) { ++na; });
            const SteppingResult rg = gpu::run_steps(*g->eval, fg, cfg, 2, [&](int, const VectorField&) { ++ng; });
            compare_steps("D hooke (LU)", ra, rg, fa, fg, na, ng);
        }
        {
            auto a = tl_case(false), g = tl_case(true);
            VectorField fa(a->mesh.n_cells), fg(g->mesh.n_cells);
            int na = 0, ng = 0;
            SolverConfig c2 = cfg;
            c2.preconditioner = PreconditionerKind::ilu1;
            const SteppingResult ra = run_steps(*a->eval, fa, c2, 3, [&](int, const VectorField&) { ++na; });
            const SteppingResult rg = gpu::run_steps(*g->eval, fg, c2, 3, [&](int, const VectorField&) { ++ng; });
            compare_steps("D neo-Hookean TL (ILU(1))", ra, rg, fa, fg, na, ng);
        }
        // a law whose parameters the adapter cannot see is refused, not guessed
        {
            auto t = tl_case(false);
            bool refused = false;
            try {
                gpu::Context bad(*t->eval);
            } catch (const InvalidArgument&) {
                refused = true;
            }
            check(refused, "E: an undescribed neo-Hookean law is refused with InvalidArgument");
        }
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        return 2;
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
