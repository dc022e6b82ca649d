/* sfv_case.h — plain-C description of one solidfv problem instance.
 *
 * These are the INPUT structs shared by the product C-ABI (include/sfv.h), the
 * CPU restatement oracle (oracle/sfv_oracle.h) and the reference driver
 * (oracle/ref_driver.cpp), so one set of Python ctypes mirrors feeds all three
 * the same bytes.  Every field restates a reference type:
 *
 *   sfv_mesh_desc   <- solidfv::Mesh            (/root/reference/proj/include/solidfv/mesh.hpp:30-49)
 *   sfv_physics     <- BoundaryConditions as built by build_simulation
 *                      (/root/reference/proj/src/io.cpp:276-279: value * (ramp ? t : 1)),
 *                      MechanicalLaw (laws.hpp:95-126) and DiscretisationConfig
 *                      (discretisation.hpp:18-25)
 *   sfv_solver_cfg  <- SolverConfig             (nonlinear.hpp:27-44)
 *   sfv_solve_report<- SolveReport / IterationRecord (nonlinear.hpp:46-65)
 */
#ifndef SFV_CASE_H
#define SFV_CASE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* PatchKind (mesh.hpp:15) */
enum { SFV_PATCH_DISPLACEMENT = 0, SFV_PATCH_TRACTION = 1, SFV_PATCH_SYMMETRY = 2 };

/* constitutive laws on the hot path (laws.hpp:95, :117) */
enum { SFV_LAW_HOOKE = 0, SFV_LAW_NEO_HOOKEAN = 1, SFV_LAW_STVK = 2, SFV_LAW_GUCCIONE = 3, SFV_LAW_J2 = 4 };

/* PreconditionerKind (nonlinear.hpp:18) */
enum {
    SFV_PRECOND_AUTO = 0,
    SFV_PRECOND_NONE = 1,
    SFV_PRECOND_ILU0 = 2,
    SFV_PRECOND_ILU1 = 3,
    SFV_PRECOND_ILU2 = 4,
    SFV_PRECOND_LU = 5
};

/* SolveStatus (nonlinear.hpp:19) */
enum { SFV_CONVERGED = 0, SFV_DIVERGED = 1, SFV_MAX_ITERS = 2 };

/* Error codes: one per solidfv exception type that can cross the hot path
 * (errors.hpp:8-46).  Non-convergence is a status, never an error. */
enum {
    SFV_OK = 0,
    SFV_ERR_INVALID_ARGUMENT = 1,
    SFV_ERR_GEOMETRY = 2,
    SFV_ERR_GRADIENT_FAILURE = 3,
    SFV_ERR_INVERTED_ELEMENT = 4,
    SFV_ERR_LAW_OVERFLOW = 5,
    SFV_ERR_RESIDUAL_NAN = 6,
    SFV_ERR_JVP_NAN = 7,
    SFV_ERR_ILU_BREAKDOWN = 8,
    SFV_ERR_LU_SINGULAR = 9,
    SFV_ERR_CUDA = 10,
    SFV_ERR_INTERNAL = 11,
    SFV_ERR_RETURN_MAP = 12
};

/* Face-addressed mesh (mesh.hpp:30-49).  Internal faces first, boundary faces in
 * contiguous patch ranges; face point lists are CSR (face_offsets has n_faces+1). */
typedef struct sfv_mesh_desc {
    int dim; /* 3 */
    int n_points;
    const double* points; /* 3 * n_points, xyz interleaved */
    int n_faces;
    const int* face_offsets; /* n_faces + 1 */
    const int* face_points;
    const int* owner;     /* n_faces */
    const int* neighbour; /* n_faces, -1 on boundary */
    int n_cells;
    int n_internal;
    int n_patches;
    const int* patch_kind;  /* n_patches, SFV_PATCH_* */
    const int* patch_start; /* n_patches */
    const int* patch_count; /* n_patches */
} sfv_mesh_desc;

/* Law + discretisation + per-patch boundary data. */
typedef struct sfv_physics {
    int law;          /* SFV_LAW_* */
    double mu;        /* Pa */
    double lambda;    /* Hooke: Lame lambda; neo-Hookean: bulk modulus kappa */
    double alpha;     /* stabilisation scale (default 1) */
    int total_lagrangian;
    int transient;
    double dt;
    double rho;
    const double* bc_value; /* 3 * n_patches; unused for symmetry patches */
    const int* bc_ramp;     /* n_patches; value * t when nonzero */
    /* SFV_LAW_GUCCIONE (GuccioneParams, laws.hpp:38-43): C, c_f, c_t, c_fs, kappa, f0 xyz */
    double guccione[8];
    /* SFV_LAW_J2 (J2PlasticLaw, mu and kappa = lambda): HardeningCurve saturation
     * a + b e + (c - a)(1 - exp(-d e)) when j2_n_table == 0, else j2_n_table (<= 16)
     * (eps_p, sigma_y) pairs, strictly increasing eps_p (laws.hpp:52-64) */
    double j2_curve[4];
    int j2_n_table;
    const double* j2_table;
} sfv_physics;

typedef struct sfv_solver_cfg {
    double a_tol;           /* 1e-50 */
    double r_tol;           /* 1e-6 (BASELINE: 1e-8) */
    double s_tol;           /* 0: inert */
    int max_outer;          /* 0 => 50 */
    double inner_reduction; /* 0 => 1e-3 */
    int restart;            /* 30 */
    int max_krylov;         /* 300, per linear solve */
    int preconditioner;     /* SFV_PRECOND_* */
    int line_search;        /* 1 */
    int algorithm;          /* SFV_ALG_JFNK (default) or SFV_ALG_SEGREGATED (Algorithm, nonlinear.hpp:17) */
    double relaxation;      /* segregated update under-relaxation in (0, 1]; 0 => 1 */
    int right_preconditioned; /* GMRES on A M^-1 (SolverConfig::right_preconditioned, nonlinear.hpp:37) */
} sfv_solver_cfg;

enum { SFV_ALG_JFNK = 0, SFV_ALG_SEGREGATED = 1 };

typedef struct sfv_iteration_record {
    int step;
    int iter;
    double r_norm;
    int krylov_iters;
    double s;
} sfv_iteration_record;

#define SFV_DETAIL_LEN 160
typedef struct sfv_solve_report {
    int status; /* SFV_CONVERGED / SFV_DIVERGED / SFV_MAX_ITERS */
    int step;
    int outer_iters;
    int krylov_iters;
    double initial_residual;
    double final_residual;
    double wall_seconds;
    int n_records; /* number of valid entries in records (<= capacity) */
    sfv_iteration_record records[64];
    char detail[SFV_DETAIL_LEN];
    int cg_diag_fallback; /* segregated: an IC(0) breakdown fell back to Jacobi (SolveReport) */
    /* SolveReport::iterations is unbounded (nonlinear.hpp:64): when the caller sets
     * all_records, every record (n_records of them, up to all_capacity) is written there
     * too; records[] keeps the first 64.  Both fields survive the solver's reset. */
    sfv_iteration_record* all_records;
    int all_capacity;
} sfv_solve_report;

#ifdef __cplusplus
}
#endif

#endif /* SFV_CASE_H */
