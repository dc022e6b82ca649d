/* sfv.h — C-ABI of the B200-native JFNK hot path (libsfv.so).
 *
 * Plain pointers and sizes only.  "_dev" arguments are CUDA device pointers of
 * 3*n_cells doubles in the reference's interleaved layout [3c + k]
 * (/root/reference/proj/src/fields.cpp:20-25); the *_host variants take host
 * buffers and do the H2D/D2H copies themselves.  All calls are stream-ordered on
 * the context's stream (sfv_set_stream), default the legacy default stream.
 *
 * Each entry point replaces one reference interface (file:line under
 * /root/reference/proj):
 *
 *   sfv_mesh_box            <- generate_box_hex + distort_mesh   include/solidfv/mesh.hpp:77-86
 *   sfv_create              <- compute_geometry + ResidualEvaluator ctor
 *                                                                mesh.hpp:89, discretisation.hpp:51-52
 *   sfv_set_time            <- ResidualEvaluator::set_time       discretisation.hpp:59
 *   sfv_set_history         <- ResidualEvaluator::set_history    discretisation.hpp:63
 *   sfv_residual            <- ResidualEvaluator::residual       discretisation.hpp:55
 *   sfv_stabilisation       <- ResidualEvaluator::stabilisation  discretisation.hpp:57
 *   sfv_jv                  <- jacobian_vector_product           nonlinear.hpp:74-77
 *   sfv_precond_create      <- assemble_approximate_jacobian + make_preconditioner
 *                                                                discretisation.hpp:98, nonlinear.hpp:122
 *   sfv_precond_apply       <- Preconditioner::solve             linalg.hpp:55-59
 *   sfv_gmres_jv            <- gmres_solve(op = J.v at u)        linalg.hpp:94-97
 *   sfv_jfnk_solve          <- jfnk_solve                        nonlinear.hpp:96-97
 *   sfv_segregated_solve    <- segregated_solve                  nonlinear.hpp:101-103
 *   sfv_run_steps           <- run_steps                         nonlinear.hpp:117-118
 *
 * Errors: every call returns SFV_OK or one SFV_ERR_* code (include/sfv_case.h), one
 * per solidfv exception type; *cell receives the offending cell where the reference
 * exception carries one (errors.hpp:18-37).  Non-convergence is a status in
 * sfv_solve_report, never an error, as in the reference.
 */
#ifndef SFV_H
#define SFV_H

#include <stddef.h>
#include <stdint.h>

#include "sfv_case.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sfv_mesh sfv_mesh;
typedef struct sfv_ctx sfv_ctx;

/* ---- mesh generators ---- */
sfv_mesh* sfv_mesh_box(const double extents[3], const int divisions[3], const int patch_kinds[6],
                       double distort_factor, uint64_t seed, char* err, int errlen);
/* The config-5 tet mesh (harness generator; on the device when one is present, else on the host
 * — the same arrays either way). */
sfv_mesh* sfv_mesh_kuhn_tets(const double extents[3], int n, const int patch_kinds[6], uint64_t perm_seed,
                             int permute, int rcm, char* err, int errlen);
/* 1 when the mesh was built by a device generator */
int sfv_mesh_built_on_device(const sfv_mesh* m);
/* counts = {n_points, n_faces, n_face_points, n_cells, n_internal, n_patches} */
void sfv_mesh_counts(const sfv_mesh* m, int counts[6]);
void sfv_mesh_export(const sfv_mesh* m, double* points, int* face_offsets, int* face_points, int* owner,
                     int* neighbour, int* patch_kind, int* patch_start, int* patch_count);
void sfv_mesh_free(sfv_mesh* m);

/* ---- evaluator context ---- */
sfv_ctx* sfv_create(const sfv_mesh_desc* mesh, const sfv_physics* phys, char* err, int errlen);
void sfv_destroy(sfv_ctx* ctx);
int sfv_set_stream(sfv_ctx* ctx, void* cuda_stream);
int sfv_n_cells(const sfv_ctx* ctx);
const char* sfv_last_error(const sfv_ctx* ctx);
/* Execution switches:
 *   "gmres_graph" 1 (default) / 0: run each GMRES restart cycle as one CUDA graph whose
 *   WHILE node holds the Arnoldi steps (J.v, preconditioner, MGS, Givens) on the device,
 *   or drive the steps from the host.  Both give bit-identical iterates.
 *   "sequential_reductions" 0 (default) / 1 (also SFV_SEQ_REDUCE=1): sum every inner product
 *   and norm of the solve (the J.v's |u| and |v|, MGS, GMRES and Newton norms) left to right
 *   from 0.0, as std::inner_product does in the reference (linalg.cpp:18-22,
 *   nonlinear.cpp:13-24), instead of a fixed-order parallel tree.  With every other step
 *   already bit-identical, a JFNK solve with an ILU(k) preconditioner then reproduces the
 *   reference's run bit for bit (residual histories, Krylov counts, field).  ~13 ms per
 *   3M-term sum: a reproducibility / verification mode, not the fast path.
 * Returns SFV_ERR_INVALID_ARGUMENT for an unknown name. */
int sfv_set_option(sfv_ctx* ctx, const char* name, int value);
/* number of device kernels this context has launched so far */
long long sfv_launch_count(const sfv_ctx* ctx);
/* bytes of device memory held by the context */
size_t sfv_device_bytes(const sfv_ctx* ctx);
/* compulsory HBM bytes of one J.v (SURVEY.md §8d byte model) */
double sfv_jv_bytes(const sfv_ctx* ctx);

/* host copies of the geometry, same layout as the oracle's orc_geometry */
int sfv_geometry(const sfv_ctx* ctx, double* volume, double* centroid, double* face_centroid, double* area,
                 double* d, double* d_mag, double* w, double* delta, double* g_inv, signed char* g_singular,
                 int* cf_offsets, int* cf_faces, double* ls_vec);

/* compute_geometry on the host only (no device needed) */
int sfv_mesh_geometry(const sfv_mesh_desc* mesh, double* volume, double* centroid, double* face_centroid,
                      double* area, double* d, double* d_mag, double* w, double* delta, double* g_inv,
                      signed char* g_singular, int* cf_offsets, int* cf_faces, double* ls_vec, char* err,
                      int errlen);

int sfv_set_time(sfv_ctx* ctx, double t);
/* DiscretisationConfig::body_force (discretisation.hpp:24): f = body_force(centroid_c) for every
 * cell (3 n_cells host doubles, interleaved; the centroids are sfv_geometry's, i.e. the
 * reference's); R gains volume_c * f_c after the stabilisation terms (discretisation.cpp:160-161).
 * NULL clears it. */
int sfv_set_body_force(sfv_ctx* ctx, const double* f);
/* Boundary values per face instead of per patch: values[3 i] is BoundaryCondition::value
 * (face_centroid, t) of boundary face n_internal + i at the current time (ResidualEvaluator::
 * bc_value, discretisation.cpp:82-85; 3 (n_faces - n_internal) host doubles).  NULL returns to
 * the per-patch values of sfv_physics. */
int sfv_set_boundary_values(sfv_ctx* ctx, const double* values);
/* The same sampled on every sfv_set_time (and every step of sfv_run_steps): fn(user, t, values)
 * fills the per-face values at time t.  fn NULL returns to the per-patch values. */
typedef void (*sfv_bc_sampler)(void* user, double t, double* values);
int sfv_set_boundary_sampler(sfv_ctx* ctx, sfv_bc_sampler fn, void* user);
int sfv_set_history(sfv_ctx* ctx, const double* u_old_dev, const double* u_old_old_dev, const double* v_old_dev,
                    const double* v_old_old_dev);

int sfv_residual(sfv_ctx* ctx, const double* u_dev, double* r_dev, int* cell);
int sfv_stabilisation(sfv_ctx* ctx, const double* u_dev, double* r_dev, int* cell);
/* ResidualEvaluator::commit (discretisation.hpp:60; discretisation.cpp:91-95): the law's trial
 * state at u becomes its committed state.  Only SFV_LAW_J2 carries state (J2PlasticLaw::commit,
 * laws.cpp:214); for the other laws it is a no-op.  Called by sfv_run_steps after every
 * converged step, as run_steps does (nonlinear.cpp:426). */
int sfv_commit(sfv_ctx* ctx, const double* u_dev);
/* Committed J2 state, host buffer of 19 doubles per cell: b_bar (row-major), eps_p, F
 * (PlasticCell, laws.hpp:66-70).  SFV_ERR_INVALID_ARGUMENT for the other laws. */
int sfv_law_state(sfv_ctx* ctx, double* state);
/* cell_gradients (discretisation.hpp:29-30): G_dev is 9*n_cells, SoA [(3i+j)*n_cells + c] */
int sfv_gradients(sfv_ctx* ctx, const double* u_dev, double* G_dev, int* cell);
int sfv_jv(sfv_ctx* ctx, const double* u_dev, const double* r_u_dev, const double* v_dev, double* out_dev,
           int* cell);
/* J.v with a caller-supplied eps (parity harness: isolates the kernel from the norm
 * reduction order); eps = 0 returns zeros */
int sfv_jv_eps(sfv_ctx* ctx, const double* u_dev, const double* r_u_dev, const double* v_dev, double eps,
               double* out_dev, int* cell);
/* Asynchronous J.v for throughput runs: no host synchronisation, errors accumulate
 * on the device until sfv_check_errors. */
int sfv_jv_async(sfv_ctx* ctx, const double* u_dev, const double* r_u_dev, const double* v_dev, double* out_dev);
int sfv_check_errors(sfv_ctx* ctx, int* cell);
/* Measurement only (bench.py): average device time in ms of each stage of `reps`
 * J.v calls, timed with CUDA events on the context stream: ms[0] |u|,|v| block partials
 * (0 when the reduction is fused into the next pass, the default), ms[1] eps + perturbed
 * state, ms[2] gradients, ms[3] boundary faces (0 when the flux pass evaluates them: Hooke,
 * small strain, no symmetry patch), ms[4] face fluxes + per-cell sums.  Returns
 * SFV_ERR_INVALID_ARGUMENT unless the default (jv_pair.cu) path is active. */
int sfv_jv_stage_times(sfv_ctx* ctx, const double* u_dev, const double* r_u_dev, const double* v_dev,
                       double* out_dev, int reps, double* ms);
/* The bytes each of those five stages moves at least once (its algorithmic traffic). */
void sfv_jv_stage_bytes(const sfv_ctx* ctx, double* bytes);

/* host-buffer conveniences (copies inside the call) */
int sfv_residual_host(sfv_ctx* ctx, const double* u, double* r, int* cell);
int sfv_jv_host(sfv_ctx* ctx, const double* u, const double* r_u, const double* v, double* out, int* cell);

int sfv_precond_create(sfv_ctx* ctx, int kind);
/* assemble_approximate_jacobian (discretisation.hpp:94-99, discretisation.cpp:216-262) in block
 * CSR on the cell graph: row_ptr[n_cells + 1], col[nnz], blocks[9 nnz] (3x3 row-major).  With
 * col or blocks NULL only nnz is returned; otherwise the arrays are filled and nnz returned
 * (< 0: an error code).  Off-diagonal blocks are c I; a diagonal block is c I, per-axis with
 * axis-aligned symmetry faces, or full (- coeff n (x) n, discretisation.cpp:250-251) when a symmetry
 * face's normal is not axis-aligned.  In that last case sfv_precond_create factors the reference's
 * expand_scalar() matrix (linalg.cpp:135-158: 3 n_cells rows, all nine entries of every block) as
 * one system and sfv_precond_apply solves it with the sync-free sweep; the segregated solver
 * refuses it as the reference does (scalar_component, linalg.cpp:120-133). */
int sfv_approximate_jacobian(const sfv_ctx* ctx, int* row_ptr, int* col, double* blocks);
/* line_search (nonlinear.hpp:81-90, nonlinear.cpp:140-163): success, the accepted s and
 * its residual norm, and (when residual_dev is not NULL) the accepted residual. */
int sfv_line_search(sfv_ctx* ctx, const double* u_dev, const double* du_dev, double r_norm0, int* success,
                    double* s, double* r_norm, double* residual_dev);
int sfv_precond_apply(sfv_ctx* ctx, const double* r_dev, double* z_dev);
/* the same with host buffers (Preconditioner::solve, linalg.hpp:53-59) */
int sfv_precond_apply_host(sfv_ctx* ctx, const double* r, double* z);
/* preconditioner facts: {kind_resolved, n_levels_fwd, n_levels_bwd, nnz_L, nnz_U} */
int sfv_precond_info(const sfv_ctx* ctx, int info[5]);
/* Device sweep of the ILU apply: 200 streamed level-synchronous (default), 300 block-
 * pipelined (SFV_PIPE=1), 100 DSMEM ring, 1..16 ELL cluster, 0 sentinel polling; -1 when
 * the preconditioner is not ILU. */
int sfv_precond_sweep(const sfv_ctx* ctx);

/* gmres_solve(op = J.v at u, b, x0 = x_dev, precond = the context's, restart, rel_reduction,
 * max_iters, right_preconditioned) (linalg.cpp:423-538); status 0 converged / 1 max_iters /
 * 2 stagnated (GmresStatus).  Any restart >= 1. */
int sfv_gmres_jv(sfv_ctx* ctx, const double* u_dev, const double* r_u_dev, const double* b_dev, double* x_dev,
                 int restart, double rel_reduction, int max_iters, int right_preconditioned, int* iters, int* status,
                 double* rel_residual);
int sfv_jfnk_solve(sfv_ctx* ctx, double* u_dev, const sfv_solver_cfg* cfg, sfv_solve_report* report);
/* the same with u in host memory (initial guess in, final iterate out) */
int sfv_jfnk_solve_host(sfv_ctx* ctx, double* u, const sfv_solver_cfg* cfg, sfv_solve_report* report);
/* segregated_solve (nonlinear.hpp:101-103; nonlinear.cpp:268-351): per outer iteration, each
 * displacement component by IC(0)-preconditioned CG on A = -J~ (Jacobi when IC(0) breaks
 * down), then u += relaxation (u_next - u).  cfg->algorithm is ignored here; sfv_run_steps
 * dispatches on it (SFV_ALG_SEGREGATED) as run_steps does. */
int sfv_segregated_solve(sfv_ctx* ctx, double* u_dev, const sfv_solver_cfg* cfg, sfv_solve_report* report);
/* StepCallback (nonlinear.hpp:106-107): when set, sfv_run_steps calls fn(user, step, field)
 * after every converged step with the field (6 x 3 n_cells doubles, the layout below) on the
 * host.  fn NULL clears it. */
typedef void (*sfv_step_callback)(void* user, int step, const double* field);
int sfv_set_step_callback(sfv_ctx* ctx, sfv_step_callback fn, void* user);
/* field_dev: 6 consecutive device arrays of 3*n_cells doubles:
 * u, u_old, u_old_old, v_old, v_old_old, a_old (VectorField, fields.hpp:29-42) */
int sfv_run_steps(sfv_ctx* ctx, double* field_dev, const sfv_solver_cfg* cfg, int n_steps,
                  sfv_solve_report* reports, int cap, int* n_reports, double* wall_seconds);
int sfv_run_steps_host(sfv_ctx* ctx, double* field, const sfv_solver_cfg* cfg, int n_steps,
                       sfv_solve_report* reports, int cap, int* n_reports, double* wall_seconds);

#ifdef __cplusplus
}
#endif

#endif /* SFV_H */
