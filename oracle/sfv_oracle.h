/* sfv_oracle.h — CPU restatement of the reference's JFNK hot path, in plain C.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load oracle/liboracle.so, and only as
 * the checker or the timed CPU baseline — never as the product path.
 *
 * Pinning: tests/test_oracle_pin.py checks this restatement bit for bit against
 * the reference itself (oracle/_ref/libsolidfv_ref.so, compiled from
 * /root/reference/proj/src) on geometry, R(u), J.v, ILU(k)/LU applies and JFNK
 * iteration histories, and against the committed golden vectors in tests/golden/
 * (generated from the reference by tests/golden/make_golden.py).
 *
 * Every function cites the reference file:line it restates.  The arithmetic is
 * written in the reference's operation order (types.hpp operators expanded by
 * hand) and compiled with -O2 -ffp-contract=off, so results are bit-identical
 * to the reference build, which has no FMA on baseline x86-64.
 */
#ifndef SFV_ORACLE_H
#define SFV_ORACLE_H

#include "sfv_case.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_case orc_case;

orc_case* orc_create(const sfv_mesh_desc* mesh, const sfv_physics* phys, char* err, int errlen);
void orc_destroy(orc_case* h);
const char* orc_last_error(orc_case* h);
int orc_n_cells(orc_case* h);

void orc_geometry(orc_case* h, double* volume, double* centroid, double* face_centroid,
                  double* area, double* d, double* d_mag, double* w, double* delta, double* g_inv,
                  signed char* g_singular, int* cf_offsets, int* cf_faces, double* ls_vec);

void orc_set_time(orc_case* h, double t);
void orc_set_history(orc_case* h, const double* u_old, const double* u_old_old,
                     const double* v_old, const double* v_old_old);

int orc_residual(orc_case* h, const double* u, double* r, int* cell);
int orc_stabilisation(orc_case* h, const double* u, double* r, int* cell);
/* ResidualEvaluator::commit (discretisation.cpp:91-95); J2 only carries state */
int orc_commit(orc_case* h, const double* u);
/* committed J2 state, 19 doubles per cell: b_bar, eps_p, F */
int orc_law_state(orc_case* h, double* out);
int orc_jv(orc_case* h, const double* u, const double* r_u, const double* v, double* out,
           int* cell);

int orc_precond_create(orc_case* h, int kind);
int orc_precond_apply(orc_case* h, const double* r, double* z);

int orc_jfnk_solve(orc_case* h, double* u, const sfv_solver_cfg* cfg, sfv_solve_report* rep);
int orc_run_steps(orc_case* h, double* field, const sfv_solver_cfg* cfg, int n_steps,
                  sfv_solve_report* reports, int cap, int* n_reports, double* wall);

/* GMRES on the J.v operator at u (used by the Krylov parity tests). */
int orc_gmres_jv(orc_case* h, const double* u, const double* r_u, const double* b, double* x,
                 int restart, double rel_reduction, int max_iters, int right, int* iters, int* status,
                 double* rel_residual);

double orc_time_jv(orc_case* h, const double* u, const double* r_u, const double* v, int reps);

/* DiscretisationConfig::body_force sampled at the cell centroids (3 nc; NULL clears) */
int orc_set_body_force(orc_case* h, const double* f);
/* per boundary face BC values (3 (nf - nint); NULL = per patch values) */
int orc_set_face_bc(orc_case* h, const double* v);

#ifdef __cplusplus
}
#endif

#endif
