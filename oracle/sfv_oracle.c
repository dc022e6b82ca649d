/* sfv_oracle.c — CPU restatement of the reference hot path.  See sfv_oracle.h.
 *
 * TEST INFRASTRUCTURE ONLY (the checker).  Reference paths below are relative to
 * /root/reference/proj/.  Operation order follows the C++ operators of
 * include/solidfv/types.hpp exactly (e.g. Vec3/s is Vec3*(1.0/s), Vec3*s scales
 * each component, dot is ((x*x' + y*y') + z*z')).
 */
#define _POSIX_C_SOURCE 199309L
#include "sfv_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ types.hpp */

typedef struct { double x, y, z; } v3;
typedef struct { double m[3][3]; } m3;

static inline double vget(v3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }
static inline void vset(v3* a, int i, double v) {
    if (i == 0) a->x = v;
    else if (i == 1) a->y = v;
    else a->z = v;
}
static inline v3 vadd(v3 a, v3 b) { return (v3){a.x + b.x, a.y + b.y, a.z + b.z}; }
static inline v3 vsub(v3 a, v3 b) { return (v3){a.x - b.x, a.y - b.y, a.z - b.z}; }
static inline v3 vscale(v3 a, double s) { return (v3){a.x * s, a.y * s, a.z * s}; } /* s*a, a*s */
static inline v3 vdiv(v3 a, double s) { return vscale(a, 1.0 / s); }             /* types.hpp:30 */
static inline v3 vneg(v3 a) { return (v3){-a.x, -a.y, -a.z}; }
static inline double vdot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline v3 vcross(v3 a, v3 b) {
    return (v3){a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
static inline double vnorm(v3 a) { return sqrt(vdot(a, a)); }
static inline int vfinite(v3 a) { return isfinite(a.x) && isfinite(a.y) && isfinite(a.z); }

static inline m3 mzero(void) { m3 r; memset(&r, 0, sizeof r); return r; }
static inline m3 mident(void) { m3 r = mzero(); r.m[0][0] = r.m[1][1] = r.m[2][2] = 1.0; return r; }
static inline m3 madd(m3 a, m3 b) {
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) a.m[i][j] += b.m[i][j];
    return a;
}
static inline m3 msub(m3 a, m3 b) {
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) a.m[i][j] -= b.m[i][j];
    return a;
}
static inline m3 mscale(m3 a, double s) {
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) a.m[i][j] *= s;
    return a;
}
static inline m3 mmul(m3 a, m3 b) { /* types.hpp:72-81 */
    m3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += a.m[i][k] * b.m[k][j];
            r.m[i][j] = s;
        }
    return r;
}
static inline v3 mvmul(m3 a, v3 v) { /* types.hpp:84-88 */
    return (v3){a.m[0][0] * v.x + a.m[0][1] * v.y + a.m[0][2] * v.z,
                a.m[1][0] * v.x + a.m[1][1] * v.y + a.m[1][2] * v.z,
                a.m[2][0] * v.x + a.m[2][1] * v.y + a.m[2][2] * v.z};
}
static inline v3 dot_left(v3 v, m3 a) { /* types.hpp:91-96 */
    return (v3){v.x * a.m[0][0] + v.y * a.m[1][0] + v.z * a.m[2][0],
                v.x * a.m[0][1] + v.y * a.m[1][1] + v.z * a.m[2][1],
                v.x * a.m[0][2] + v.y * a.m[1][2] + v.z * a.m[2][2]};
}
static inline m3 outer(v3 a, v3 b) {
    m3 r;
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) r.m[i][j] = vget(a, i) * vget(b, j);
    return r;
}
static inline m3 mtrans(m3 a) {
    m3 r;
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[j][i];
    return r;
}
static inline double mtrace(m3 a) { return a.m[0][0] + a.m[1][1] + a.m[2][2]; }
static inline m3 mdev(m3 a) { /* types.hpp:118-125 */
    const double t = mtrace(a) / 3.0;
    a.m[0][0] -= t; a.m[1][1] -= t; a.m[2][2] -= t;
    return a;
}
static inline double mdet(m3 a) { /* types.hpp:127-131 */
    return a.m[0][0] * (a.m[1][1] * a.m[2][2] - a.m[1][2] * a.m[2][1]) -
           a.m[0][1] * (a.m[1][0] * a.m[2][2] - a.m[1][2] * a.m[2][0]) +
           a.m[0][2] * (a.m[1][0] * a.m[2][1] - a.m[1][1] * a.m[2][0]);
}
static inline m3 minverse(m3 a) { /* types.hpp:133-148 (caller checks d != 0) */
    const double id = 1.0 / mdet(a);
    m3 r;
    r.m[0][0] = (a.m[1][1] * a.m[2][2] - a.m[1][2] * a.m[2][1]) * id;
    r.m[0][1] = (a.m[0][2] * a.m[2][1] - a.m[0][1] * a.m[2][2]) * id;
    r.m[0][2] = (a.m[0][1] * a.m[1][2] - a.m[0][2] * a.m[1][1]) * id;
    r.m[1][0] = (a.m[1][2] * a.m[2][0] - a.m[1][0] * a.m[2][2]) * id;
    r.m[1][1] = (a.m[0][0] * a.m[2][2] - a.m[0][2] * a.m[2][0]) * id;
    r.m[1][2] = (a.m[0][2] * a.m[1][0] - a.m[0][0] * a.m[1][2]) * id;
    r.m[2][0] = (a.m[1][0] * a.m[2][1] - a.m[1][1] * a.m[2][0]) * id;
    r.m[2][1] = (a.m[0][1] * a.m[2][0] - a.m[0][0] * a.m[2][1]) * id;
    r.m[2][2] = (a.m[0][0] * a.m[1][1] - a.m[0][1] * a.m[1][0]) * id;
    return r;
}
static inline m3 reflection(v3 n) { return msub(mident(), mscale(outer(n, n), 2.0)); }
static inline m3 interp(m3 a, m3 b, double w) { /* fields.hpp:49-52 */
    return madd(mscale(a, w), mscale(b, 1.0 - w));
}

/* ------------------------------------------------------------------ error state */

typedef struct {
    int code;
    int cell;
    char msg[SFV_DETAIL_LEN];
} orc_err;

static int fail(orc_err* e, int code, int cell, const char* msg) {
    e->code = code;
    e->cell = cell;
    snprintf(e->msg, sizeof e->msg, "%s", msg);
    return code;
}

/* ------------------------------------------------------------------ the case */

typedef struct {
    int n, nnz;
    int* row_ptr;
    int* col;
    double* val;
} csr;

static void csr_free(csr* a) {
    free(a->row_ptr); free(a->col); free(a->val);
    memset(a, 0, sizeof *a);
}

struct orc_case {
    /* mesh (mesh.hpp:30-49) */
    int nc, nf, nint, np, npatch;
    v3* points;
    int* face_off;
    int* face_pts;
    int* owner;
    int* neigh;
    int* patch_kind;
    int* patch_start;
    int* patch_count;
    int* face_patch;
    int* cf_off; /* cell_faces CSR, ascending face index (mesh.cpp:55-59) */
    int* cf;
    /* geometry (mesh.hpp:52-73) */
    double* volume;
    v3* centroid;
    m3* g_inv;
    signed char* g_singular;
    v3* face_centroid;
    v3* area;
    double* area_mag;
    v3* normal;
    v3* d;
    double* d_mag;
    double* w;
    v3* delta;
    double* delta_mag;
    m3* reflect;
    v3* ls; /* aligned with cf */
    /* physics */
    int law;
    double mu, lam;
    double gc[8]; /* Guccione: C, c_f, c_t, c_fs, kappa, f0 */
    /* J2: HardeningCurve (saturation a, b, c, d, or jn table pairs) and committed PlasticCell */
    double ja, jb, jc, jd, jt[32];
    int jn;
    m3 *j2_bbar, *j2_F;
    double* j2_eps;
    double alpha;
    int tl, transient;
    double dt, rho;
    v3* bc_value;
    int* bc_ramp;
    double time;
    v3 *u_old, *u_old_old, *v_old, *v_old_old;
    v3* body_vol; /* volume * body_force(centroid) per cell, NULL = none */
    v3* face_bc;  /* per boundary face value(face_centroid, t), NULL = per patch */
    /* scratch */
    m3 *grad, *sigma, *fdef;
    /* preconditioner */
    int pc_kind; /* 0 none, 1 ilu, 2 lu */
    csr ilu;
    void* lu;
    orc_err err;
};

static int kind_of_face(const orc_case* h, int f) { return h->patch_kind[h->face_patch[f]]; }

static void* xcalloc(size_t n, size_t s) {
    void* p = calloc(n ? n : 1, s);
    if (!p) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
    return p;
}

/* compute_geometry, 3-D branch (mesh.cpp:347-510) */
static int compute_geometry(orc_case* h) {
    const int nf = h->nf, nc = h->nc;
    h->face_centroid = xcalloc(nf, sizeof(v3));
    h->area = xcalloc(nf, sizeof(v3));
    h->area_mag = xcalloc(nf, sizeof(double));
    h->normal = xcalloc(nf, sizeof(v3));
    h->d = xcalloc(nf, sizeof(v3));
    h->d_mag = xcalloc(nf, sizeof(double));
    h->w = xcalloc(nf, sizeof(double));
    h->delta = xcalloc(nf, sizeof(v3));
    h->delta_mag = xcalloc(nf, sizeof(double));
    h->reflect = xcalloc(nf, sizeof(m3));
    for (int f = 0; f < nf; ++f) {
        h->w[f] = 1.0;
        h->reflect[f] = mident();
    }
    /* pass 1 (mesh.cpp:361-390) */
    for (int f = 0; f < nf; ++f) {
        const int* pts = h->face_pts + h->face_off[f];
        const int npt = h->face_off[f + 1] - h->face_off[f];
        v3 centre = {0, 0, 0};
        for (int i = 0; i < npt; ++i) centre = vadd(centre, h->points[pts[i]]);
        centre = vdiv(centre, (double)npt);
        v3 area = {0, 0, 0}, cacc = {0, 0, 0};
        double aacc = 0.0;
        for (int i = 0; i < npt; ++i) {
            const v3 p0 = h->points[pts[i]], p1 = h->points[pts[(i + 1) % npt]];
            const v3 tri = vscale(vcross(vsub(p0, centre), vsub(p1, centre)), 0.5);
            const double tmag = vnorm(tri);
            area = vadd(area, tri);
            cacc = vadd(cacc, vscale(vdiv(vadd(vadd(centre, p0), p1), 3.0), tmag));
            aacc += tmag;
        }
        h->area[f] = area;
        h->face_centroid[f] = aacc > 0.0 ? vdiv(cacc, aacc) : centre;
        h->area_mag[f] = vnorm(area);
        if (h->area_mag[f] <= 0.0) return fail(&h->err, SFV_ERR_GEOMETRY, -1, "compute_geometry: zero-area face");
        h->normal[f] = vdiv(area, h->area_mag[f]);
    }
    /* pass 2 (mesh.cpp:392-435) */
    v3* apex = xcalloc(nc, sizeof(v3));
    int* cnt = xcalloc(nc, sizeof(int));
    for (int f = 0; f < nf; ++f)
        for (int q = h->face_off[f]; q < h->face_off[f + 1]; ++q)
            for (int side = 0; side < 2; ++side) {
                const int c = side == 0 ? h->owner[f] : h->neigh[f];
                if (c < 0) continue;
                apex[c] = vadd(apex[c], h->points[h->face_pts[q]]);
                ++cnt[c];
            }
    for (int c = 0; c < nc; ++c) apex[c] = vdiv(apex[c], (double)cnt[c]);
    h->volume = xcalloc(nc, sizeof(double));
    h->centroid = xcalloc(nc, sizeof(v3));
    for (int f = 0; f < nf; ++f) {
        const int* pts = h->face_pts + h->face_off[f];
        const int npt = h->face_off[f + 1] - h->face_off[f];
        for (int side = 0; side < 2; ++side) {
            const int c = side == 0 ? h->owner[f] : h->neigh[f];
            if (c < 0) continue;
            const double sign = side == 0 ? 1.0 : -1.0;
            for (int i = 0; i < npt; ++i) {
                const v3 p0 = h->points[pts[i]], p1 = h->points[pts[(i + 1) % npt]];
                const v3 fc = h->face_centroid[f];
                const double v =
                    sign * vdot(vsub(fc, apex[c]), vcross(vsub(p0, apex[c]), vsub(p1, apex[c]))) / 6.0;
                h->volume[c] += v;
                h->centroid[c] =
                    vadd(h->centroid[c], vscale(vadd(vadd(vadd(apex[c], fc), p0), p1), v * 0.25));
            }
        }
    }
    free(apex);
    free(cnt);
    for (int c = 0; c < nc; ++c) {
        if (!(h->volume[c] > 0.0))
            return fail(&h->err, SFV_ERR_GEOMETRY, c, "compute_geometry: non-positive volume");
        h->centroid[c] = vdiv(h->centroid[c], h->volume[c]);
    }
    /* pass 3 (mesh.cpp:437-463) */
    for (int f = 0; f < nf; ++f) {
        const v3 n = h->normal[f];
        const v3 xp = h->centroid[h->owner[f]];
        if (f < h->nint) {
            const v3 xn = h->centroid[h->neigh[f]];
            h->d[f] = vsub(xn, xp);
            const double denom = vdot(n, vsub(xn, xp));
            if (!(denom > 0.0))
                return fail(&h->err, SFV_ERR_GEOMETRY, f, "compute_geometry: area vector does not leave the owner");
            h->w[f] = vdot(n, vsub(xn, h->face_centroid[f])) / denom;
        } else if (kind_of_face(h, f) == SFV_PATCH_SYMMETRY) {
            h->reflect[f] = reflection(n);
            h->d[f] = vscale(n, -2.0 * vdot(vsub(xp, h->face_centroid[f]), n));
            h->w[f] = 0.5;
        } else {
            h->d[f] = vsub(h->face_centroid[f], xp);
        }
        h->d_mag[f] = vnorm(h->d[f]);
        const double dn = vdot(h->d[f], n);
        if (!(dn > 0.0))
            return fail(&h->err, SFV_ERR_GEOMETRY, f, "compute_geometry: degenerate centroid geometry");
        h->delta[f] = vdiv(h->d[f], dn);
        h->delta_mag[f] = vnorm(h->delta[f]);
    }
    /* pass 4 (mesh.cpp:465-508) */
    h->g_inv = xcalloc(nc, sizeof(m3));
    h->g_singular = xcalloc(nc, 1);
    m3* gt = xcalloc(nc, sizeof(m3));
    for (int f = 0; f < nf; ++f) {
        const int incl = f < h->nint || kind_of_face(h, f) == SFV_PATCH_SYMMETRY;
        if (!incl) continue;
        const m3 dd = mscale(outer(h->d[f], h->d[f]), h->area_mag[f] / vdot(h->d[f], h->d[f]));
        gt[h->owner[f]] = madd(gt[h->owner[f]], mscale(dd, h->w[f]));
        if (f < h->nint) gt[h->neigh[f]] = madd(gt[h->neigh[f]], mscale(dd, 1.0 - h->w[f]));
    }
    for (int c = 0; c < nc; ++c) {
        const m3 G = gt[c];
        double scale = 0.0;
        for (int i = 0; i < 3; ++i) scale = fmax(scale, fabs(G.m[i][i]));
        if (scale <= 0.0 || fabs(mdet(G)) < 1e-10 * scale * scale * scale) {
            h->g_singular[c] = 1;
            continue;
        }
        h->g_inv[c] = minverse(G);
    }
    free(gt);
    h->ls = xcalloc(h->cf_off[nc], sizeof(v3));
    for (int c = 0; c < nc; ++c) {
        if (h->g_singular[c]) continue;
        for (int q = h->cf_off[c]; q < h->cf_off[c + 1]; ++q) {
            const int f = h->cf[q];
            const int incl = f < h->nint || kind_of_face(h, f) == SFV_PATCH_SYMMETRY;
            if (!incl) continue;
            v3 d = h->d[f];
            double w = h->w[f];
            if (f < h->nint && h->neigh[f] == c) {
                d = vneg(d);
                w = 1.0 - w;
            }
            h->ls[q] = vscale(mvmul(h->g_inv[c], d), w * h->area_mag[f] / vdot(d, d));
        }
    }
    return SFV_OK;
}

orc_case* orc_create(const sfv_mesh_desc* md, const sfv_physics* ph, char* errbuf, int errlen) {
    orc_case* h = xcalloc(1, sizeof(orc_case));
    if (md->dim != 3) {
        if (errbuf) snprintf(errbuf, errlen, "oracle: only 3-D meshes are on the hot path");
        free(h);
        return NULL;
    }
    h->nc = md->n_cells;
    h->nf = md->n_faces;
    h->nint = md->n_internal;
    h->np = md->n_points;
    h->npatch = md->n_patches;
    h->points = xcalloc(h->np, sizeof(v3));
    for (int i = 0; i < h->np; ++i)
        h->points[i] = (v3){md->points[3 * i], md->points[3 * i + 1], md->points[3 * i + 2]};
    h->face_off = xcalloc(h->nf + 1, sizeof(int));
    memcpy(h->face_off, md->face_offsets, sizeof(int) * (h->nf + 1));
    h->face_pts = xcalloc(h->face_off[h->nf], sizeof(int));
    memcpy(h->face_pts, md->face_points, sizeof(int) * h->face_off[h->nf]);
    h->owner = xcalloc(h->nf, sizeof(int));
    h->neigh = xcalloc(h->nf, sizeof(int));
    memcpy(h->owner, md->owner, sizeof(int) * h->nf);
    memcpy(h->neigh, md->neighbour, sizeof(int) * h->nf);
    h->patch_kind = xcalloc(h->npatch, sizeof(int));
    h->patch_start = xcalloc(h->npatch, sizeof(int));
    h->patch_count = xcalloc(h->npatch, sizeof(int));
    memcpy(h->patch_kind, md->patch_kind, sizeof(int) * h->npatch);
    memcpy(h->patch_start, md->patch_start, sizeof(int) * h->npatch);
    memcpy(h->patch_count, md->patch_count, sizeof(int) * h->npatch);

    /* Mesh::finalise (mesh.cpp:29-62) */
    const char* bad = NULL;
    h->face_patch = xcalloc(h->nf, sizeof(int));
    for (int f = 0; f < h->nf; ++f) h->face_patch[f] = -1;
    for (int p = 0; p < h->npatch && !bad; ++p) {
        if (h->patch_start[p] < h->nint || h->patch_start[p] + h->patch_count[p] > h->nf)
            bad = "mesh: patch range outside boundary faces";
        for (int f = h->patch_start[p]; f < h->patch_start[p] + h->patch_count[p] && !bad; ++f) {
            if (h->face_patch[f] != -1) bad = "mesh: face in two patches";
            h->face_patch[f] = p;
        }
    }
    for (int f = 0; f < h->nf && !bad; ++f) {
        const int boundary = h->neigh[f] < 0;
        if (boundary != (f >= h->nint)) bad = "mesh: internal faces must precede boundary faces";
        else if (boundary && h->face_patch[f] == -1) bad = "mesh: boundary face not in any patch";
        else if (h->owner[f] < 0 || h->owner[f] >= h->nc || h->neigh[f] >= h->nc)
            bad = "mesh: face cell index out of range";
    }
    if (!bad) {
        h->cf_off = xcalloc(h->nc + 1, sizeof(int));
        for (int f = 0; f < h->nf; ++f) {
            ++h->cf_off[h->owner[f] + 1];
            if (h->neigh[f] >= 0) ++h->cf_off[h->neigh[f] + 1];
        }
        for (int c = 0; c < h->nc; ++c) {
            if (h->cf_off[c + 1] == 0) bad = "mesh: cell without faces";
            h->cf_off[c + 1] += h->cf_off[c];
        }
        h->cf = xcalloc(h->cf_off[h->nc], sizeof(int));
        int* fill = xcalloc(h->nc, sizeof(int));
        for (int f = 0; f < h->nf; ++f) {
            const int o = h->owner[f];
            h->cf[h->cf_off[o] + fill[o]++] = f;
            const int n = h->neigh[f];
            if (n >= 0) h->cf[h->cf_off[n] + fill[n]++] = f;
        }
        free(fill);
    }
    if (!bad && compute_geometry(h) != SFV_OK) bad = h->err.msg;
    if (bad) {
        if (errbuf) snprintf(errbuf, errlen, "%s", bad);
        orc_destroy(h);
        return NULL;
    }
    /* ResidualEvaluator ctor checks (discretisation.cpp:64-67) */
    if (!(ph->alpha > 0.0) || (ph->transient && !(ph->dt > 0.0))) {
        if (errbuf) snprintf(errbuf, errlen, "discretisation: bad alpha or dt");
        orc_destroy(h);
        return NULL;
    }
    h->law = ph->law;
    for (int k = 0; k < 8; ++k) h->gc[k] = ph->guccione[k];
    h->mu = ph->mu;
    h->lam = ph->lambda;
    h->alpha = ph->alpha;
    h->tl = ph->total_lagrangian;
    h->transient = ph->transient;
    h->dt = ph->dt;
    h->rho = ph->rho;
    h->bc_value = xcalloc(h->npatch, sizeof(v3));
    h->bc_ramp = xcalloc(h->npatch, sizeof(int));
    for (int p = 0; p < h->npatch; ++p) {
        h->bc_value[p] = (v3){ph->bc_value[3 * p], ph->bc_value[3 * p + 1], ph->bc_value[3 * p + 2]};
        h->bc_ramp[p] = ph->bc_ramp[p];
    }
    h->u_old = xcalloc(h->nc, sizeof(v3));
    h->u_old_old = xcalloc(h->nc, sizeof(v3));
    h->v_old = xcalloc(h->nc, sizeof(v3));
    h->v_old_old = xcalloc(h->nc, sizeof(v3));
    h->grad = xcalloc(h->nc, sizeof(m3));
    h->sigma = xcalloc(h->nc, sizeof(m3));
    h->fdef = xcalloc(h->nc, sizeof(m3));
    h->ja = ph->j2_curve[0];
    h->jb = ph->j2_curve[1];
    h->jc = ph->j2_curve[2];
    h->jd = ph->j2_curve[3];
    h->jn = ph->law == SFV_LAW_J2 ? ph->j2_n_table : 0;
    for (int k = 0; k < 2 * h->jn && k < 32; ++k) h->jt[k] = ph->j2_table[k];
    if (ph->law == SFV_LAW_J2) { /* J2PlasticLaw::resize (laws.cpp:196-199): PlasticCell{} */
        h->j2_bbar = xcalloc(h->nc, sizeof(m3));
        h->j2_F = xcalloc(h->nc, sizeof(m3));
        h->j2_eps = xcalloc(h->nc, sizeof(double));
        for (int c = 0; c < h->nc; ++c) h->j2_bbar[c] = h->j2_F[c] = mident();
    }
    return h;
}

static void lu_free(void* p);

void orc_destroy(orc_case* h) {
    if (!h) return;
    void* ptrs[] = {h->points, h->face_off, h->face_pts, h->owner, h->neigh, h->patch_kind,
                    h->patch_start, h->patch_count, h->face_patch, h->cf_off, h->cf, h->volume,
                    h->centroid, h->g_inv, h->g_singular, h->face_centroid, h->area, h->area_mag,
                    h->normal, h->d, h->d_mag, h->w, h->delta, h->delta_mag, h->reflect, h->ls,
                    h->bc_value, h->bc_ramp, h->u_old, h->u_old_old, h->v_old, h->v_old_old,
                    h->grad, h->sigma, h->fdef, h->j2_bbar, h->j2_F, h->j2_eps, h->body_vol, h->face_bc};
    for (size_t i = 0; i < sizeof ptrs / sizeof ptrs[0]; ++i) free(ptrs[i]);
    csr_free(&h->ilu);
    lu_free(h->lu);
    free(h);
}

const char* orc_last_error(orc_case* h) { return h->err.msg; }
int orc_n_cells(orc_case* h) { return h->nc; }

void orc_geometry(orc_case* h, double* volume, double* centroid, double* face_centroid,
                  double* area, double* d, double* d_mag, double* w, double* delta, double* g_inv,
                  signed char* g_singular, int* cf_offsets, int* cf_faces, double* ls_vec) {
    for (int c = 0; c < h->nc; ++c) {
        volume[c] = h->volume[c];
        for (int k = 0; k < 3; ++k) centroid[3 * c + k] = vget(h->centroid[c], k);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) g_inv[9 * c + 3 * i + j] = h->g_inv[c].m[i][j];
        g_singular[c] = h->g_singular[c];
    }
    for (int f = 0; f < h->nf; ++f) {
        for (int k = 0; k < 3; ++k) {
            face_centroid[3 * f + k] = vget(h->face_centroid[f], k);
            area[3 * f + k] = vget(h->area[f], k);
            d[3 * f + k] = vget(h->d[f], k);
            delta[3 * f + k] = vget(h->delta[f], k);
        }
        d_mag[f] = h->d_mag[f];
        w[f] = h->w[f];
    }
    for (int c = 0; c <= h->nc; ++c) cf_offsets[c] = h->cf_off[c];
    for (int q = 0; q < h->cf_off[h->nc]; ++q) {
        cf_faces[q] = h->cf[q];
        for (int k = 0; k < 3; ++k) ls_vec[3 * q + k] = vget(h->ls[q], k);
    }
}

void orc_set_time(orc_case* h, double t) { h->time = t; }

static void load_cells(v3* dst, const double* flat, int n) {
    for (int c = 0; c < n; ++c) dst[c] = (v3){flat[3 * c], flat[3 * c + 1], flat[3 * c + 2]};
}
static void store_cells(double* flat, const v3* src, int n) {
    for (int c = 0; c < n; ++c) {
        flat[3 * c] = src[c].x;
        flat[3 * c + 1] = src[c].y;
        flat[3 * c + 2] = src[c].z;
    }
}

void orc_set_history(orc_case* h, const double* u_old, const double* u_old_old, const double* v_old,
                     const double* v_old_old) {
    load_cells(h->u_old, u_old, h->nc);
    load_cells(h->u_old_old, u_old_old, h->nc);
    load_cells(h->v_old, v_old, h->nc);
    load_cells(h->v_old_old, v_old_old, h->nc);
}

/* ------------------------------------------------------------------ residual */

/* ResidualEvaluator::bc_value with the config-built BC (io.cpp:278-279) */
/* ResidualEvaluator::bc_value (discretisation.cpp:82-85): value(face_centroid, t) — the
   caller's sampled per-face values when given, else the patch value (times t when ramped) */
static v3 bc_value(const orc_case* h, int f) {
    if (h->face_bc) return h->face_bc[f - h->nint];
    const int p = h->face_patch[f];
    return h->bc_ramp[p] ? vscale(h->bc_value[p], h->time) : h->bc_value[p];
}

/* cell_gradients (discretisation.cpp:10-31) */
static int cell_gradients(orc_case* h, const v3* u, m3* grad) {
    for (int c = 0; c < h->nc; ++c) {
        if (h->g_singular[c])
            return fail(&h->err, SFV_ERR_GRADIENT_FAILURE, c, "cell_gradients: singular least-squares stencil");
        m3 g = mzero();
        for (int q = h->cf_off[c]; q < h->cf_off[c + 1]; ++q) {
            const int f = h->cf[q];
            v3 du;
            if (f < h->nint) {
                const int other = h->owner[f] == c ? h->neigh[f] : h->owner[f];
                du = vsub(u[other], u[c]);
            } else if (kind_of_face(h, f) == SFV_PATCH_SYMMETRY) {
                du = vsub(mvmul(h->reflect[f], u[c]), u[c]);
            } else {
                continue;
            }
            g = madd(g, outer(h->ls[q], du));
        }
        grad[c] = g;
    }
    return SFV_OK;
}

/* hooke_stress (laws.cpp:20-27) */
static m3 hooke(m3 g, double mu, double lam) {
    m3 s = mscale(madd(g, mtrans(g)), mu);
    const double t = lam * mtrace(g);
    s.m[0][0] += t; s.m[1][1] += t; s.m[2][2] += t;
    return s;
}

/* neo_hookean_stress via kinematics (laws.cpp:9-18, :39-47); returns 0 on det F <= 0 */
static int neo_hookean(m3 g, double mu, double kappa, m3* out) {
    const m3 F = madd(mident(), mtrans(g));
    const double J = mdet(F);
    if (!(J > 0.0)) return 0;
    const m3 bbar = mscale(mmul(F, mtrans(F)), pow(J, -2.0 / 3.0));
    m3 s = mscale(mdev(bbar), mu / J);
    const double p = 0.5 * kappa * (J * J - 1.0) / J;
    s.m[0][0] += p; s.m[1][1] += p; s.m[2][2] += p;
    *out = s;
    return 1;
}

/* kinematics E (laws.cpp:15): 0.5 * (G + G^T + G G^T) */
static m3 green_strain(m3 g) { return mscale(madd(madd(g, mtrans(g)), mmul(g, mtrans(g))), 0.5); }
static double mddot(m3 a, m3 b) { /* types.hpp:158-164 */
    double s = 0.0;
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) s += a.m[i][j] * b.m[i][j];
    return s;
}

/* stvk_stress (laws.cpp:29-37); returns 0 on det F <= 0 */
static int stvk(m3 g, double mu, double lam, m3* out) {
    const m3 F = madd(mident(), mtrans(g));
    const double J = mdet(F);
    if (!(J > 0.0)) return 0;
    const m3 E = green_strain(g);
    m3 S = mscale(E, 2.0 * mu);
    const double t = lam * mtrace(E);
    S.m[0][0] += t; S.m[1][1] += t; S.m[2][2] += t;
    *out = mscale(mmul(mmul(F, S), mtrans(F)), 1.0 / J);
    return 1;
}

/* guccione_stress with guccione_Q / guccione_dQ_dE (laws.cpp:49-77); gc = C, c_f, c_t, c_fs,
 * kappa, f0 xyz.  Returns 1 ok, 0 det F <= 0 (InvertedElement), -1 exponent overflow
 * (LawOverflow: Q > 500 or not finite). */
static int guccione(m3 g, const double* gc, m3* out) {
    const m3 F = madd(mident(), mtrans(g));
    const double J = mdet(F);
    if (!(J > 0.0)) return 0;
    const m3 E = green_strain(g);
    const double C = gc[0], cf = gc[1], ct = gc[2], cfs = gc[3], kappa = gc[4];
    const v3 f0 = {gc[5], gc[6], gc[7]};
    const m3 ff = outer(f0, f0);
    const double i1 = mtrace(E);
    const double i2 = 0.5 * (i1 * i1 - mtrace(mmul(E, E)));
    const double i4 = mddot(E, ff);
    const double i5 = mddot(mmul(E, E), ff);
    const double Q = ct * i1 * i1 - 2.0 * ct * i2 + (cf - 2.0 * cfs + ct) * i4 * i4 + 2.0 * (cfs - ct) * i5;
    if (Q > 500.0 || !isfinite(Q)) return -1;
    const m3 dq = madd(madd(mscale(E, 2.0 * ct), mscale(ff, 2.0 * (cf - 2.0 * cfs + ct) * i4)),
                       mscale(madd(mmul(E, ff), mmul(ff, E)), 2.0 * (cfs - ct)));
    m3 S = mscale(dq, 0.5 * C * exp(Q));
    const double pen = 0.5 * kappa * (J * J - 1.0) / J;
    S.m[0][0] += pen; S.m[1][1] += pen; S.m[2][2] += pen;
    *out = mscale(mmul(mmul(F, S), mtrans(F)), 1.0 / J);
    return 1;
}

/* HardeningCurve::value / slope (laws.cpp:79-102) */
static double hard_value(const orc_case* h, double e) {
    if (h->jn > 0) {
        if (e <= h->jt[0]) return h->jt[1];
        for (int i = 1; i < h->jn; ++i)
            if (e <= h->jt[2 * i]) {
                const double e0 = h->jt[2 * i - 2], s0 = h->jt[2 * i - 1], e1 = h->jt[2 * i], s1 = h->jt[2 * i + 1];
                return s0 + (s1 - s0) * (e - e0) / (e1 - e0);
            }
        return h->jt[2 * h->jn - 1];
    }
    return h->ja + h->jb * e + (h->jc - h->ja) * (1.0 - exp(-h->jd * e));
}
static double hard_slope(const orc_case* h, double e) {
    if (h->jn > 0) {
        if (e <= h->jt[0] || e >= h->jt[2 * h->jn - 2]) return 0.0;
        for (int i = 1; i < h->jn; ++i)
            if (e <= h->jt[2 * i]) return (h->jt[2 * i + 1] - h->jt[2 * i - 1]) / (h->jt[2 * i] - h->jt[2 * i - 2]);
        return 0.0;
    }
    return h->jb + (h->jc - h->ja) * h->jd * exp(-h->jd * e);
}
static double mfrob(m3 a) { /* types.hpp:150-155 */
    double s = 0.0;
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) s += a.m[i][j] * a.m[i][j];
    return sqrt(s);
}

/* j2_radial_return (laws.cpp:104-168) on cell c's committed state; trial state into the out
 * pointers.  Returns 1 ok, 0 det F <= 0 / inverted increment (InvertedElement), -2 hardening
 * Newton did not converge (ReturnMapFailure). */
static int j2_return(const orc_case* h, int c, m3 g, m3* sigma, m3* bbar_out, double* eps_out, m3* F_out) {
    const double mu = h->mu, kappa = h->lam;
    const m3 F_new = madd(mident(), mtrans(g));
    const double J = mdet(F_new);
    if (!(J > 0.0)) return 0;
    const m3 f_rel = mmul(F_new, minverse(h->j2_F[c]));
    const double det_f = mdet(f_rel);
    if (!(det_f > 0.0)) return 0;
    const m3 f_bar = mscale(f_rel, pow(det_f, -1.0 / 3.0));
    const m3 bt0 = mmul(mmul(f_bar, h->j2_bbar[c]), mtrans(f_bar));
    const m3 b_trial = mscale(madd(bt0, mtrans(bt0)), 0.5);
    const m3 s_trial = mscale(mdev(b_trial), mu / J);
    const double s_norm = mfrob(s_trial);
    const double sq23 = sqrt(2.0 / 3.0);
    const double epc = h->j2_eps[c];
    const double f_yield = s_norm - sq23 * hard_value(h, epc);
    m3 s = s_trial;
    m3 bnew = b_trial;
    double epn = epc;
    if (!(f_yield <= 0.0)) {
        const double mu_bar = mu * mtrace(b_trial) / (3.0 * J);
        double dg = 0.0;
        int done = 0;
        const double tol = 1e-12 * fmax(s_norm, hard_value(h, 0.0));
        for (int it = 0; it < 50; ++it) {
            const double eps = epc + sq23 * dg;
            const double gg = s_norm - 2.0 * mu_bar * dg - sq23 * hard_value(h, eps);
            if (fabs(gg) <= tol) {
                done = 1;
                break;
            }
            const double gp = -2.0 * mu_bar - (2.0 / 3.0) * hard_slope(h, eps);
            const double next = dg - gg / gp;
            dg = next > 0.0 ? next : 0.5 * dg;
        }
        if (!done) return -2;
        const m3 n_dir = mscale(s_trial, 1.0 / s_norm);
        s = msub(s_trial, mscale(n_dir, 2.0 * mu_bar * dg));
        epn = epc + sq23 * dg;
        bnew = mscale(s, J / mu);
        const double iso = mtrace(b_trial) / 3.0;
        bnew.m[0][0] += iso; bnew.m[1][1] += iso; bnew.m[2][2] += iso;
    }
    if (bbar_out) *bbar_out = bnew;
    if (eps_out) *eps_out = epn;
    if (F_out) *F_out = F_new;
    const double p = 0.5 * kappa * (J * J - 1.0) / J;
    s.m[0][0] += p; s.m[1][1] += p; s.m[2][2] += p;
    *sigma = s;
    return 1;
}

/* rhie_chow_face (discretisation.cpp:33-37) */
static v3 rhie_chow(v3 up, v3 uo, m3 gf, v3 delta, double d_mag, double area_mag, double alpha,
                    double kbar) {
    const v3 compact = vscale(vsub(uo, up), vnorm(delta) / d_mag);
    return vscale(vsub(compact, dot_left(delta, gf)), alpha * kbar * area_mag);
}

/* transform_area (discretisation.cpp:100-104); returns 0 when det <= 0 */
static int transform_area(v3 gamma, m3 ff, v3* out) {
    const double j = mdet(ff);
    if (!(j > 0.0)) return 0;
    *out = vscale(dot_left(gamma, minverse(ff)), j);
    return 1;
}

static double kbar_of(const orc_case* h) { /* laws.hpp:100, :111, :122, :133, :147 */
    if (h->law == SFV_LAW_NEO_HOOKEAN || h->law == SFV_LAW_J2) return 4.0 / 3.0 * h->mu + h->lam;
    if (h->law == SFV_LAW_GUCCIONE) return 4.0 / 3.0 * (h->gc[0] * h->gc[2]) + h->gc[4];
    return 2.0 * h->mu + h->lam;
}

/* add_stabilisation (discretisation.cpp:176-208) */
static void add_stabilisation(orc_case* h, const v3* u, const m3* grad, v3* r) {
    const double kb = kbar_of(h);
    for (int f = 0; f < h->nf; ++f) {
        const int p = h->owner[f];
        if (f < h->nint) {
            const int n = h->neigh[f];
            const m3 gf = interp(grad[p], grad[n], h->w[f]);
            const v3 dp = rhie_chow(u[p], u[n], gf, h->delta[f], h->d_mag[f], h->area_mag[f], h->alpha, kb);
            r[p] = vadd(r[p], dp);
            r[n] = vsub(r[n], dp);
            continue;
        }
        const int k = kind_of_face(h, f);
        if (k == SFV_PATCH_DISPLACEMENT) {
            r[p] = vadd(r[p], rhie_chow(u[p], bc_value(h, f), grad[p], h->delta[f], h->d_mag[f],
                                        h->area_mag[f], h->alpha, kb));
        } else if (k == SFV_PATCH_SYMMETRY) {
            const m3 refl = h->reflect[f];
            const v3 um = mvmul(refl, u[p]);
            const m3 gs = mscale(madd(grad[p], mmul(mmul(refl, grad[p]), refl)), 0.5);
            r[p] = vadd(r[p], rhie_chow(u[p], um, gs, h->delta[f], h->d_mag[f], h->area_mag[f], h->alpha, kb));
        }
    }
}

/* bdf2_velocity / bdf2_acceleration (discretisation.cpp:48-57) */
static v3 bdf2_vel(v3 un, v3 ut, v3 utm1, double dt) {
    return vdiv(vadd(vsub(vscale(un, 3.0), vscale(ut, 4.0)), utm1), 2.0 * dt);
}
static v3 bdf2_acc(v3 un, v3 ut, v3 utm1, v3 vt, v3 vtm1, double dt) {
    const v3 vn = bdf2_vel(un, ut, utm1, dt);
    return vdiv(vadd(vsub(vscale(vn, 3.0), vscale(vt, 4.0)), vtm1), 2.0 * dt);
}

/* ResidualEvaluator::residual (discretisation.cpp:108-174) */
static int residual(orc_case* h, const v3* u, v3* r) {
    const int nc = h->nc;
    int rc = cell_gradients(h, u, h->grad);
    if (rc) return rc;
    for (int c = 0; c < nc; ++c) {
        if (h->law == SFV_LAW_NEO_HOOKEAN) {
            if (!neo_hookean(h->grad[c], h->mu, h->lam, &h->sigma[c]))
                return fail(&h->err, SFV_ERR_INVERTED_ELEMENT, c, "kinematics: det F <= 0");
        } else if (h->law == SFV_LAW_STVK) {
            if (!stvk(h->grad[c], h->mu, h->lam, &h->sigma[c]))
                return fail(&h->err, SFV_ERR_INVERTED_ELEMENT, c, "kinematics: det F <= 0");
        } else if (h->law == SFV_LAW_J2) {
            const int k = j2_return(h, c, h->grad[c], &h->sigma[c], NULL, NULL, NULL);
            if (k == 0) return fail(&h->err, SFV_ERR_INVERTED_ELEMENT, c, "j2_radial_return: det F <= 0");
            if (k < 0) return fail(&h->err, SFV_ERR_RETURN_MAP, c, "j2_radial_return: hardening Newton did not converge");
        } else if (h->law == SFV_LAW_GUCCIONE) {
            const int k = guccione(h->grad[c], h->gc, &h->sigma[c]);
            if (k == 0) return fail(&h->err, SFV_ERR_INVERTED_ELEMENT, c, "kinematics: det F <= 0");
            if (k < 0) return fail(&h->err, SFV_ERR_LAW_OVERFLOW, c, "guccione_stress: exponent overflow");
        } else {
            h->sigma[c] = hooke(h->grad[c], h->mu, h->lam);
        }
    }
    if (h->tl)
        for (int c = 0; c < nc; ++c) h->fdef[c] = madd(mident(), mtrans(h->grad[c]));
    for (int c = 0; c < nc; ++c) r[c] = (v3){0, 0, 0};
    for (int f = 0; f < h->nf; ++f) {
        const int p = h->owner[f];
        if (f < h->nint) {
            const int n = h->neigh[f];
            const double w = h->w[f];
            v3 gamma = h->area[f];
            if (h->tl && !transform_area(gamma, interp(h->fdef[p], h->fdef[n], w), &gamma))
                return fail(&h->err, SFV_ERR_INVERTED_ELEMENT, p, "face deformation gradient is not invertible");
            const v3 flux = dot_left(gamma, interp(h->sigma[p], h->sigma[n], w));
            r[p] = vadd(r[p], flux);
            r[n] = vsub(r[n], flux);
            continue;
        }
        const int k = kind_of_face(h, f);
        if (k == SFV_PATCH_DISPLACEMENT) {
            v3 gamma = h->area[f];
            if (h->tl && !transform_area(gamma, h->fdef[p], &gamma))
                return fail(&h->err, SFV_ERR_INVERTED_ELEMENT, p, "face deformation gradient is not invertible");
            r[p] = vadd(r[p], dot_left(gamma, h->sigma[p]));
        } else if (k == SFV_PATCH_SYMMETRY) {
            const m3 refl = h->reflect[f];
            const m3 sig_s = mscale(madd(h->sigma[p], mmul(mmul(refl, h->sigma[p]), refl)), 0.5);
            v3 gamma = h->area[f];
            if (h->tl) {
                const m3 fs = mscale(madd(h->fdef[p], mmul(mmul(refl, h->fdef[p]), refl)), 0.5);
                if (!transform_area(gamma, fs, &gamma))
                    return fail(&h->err, SFV_ERR_INVERTED_ELEMENT, p, "face deformation gradient is not invertible");
            }
            r[p] = vadd(r[p], dot_left(gamma, sig_s));
        } else {
            r[p] = vadd(r[p], vscale(bc_value(h, f), h->area_mag[f]));
        }
    }
    add_stabilisation(h, u, h->grad, r);
    if (h->body_vol) /* discretisation.cpp:160-161 */
        for (int c = 0; c < nc; ++c) r[c] = vadd(r[c], h->body_vol[c]);
    if (h->transient)
        for (int c = 0; c < nc; ++c) {
            const v3 a = bdf2_acc(u[c], h->u_old[c], h->u_old_old[c], h->v_old[c], h->v_old_old[c], h->dt);
            r[c] = vsub(r[c], vscale(a, h->rho * h->volume[c]));
        }
    for (int c = 0; c < nc; ++c)
        if (!vfinite(r[c])) return fail(&h->err, SFV_ERR_RESIDUAL_NAN, c, "residual: non-finite entry");
    return SFV_OK;
}

int orc_residual(orc_case* h, const double* uf, double* rf, int* cell) {
    v3* u = xcalloc(h->nc, sizeof(v3));
    v3* r = xcalloc(h->nc, sizeof(v3));
    load_cells(u, uf, h->nc);
    h->err.code = 0;
    h->err.cell = -1;
    const int rc = residual(h, u, r);
    if (!rc) store_cells(rf, r, h->nc);
    if (cell) *cell = rc ? h->err.cell : -1;
    free(u);
    free(r);
    return rc;
}

/* ResidualEvaluator::commit (discretisation.cpp:91-95) with J2PlasticLaw::commit (laws.cpp:214):
 * the stress at u in every cell (in cell order: the first failure aborts, nothing committed),
 * then every trial state becomes the committed one */
static int commit_state(orc_case* h, const v3* u) {
    if (h->law != SFV_LAW_J2) return SFV_OK;
    int rc = cell_gradients(h, u, h->grad);
    if (rc) return rc;
    m3* nb = xcalloc(h->nc, sizeof(m3));
    m3* nf = xcalloc(h->nc, sizeof(m3));
    double* ne = xcalloc(h->nc, sizeof(double));
    for (int c = 0; c < h->nc && !rc; ++c) {
        m3 sig;
        const int k = j2_return(h, c, h->grad[c], &sig, &nb[c], &ne[c], &nf[c]);
        if (k == 0) rc = fail(&h->err, SFV_ERR_INVERTED_ELEMENT, c, "j2_radial_return: det F <= 0");
        if (k < 0) rc = fail(&h->err, SFV_ERR_RETURN_MAP, c, "j2_radial_return: hardening Newton did not converge");
    }
    if (!rc) {
        memcpy(h->j2_bbar, nb, sizeof(m3) * h->nc);
        memcpy(h->j2_F, nf, sizeof(m3) * h->nc);
        memcpy(h->j2_eps, ne, sizeof(double) * h->nc);
    }
    free(nb);
    free(nf);
    free(ne);
    return rc;
}

int orc_commit(orc_case* h, const double* uf) {
    v3* u = xcalloc(h->nc, sizeof(v3));
    load_cells(u, uf, h->nc);
    h->err.code = 0;
    h->err.cell = -1;
    const int rc = commit_state(h, u);
    free(u);
    return rc;
}

int orc_law_state(orc_case* h, double* out) {
    if (h->law != SFV_LAW_J2) return fail(&h->err, SFV_ERR_INVALID_ARGUMENT, -1, "law_state: J2 only");
    for (int c = 0; c < h->nc; ++c) {
        for (int q = 0; q < 9; ++q) {
            out[19 * (size_t)c + q] = h->j2_bbar[c].m[q / 3][q % 3];
            out[19 * (size_t)c + 10 + q] = h->j2_F[c].m[q / 3][q % 3];
        }
        out[19 * (size_t)c + 9] = h->j2_eps[c];
    }
    return SFV_OK;
}

int orc_stabilisation(orc_case* h, const double* uf, double* rf, int* cell) {
    v3* u = xcalloc(h->nc, sizeof(v3));
    v3* r = xcalloc(h->nc, sizeof(v3));
    load_cells(u, uf, h->nc);
    int rc = cell_gradients(h, u, h->grad);
    if (!rc) {
        add_stabilisation(h, u, h->grad, r);
        store_cells(rf, r, h->nc);
    }
    if (cell) *cell = rc ? h->err.cell : -1;
    free(u);
    free(r);
    return rc;
}

/* ------------------------------------------------------------------ J.v */

static double vec_norm(const double* v, int n) { /* nonlinear.cpp:13-17 */
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += v[i] * v[i];
    return sqrt(s);
}

/* jacobian_vector_product (nonlinear.cpp:105-138); u, r_u, v, out interleaved 3n */
static int jv(orc_case* h, const double* u, const double* r_u, const double* v, double* out,
              v3* up_scratch, v3* r_scratch) {
    const int n = 3 * h->nc;
    const double v_norm = vec_norm(v, n);
    if (v_norm == 0.0) {
        memset(out, 0, sizeof(double) * n);
        return SFV_OK;
    }
    const double u_norm = vec_norm(u, n); /* field_norm over dim=3 comps, same order */
    const double eps = sqrt(DBL_EPSILON) * sqrt(1.0 + u_norm) / v_norm;
    for (int c = 0; c < h->nc; ++c)
        up_scratch[c] = (v3){u[3 * c] + eps * v[3 * c], u[3 * c + 1] + eps * v[3 * c + 1],
                             u[3 * c + 2] + eps * v[3 * c + 2]};
    const int rc = residual(h, up_scratch, r_scratch);
    if (rc == SFV_ERR_RESIDUAL_NAN || rc == SFV_ERR_INVERTED_ELEMENT || rc == SFV_ERR_LAW_OVERFLOW) {
        char msg[SFV_DETAIL_LEN];
        snprintf(msg, sizeof msg, "jvp: %s", h->err.msg);
        return fail(&h->err, SFV_ERR_JVP_NAN, -1, msg);
    }
    if (rc) return rc;
    for (int c = 0; c < h->nc; ++c)
        for (int k = 0; k < 3; ++k) {
            const int i = 3 * c + k;
            out[i] = (vget(r_scratch[c], k) - r_u[i]) / eps;
            if (!isfinite(out[i])) return fail(&h->err, SFV_ERR_JVP_NAN, -1, "jvp: non-finite difference quotient");
        }
    return SFV_OK;
}

int orc_jv(orc_case* h, const double* u, const double* r_u, const double* v, double* out, int* cell) {
    v3* a = xcalloc(h->nc, sizeof(v3));
    v3* b = xcalloc(h->nc, sizeof(v3));
    h->err.cell = -1;
    const int rc = jv(h, u, r_u, v, out, a, b);
    if (cell) *cell = rc ? h->err.cell : -1;
    free(a);
    free(b);
    return rc;
}

double orc_time_jv(orc_case* h, const double* u, const double* r_u, const double* v, int reps) {
    const int n = 3 * h->nc;
    v3* a = xcalloc(h->nc, sizeof(v3));
    v3* b = xcalloc(h->nc, sizeof(v3));
    double* out = xcalloc(n, sizeof(double));
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (int r = 0; r < reps; ++r) jv(h, u, r_u, v, out, a, b);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    free(a);
    free(b);
    free(out);
    return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}

/* ------------------------------------------------------------------ approximate Jacobian */

/* assemble_approximate_jacobian (discretisation.cpp:216-262) followed by
 * BlockSparseMatrix::expand_scalar (linalg.cpp:135-158): the 3n x 3n scalar CSR with
 * every block entry kept, explicit zeros included. */
static m3* block_jacobian(const orc_case* h, int** rp_out, int** col_out) {
    const int nc = h->nc;
    int* rp = xcalloc(nc + 1, sizeof(int));
    for (int c = 0; c < nc; ++c) rp[c + 1] = 1;
    for (int f = 0; f < h->nint; ++f) {
        ++rp[h->owner[f] + 1];
        ++rp[h->neigh[f] + 1];
    }
    for (int c = 0; c < nc; ++c) rp[c + 1] += rp[c];
    int* col = xcalloc(rp[nc], sizeof(int));
    int* fill = xcalloc(nc, sizeof(int));
    for (int c = 0; c < nc; ++c) col[rp[c] + fill[c]++] = c;
    for (int f = 0; f < h->nint; ++f) {
        const int o = h->owner[f], n = h->neigh[f];
        col[rp[o] + fill[o]++] = n;
        col[rp[n] + fill[n]++] = o;
    }
    for (int c = 0; c < nc; ++c) /* insertion sort per row (std::sort, distinct keys) */
        for (int i = rp[c] + 1; i < rp[c + 1]; ++i) {
            const int key = col[i];
            int j = i - 1;
            while (j >= rp[c] && col[j] > key) { col[j + 1] = col[j]; --j; }
            col[j + 1] = key;
        }
    m3* blocks = xcalloc(rp[nc], sizeof(m3));
    const double kbar = kbar_of(h);
    for (int f = 0; f < h->nf; ++f) {
        const double coeff = kbar * h->delta_mag[f] / h->d_mag[f] * h->area_mag[f];
        const int p = h->owner[f];
        const m3 ci = mscale(mident(), coeff);
        const m3 mci = mscale(mident(), -coeff);
        if (f < h->nint) {
            const int n = h->neigh[f];
            int q;
            for (q = rp[p]; col[q] != n; ++q) {}
            blocks[q] = madd(blocks[q], ci);
            for (q = rp[n]; col[q] != p; ++q) {}
            blocks[q] = madd(blocks[q], ci);
            for (q = rp[p]; col[q] != p; ++q) {}
            blocks[q] = madd(blocks[q], mci);
            for (q = rp[n]; col[q] != n; ++q) {}
            blocks[q] = madd(blocks[q], mci);
        } else if (kind_of_face(h, f) == SFV_PATCH_DISPLACEMENT) {
            int q;
            for (q = rp[p]; col[q] != p; ++q) {}
            blocks[q] = madd(blocks[q], mci);
        } else if (kind_of_face(h, f) == SFV_PATCH_SYMMETRY) {
            int q;
            for (q = rp[p]; col[q] != p; ++q) {}
            blocks[q] = madd(blocks[q], mscale(outer(h->normal[f], h->normal[f]), -coeff));
        }
    }
    if (h->transient)
        for (int c = 0; c < nc; ++c) {
            int q;
            for (q = rp[c]; col[q] != c; ++q) {}
            blocks[q] = madd(blocks[q], mscale(mident(), -2.25 * h->rho * h->volume[c] / (h->dt * h->dt)));
        }
    free(fill);
    *rp_out = rp;
    *col_out = col;
    return blocks;
}

static csr expanded_jacobian(const orc_case* h) {
    const int nc = h->nc;
    int *rp, *col;
    m3* blocks = block_jacobian(h, &rp, &col);
    csr m;
    m.n = 3 * nc;
    m.row_ptr = xcalloc(m.n + 1, sizeof(int));
    for (int i = 0; i < nc; ++i)
        for (int a = 0; a < 3; ++a) m.row_ptr[3 * i + a + 1] = (rp[i + 1] - rp[i]) * 3;
    for (int r = 0; r < m.n; ++r) m.row_ptr[r + 1] += m.row_ptr[r];
    m.nnz = m.row_ptr[m.n];
    m.col = xcalloc(m.nnz, sizeof(int));
    m.val = xcalloc(m.nnz, sizeof(double));
    for (int i = 0; i < nc; ++i)
        for (int a = 0; a < 3; ++a) {
            int q = m.row_ptr[3 * i + a];
            for (int p = rp[i]; p < rp[i + 1]; ++p)
                for (int b = 0; b < 3; ++b, ++q) {
                    m.col[q] = col[p] * 3 + b;
                    m.val[q] = blocks[p].m[a][b];
                }
        }
    free(rp);
    free(col);
    free(blocks);
    return m;
}

/* BlockSparseMatrix::scalar_component (linalg.cpp:114-133) for c = 0..2, negated (A = -J~,
 * nonlinear.cpp:278-281); 0, or -1 when a block is not diagonal (InvalidArgument) */
static int negated_components(const orc_case* h, csr comps[3]) {
    const int nc = h->nc;
    int *rp, *col;
    m3* blocks = block_jacobian(h, &rp, &col);
    double scale = 0.0;
    for (int p = 0; p < rp[nc]; ++p)
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) scale = fmax(scale, fabs(blocks[p].m[a][b]));
    int rc = 0;
    for (int p = 0; p < rp[nc] && !rc; ++p)
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
                if (a != b && fabs(blocks[p].m[a][b]) > 1e-12 * scale) rc = -1;
    for (int c = 0; c < 3; ++c) {
        comps[c].n = nc;
        comps[c].nnz = rp[nc];
        comps[c].row_ptr = xcalloc(nc + 1, sizeof(int));
        memcpy(comps[c].row_ptr, rp, sizeof(int) * (nc + 1));
        comps[c].col = xcalloc(rp[nc] > 0 ? rp[nc] : 1, sizeof(int));
        memcpy(comps[c].col, col, sizeof(int) * rp[nc]);
        comps[c].val = xcalloc(rp[nc] > 0 ? rp[nc] : 1, sizeof(double));
        for (int p = 0; p < rp[nc]; ++p) comps[c].val[p] = -blocks[p].m[c][c];
    }
    free(rp);
    free(col);
    free(blocks);
    return rc;
}

/* ------------------------------------------------------------------ ILU(k) */

/* IlukPrecond ctor (linalg.cpp:251-300).  Symbolic: level-of-fill row merge in
 * ascending column order, rows of already-processed k read from their final
 * pattern; numeric: IKJ on the fixed pattern. */
static int ilu_factor(const csr* a, int level, csr* out, orc_err* err) {
    const int n = a->n;
    int* rp = xcalloc(n + 1, sizeof(int));
    int cap = a->nnz * 2 + n;
    int* cols = xcalloc(cap, sizeof(int));
    int* levs = xcalloc(cap, sizeof(int));
    int* pos = xcalloc(n, sizeof(int)); /* marker: position+1 in the working row */
    int* wcol = xcalloc(n, sizeof(int));
    int* wlev = xcalloc(n, sizeof(int));
    for (int i = 0; i < n; ++i) {
        int len = 0;
        /* working row: sorted by column, built from A's row + diagonal */
        for (int p = a->row_ptr[i]; p < a->row_ptr[i + 1]; ++p) {
            const int j = a->col[p];
            if (pos[j]) { wlev[pos[j] - 1] = 0; continue; }
            wcol[len] = j; wlev[len] = 0; pos[j] = ++len;
        }
        if (!pos[i]) { wcol[len] = i; wlev[len] = 0; pos[i] = ++len; }
        /* sort (insertion) and re-mark */
        for (int x = 1; x < len; ++x) {
            const int cj = wcol[x], lj = wlev[x];
            int y = x - 1;
            while (y >= 0 && wcol[y] > cj) { wcol[y + 1] = wcol[y]; wlev[y + 1] = wlev[y]; --y; }
            wcol[y + 1] = cj; wlev[y + 1] = lj;
        }
        for (int x = 0; x < len; ++x) pos[wcol[x]] = x + 1;
        for (int it = 0; it < len && wcol[it] < i; ++it) {
            const int k = wcol[it], lev_ik = wlev[it];
            if (lev_ik >= level) continue;
            for (int q = rp[k]; q < rp[k + 1]; ++q) {
                const int j = cols[q];
                if (j <= k) continue;
                const int lev = lev_ik + levs[q] + 1;
                if (lev > level) continue;
                if (pos[j]) {
                    if (wlev[pos[j] - 1] > lev) wlev[pos[j] - 1] = lev;
                } else { /* sorted insert; j > k so it lands after position it */
                    int y = len - 1;
                    while (y >= 0 && wcol[y] > j) { wcol[y + 1] = wcol[y]; wlev[y + 1] = wlev[y]; pos[wcol[y + 1]] = y + 2; --y; }
                    wcol[y + 1] = j; wlev[y + 1] = lev; pos[j] = y + 2;
                    ++len;
                }
            }
        }
        if (rp[i] + len > cap) {
            cap = (rp[i] + len) * 2;
            cols = realloc(cols, sizeof(int) * cap);
            levs = realloc(levs, sizeof(int) * cap);
        }
        for (int x = 0; x < len; ++x) {
            cols[rp[i] + x] = wcol[x];
            levs[rp[i] + x] = wlev[x];
            pos[wcol[x]] = 0;
        }
        rp[i + 1] = rp[i] + len;
    }
    free(levs);
    free(wcol);
    free(wlev);
    out->n = n;
    out->nnz = rp[n];
    out->row_ptr = rp;
    out->col = cols;
    out->val = xcalloc(rp[n], sizeof(double));
    /* scatter A's values */
    for (int i = 0; i < n; ++i) {
        for (int q = rp[i]; q < rp[i + 1]; ++q) pos[cols[q]] = q + 1;
        for (int p = a->row_ptr[i]; p < a->row_ptr[i + 1]; ++p) out->val[pos[a->col[p]] - 1] = a->val[p];
        for (int q = rp[i]; q < rp[i + 1]; ++q) pos[cols[q]] = 0;
    }
    /* diagonal positions */
    int* diag = xcalloc(n, sizeof(int));
    for (int i = 0; i < n; ++i)
        for (int q = rp[i]; q < rp[i + 1]; ++q)
            if (cols[q] == i) diag[i] = q;
    double* val = out->val;
    int rc = SFV_OK;
    for (int i = 0; i < n && !rc; ++i) {
        for (int q = rp[i]; q < rp[i + 1]; ++q) pos[cols[q]] = q + 1;
        for (int p = rp[i]; p < rp[i + 1] && cols[p] < i; ++p) {
            const int k = cols[p];
            const double pivot = val[diag[k]];
            if (pivot == 0.0 || !isfinite(pivot)) {
                char msg[64];
                snprintf(msg, sizeof msg, "ilu: zero pivot in row %d", k);
                rc = fail(err, SFV_ERR_ILU_BREAKDOWN, -1, msg);
                break;
            }
            const double lik = (val[p] /= pivot);
            for (int q = rp[k]; q < rp[k + 1]; ++q) {
                if (cols[q] <= k) continue;
                if (pos[cols[q]]) val[pos[cols[q]] - 1] -= lik * val[q];
            }
        }
        for (int q = rp[i]; q < rp[i + 1]; ++q) pos[cols[q]] = 0;
        if (rc) break;
        const double d = val[diag[i]];
        if (d == 0.0 || !isfinite(d)) {
            char msg[64];
            snprintf(msg, sizeof msg, "ilu: zero pivot in row %d", i);
            rc = fail(err, SFV_ERR_ILU_BREAKDOWN, -1, msg);
        }
    }
    free(diag);
    free(pos);
    if (rc) csr_free(out);
    return rc;
}

/* IlukPrecond::solve (linalg.cpp:302-316) */
static void ilu_solve(const csr* m, const double* r, double* z) {
    const int n = m->n;
    memcpy(z, r, sizeof(double) * n);
    for (int i = 0; i < n; ++i)
        for (int p = m->row_ptr[i]; p < m->row_ptr[i + 1] && m->col[p] < i; ++p)
            z[i] -= m->val[p] * z[m->col[p]];
    for (int i = n - 1; i >= 0; --i) {
        double diag = 0.0;
        for (int p = m->row_ptr[i + 1] - 1; p >= m->row_ptr[i] && m->col[p] >= i; --p) {
            if (m->col[p] == i) diag = m->val[p];
            else z[i] -= m->val[p] * z[m->col[p]];
        }
        z[i] /= diag;
    }
}

/* ------------------------------------------------------------------ exact LU */

/* Exact sparse solve standing in for Eigen::SparseLU (linalg.cpp:336-359; Eigen is
 * absent): reverse Cuthill-McKee on the nonzero pattern, then banded
 * Gaussian elimination with partial pivoting. */
typedef struct {
    int n, kl, ku, w;
    double* ab;
    int *rowend, *piv, *perm;
} band_lu;

static void lu_free(void* p) {
    band_lu* b = p;
    if (!b) return;
    free(b->ab); free(b->rowend); free(b->piv); free(b->perm);
    free(b);
}

static int* rcm_order(int n, const int* adj_off, const int* adj) {
    int* order = xcalloc(n, sizeof(int));
    char* seen = xcalloc(n, 1);
    int* level = xcalloc(n, sizeof(int));
    int* q = xcalloc(n, sizeof(int));
    int* by_deg = xcalloc(n, sizeof(int));
    for (int i = 0; i < n; ++i) { by_deg[i] = i; level[i] = -1; }
    /* stable counting sort by degree */
    int maxd = 0;
    for (int i = 0; i < n; ++i) if (adj_off[i + 1] - adj_off[i] > maxd) maxd = adj_off[i + 1] - adj_off[i];
    int* dc = xcalloc(maxd + 2, sizeof(int));
    for (int i = 0; i < n; ++i) ++dc[adj_off[i + 1] - adj_off[i] + 1];
    for (int d = 0; d <= maxd; ++d) dc[d + 1] += dc[d];
    for (int i = 0; i < n; ++i) by_deg[dc[adj_off[i + 1] - adj_off[i]]++] = i;
    free(dc);
    int len = 0;
    for (int s = 0; s < n; ++s) {
        int start = by_deg[s];
        if (seen[start]) continue;
        for (int pass = 0; pass < 4; ++pass) {
            int qh = 0, qt = 0, far = start;
            q[qt++] = start;
            level[start] = 0;
            while (qh < qt) {
                const int u = q[qh++];
                for (int e = adj_off[u]; e < adj_off[u + 1]; ++e) {
                    const int v = adj[e];
                    if (level[v] >= 0) continue;
                    level[v] = level[u] + 1;
                    q[qt++] = v;
                    const int dv = adj_off[v + 1] - adj_off[v], df = adj_off[far + 1] - adj_off[far];
                    if (level[v] > level[far] || (level[v] == level[far] && dv < df)) far = v;
                }
            }
            for (int t = 0; t < qt; ++t) level[q[t]] = -1;
            if (far == start) break;
            start = far;
        }
        const int base = len;
        order[len++] = start;
        seen[start] = 1;
        for (int hh = base; hh < len; ++hh) {
            const int u = order[hh];
            const int first = len;
            for (int e = adj_off[u]; e < adj_off[u + 1]; ++e)
                if (!seen[adj[e]]) { seen[adj[e]] = 1; order[len++] = adj[e]; }
            for (int x = first + 1; x < len; ++x) { /* stable insertion sort by degree */
                const int v = order[x], dv = adj_off[v + 1] - adj_off[v];
                int y = x - 1;
                while (y >= first && adj_off[order[y] + 1] - adj_off[order[y]] > dv) { order[y + 1] = order[y]; --y; }
                order[y + 1] = v;
            }
        }
    }
    for (int i = 0; i < n / 2; ++i) { const int t = order[i]; order[i] = order[n - 1 - i]; order[n - 1 - i] = t; }
    free(seen); free(level); free(q); free(by_deg);
    return order;
}

static int lu_factor(const csr* a, band_lu** out, orc_err* err) {
    const int n = a->n;
    int* deg = xcalloc(n + 1, sizeof(int));
    for (int i = 0; i < n; ++i)
        for (int p = a->row_ptr[i]; p < a->row_ptr[i + 1]; ++p)
            if (a->col[p] != i && a->val[p] != 0.0) { ++deg[i + 1]; ++deg[a->col[p] + 1]; }
    for (int i = 0; i < n; ++i) deg[i + 1] += deg[i];
    int* adj = xcalloc(deg[n], sizeof(int));
    int* fill = xcalloc(n, sizeof(int));
    for (int i = 0; i < n; ++i)
        for (int p = a->row_ptr[i]; p < a->row_ptr[i + 1]; ++p) {
            const int j = a->col[p];
            if (j == i || a->val[p] == 0.0) continue;
            adj[deg[i] + fill[i]++] = j;
            adj[deg[j] + fill[j]++] = i;
        }
    free(fill);
    /* sorted, de-duplicated adjacency (the symmetric pattern lists each edge twice) */
    {
        int w = 0;
        for (int i = 0; i < n; ++i) {
            const int b0 = deg[i], e0 = deg[i + 1];
            for (int x = b0 + 1; x < e0; ++x) {
                const int key = adj[x];
                int y = x - 1;
                while (y >= b0 && adj[y] > key) { adj[y + 1] = adj[y]; --y; }
                adj[y + 1] = key;
            }
            deg[i] = w;
            for (int x = b0; x < e0; ++x)
                if (x == b0 || adj[x] != adj[x - 1]) adj[w++] = adj[x];
        }
        deg[n] = w;
    }
    band_lu* b = xcalloc(1, sizeof(band_lu));
    b->n = n;
    b->perm = rcm_order(n, deg, adj);
    free(deg);
    free(adj);
    int* inv = xcalloc(n, sizeof(int));
    for (int i = 0; i < n; ++i) inv[b->perm[i]] = i;
    for (int i = 0; i < n; ++i)
        for (int p = a->row_ptr[i]; p < a->row_ptr[i + 1]; ++p) {
            if (a->val[p] == 0.0) continue;
            const int bi = inv[i], bj = inv[a->col[p]];
            if (bi - bj > b->kl) b->kl = bi - bj;
            if (bj - bi > b->ku) b->ku = bj - bi;
        }
    b->w = 2 * b->kl + b->ku + 1;
    b->ab = xcalloc((size_t)n * b->w, sizeof(double));
    b->rowend = xcalloc(n, sizeof(int));
    b->piv = xcalloc(n, sizeof(int));
#define AT(i, j) b->ab[(size_t)(i) * b->w + ((j) - (i) + b->kl)]
    for (int i = 0; i < n; ++i) b->rowend[i] = i;
    for (int i = 0; i < n; ++i)
        for (int p = a->row_ptr[i]; p < a->row_ptr[i + 1]; ++p) {
            if (a->val[p] == 0.0) continue;
            const int bi = inv[i], bj = inv[a->col[p]];
            AT(bi, bj) += a->val[p];
            if (bj > b->rowend[bi]) b->rowend[bi] = bj;
        }
    free(inv);
    for (int k = 0; k < n; ++k) {
        const int last = k + b->kl < n - 1 ? k + b->kl : n - 1;
        int p = k;
        double best = fabs(AT(k, k));
        for (int i = k + 1; i <= last; ++i)
            if (fabs(AT(i, k)) > best) { best = fabs(AT(i, k)); p = i; }
        if (!(best > 0.0) || !isfinite(best)) {
            lu_free(b);
            return fail(err, SFV_ERR_LU_SINGULAR, -1, "lu: factorisation failed");
        }
        b->piv[k] = p;
        if (p != k) {
            const int end = b->rowend[k] > b->rowend[p] ? b->rowend[k] : b->rowend[p];
            for (int j = k; j <= end; ++j) { const double t = AT(k, j); AT(k, j) = AT(p, j); AT(p, j) = t; }
            b->rowend[k] = b->rowend[p] = end;
        }
        const double pivot = AT(k, k);
        const int uend = b->rowend[k];
        for (int i = k + 1; i <= last; ++i) {
            if (AT(i, k) == 0.0) continue;
            const double l = (AT(i, k) /= pivot);
            for (int j = k + 1; j <= uend; ++j) AT(i, j) -= l * AT(k, j);
            if (uend > b->rowend[i]) b->rowend[i] = uend;
        }
    }
    *out = b;
    return SFV_OK;
}

static void lu_solve(const band_lu* b, const double* r, double* z) {
    const int n = b->n;
    double* c = xcalloc(n, sizeof(double));
    for (int i = 0; i < n; ++i) c[i] = r[b->perm[i]];
    for (int k = 0; k < n; ++k) {
        if (b->piv[k] != k) { const double t = c[k]; c[k] = c[b->piv[k]]; c[b->piv[k]] = t; }
        const int last = k + b->kl < n - 1 ? k + b->kl : n - 1;
        for (int i = k + 1; i <= last; ++i) {
            const double l = AT(i, k);
            if (l != 0.0) c[i] -= l * c[k];
        }
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = c[i];
        for (int j = i + 1; j <= b->rowend[i]; ++j) s -= AT(i, j) * c[j];
        c[i] = s / AT(i, i);
    }
    for (int i = 0; i < n; ++i) z[b->perm[i]] = c[i];
    free(c);
#undef AT
}

/* make_preconditioner (nonlinear.cpp:353-380) on expand_scalar(J~) */
int orc_precond_create(orc_case* h, int kind) {
    csr_free(&h->ilu);
    lu_free(h->lu);
    h->lu = NULL;
    h->pc_kind = 0;
    csr a = expanded_jacobian(h);
    if (kind == SFV_PRECOND_AUTO) kind = a.n <= 30000 ? SFV_PRECOND_LU : SFV_PRECOND_ILU1;
    int rc = SFV_OK;
    if (kind == SFV_PRECOND_ILU0 || kind == SFV_PRECOND_ILU1 || kind == SFV_PRECOND_ILU2) {
        const int level = kind == SFV_PRECOND_ILU0 ? 0 : kind == SFV_PRECOND_ILU1 ? 1 : 2;
        rc = ilu_factor(&a, level, &h->ilu, &h->err);
        if (rc == SFV_ERR_ILU_BREAKDOWN) { /* one retry with a 1e-12 |diag| shift */
            double dn = 0.0;
            for (int i = 0; i < a.n; ++i)
                for (int p = a.row_ptr[i]; p < a.row_ptr[i + 1]; ++p)
                    if (a.col[p] == i) dn += a.val[p] * a.val[p];
            dn = sqrt(dn);
            for (int i = 0; i < a.n; ++i)
                for (int p = a.row_ptr[i]; p < a.row_ptr[i + 1]; ++p)
                    if (a.col[p] == i) a.val[p] += 1e-12 * dn;
            rc = ilu_factor(&a, level, &h->ilu, &h->err);
        }
        if (!rc) h->pc_kind = 1;
    } else if (kind == SFV_PRECOND_LU) {
        band_lu* b = NULL;
        rc = lu_factor(&a, &b, &h->err);
        if (!rc) { h->lu = b; h->pc_kind = 2; }
    }
    csr_free(&a);
    return rc;
}

static void precond_solve(const orc_case* h, const double* r, double* z, int n) {
    if (h->pc_kind == 1) ilu_solve(&h->ilu, r, z);
    else if (h->pc_kind == 2) lu_solve(h->lu, r, z);
    else memcpy(z, r, sizeof(double) * n);
}

int orc_precond_apply(orc_case* h, const double* r, double* z) {
    precond_solve(h, r, z, 3 * h->nc);
    return SFV_OK;
}

/* ------------------------------------------------------------------ GMRES */

static double ddot(const double* a, const double* b, int n) { /* std::inner_product */
    /* ORC_DOT_BLOCK=k (experiments only, scripts/order_sensitivity.py): sequential sums of k
       consecutive products, then of the block sums — another valid evaluation order */
    static int blk = -1;
    if (blk < 0) {
        const char* e = getenv("ORC_DOT_BLOCK");
        blk = e ? atoi(e) : 0;
    }
    if (blk > 0) {
        double t = 0.0;
        for (int i0 = 0; i0 < n; i0 += blk) {
            double s = 0.0;
            const int i1 = i0 + blk < n ? i0 + blk : n;
            for (int i = i0; i < i1; ++i) s = s + a[i] * b[i];
            t = t + s;
        }
        return t;
    }
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = s + a[i] * b[i];
    return s;
}
static double dnorm(const double* a, int n) { return sqrt(ddot(a, a, n)); }
static void daxpy(double alpha, const double* x, double* y, int n) {
    for (int i = 0; i < n; ++i) y[i] += alpha * x[i];
}

typedef struct {
    orc_case* h;
    const double* u;
    const double* r_u;
    v3 *s1, *s2;
} jv_op;

static int op_apply(jv_op* op, const double* v, double* out) {
    return jv(op->h, op->u, op->r_u, v, out, op->s1, op->s2);
}

enum { G_CONVERGED = 0, G_MAX_ITERS = 1, G_STAGNATED = 2 };

/* gmres_solve (linalg.cpp:423-538): left preconditioned, or right preconditioned (right != 0:
   residuals unpreconditioned :437, w = op(M^-1 v_j) :466-467, dx = M^-1 (V y) :514) */
static int gmres(jv_op* op, const double* b, double* x, int n, int restart, double rel_reduction,
                 int max_iters, int right, int* iters_out, int* status_out, double* rel_out) {
    orc_case* h = op->h;
    double* r = xcalloc(n, sizeof(double));
    double* tmp = xcalloc(n, sizeof(double));
    double* V = xcalloc((size_t)(restart + 1) * n, sizeof(double));
    double* w = xcalloc(n, sizeof(double));
    double* H = xcalloc((size_t)restart * (restart + 1), sizeof(double));
    double* cs = xcalloc(restart + 1, sizeof(double));
    double* sn = xcalloc(restart + 1, sizeof(double));
    double* g = xcalloc(restart + 2, sizeof(double));
    double* y = xcalloc(restart + 1, sizeof(double));
    double* dx = xcalloc(n, sizeof(double));
    int rc = SFV_OK, status = G_MAX_ITERS, total = 0;
    double rel = 1.0;
#define RESID(xx)                                                      \
    do {                                                               \
        rc = op_apply(op, (xx), tmp);                                  \
        if (rc) goto done;                                             \
        for (int i = 0; i < n; ++i) tmp[i] = b[i] - tmp[i];            \
        if (right)                                                     \
            for (int i = 0; i < n; ++i) r[i] = tmp[i];                 \
        else                                                           \
            precond_solve(h, tmp, r, n);                               \
    } while (0)
    RESID(x);
    const double r0 = dnorm(r, n);
    if (r0 == 0.0) {
        status = G_CONVERGED;
        rel = 0.0;
        goto done;
    }
    const double target = rel_reduction * r0;
    double beta = r0;
    while (total < max_iters) {
        const double cycle_start = beta;
        for (int i = 0; i < n; ++i) V[i] = r[i] / beta;
        g[0] = beta;
        int j = 0, happy = 0;
        while (j < restart && total < max_iters) {
            if (right) {
                precond_solve(h, V + (size_t)j * n, tmp, n);
                rc = op_apply(op, tmp, w);
            } else {
                rc = op_apply(op, V + (size_t)j * n, tmp);
                if (!rc) precond_solve(h, tmp, w, n);
            }
            if (rc) goto done;
            double* hj = H + (size_t)j * (restart + 1);
            for (int i = 0; i <= j + 1; ++i) hj[i] = 0.0;
            for (int i = 0; i <= j; ++i) {
                hj[i] = ddot(w, V + (size_t)i * n, n);
                daxpy(-hj[i], V + (size_t)i * n, w, n);
            }
            hj[j + 1] = dnorm(w, n);
            for (int i = 0; i < j; ++i) {
                const double t = cs[i] * hj[i] + sn[i] * hj[i + 1];
                hj[i + 1] = -sn[i] * hj[i] + cs[i] * hj[i + 1];
                hj[i] = t;
            }
            const double denom = hypot(hj[j], hj[j + 1]);
            const double c = denom == 0.0 ? 1.0 : hj[j] / denom;
            const double s = denom == 0.0 ? 0.0 : hj[j + 1] / denom;
            cs[j] = c;
            sn[j] = s;
            g[j + 1] = -s * g[j];
            g[j] = c * g[j];
            hj[j] = denom;
            const double subdiag = hj[j + 1];
            hj[j + 1] = 0.0;
            ++total;
            ++j;
            if (subdiag <= 1e-14 * fmax(denom, 1e-300)) { happy = 1; break; }
            if (fabs(g[j]) <= target) break;
            if (j < restart)
                for (int i = 0; i < n; ++i) V[(size_t)j * n + i] = w[i] / subdiag;
        }
        for (int i = j - 1; i >= 0; --i) {
            double s = g[i];
            for (int k = i + 1; k < j; ++k) s -= H[(size_t)k * (restart + 1) + i] * y[k];
            y[i] = s / H[(size_t)i * (restart + 1) + i];
        }
        for (int i = 0; i < n; ++i) dx[i] = 0.0;
        for (int i = 0; i < j; ++i) daxpy(y[i], V + (size_t)i * n, dx, n);
        if (right) {
            precond_solve(h, dx, tmp, n);
            for (int i = 0; i < n; ++i) dx[i] = tmp[i];
        }
        daxpy(1.0, dx, x, n);
        RESID(x);
        beta = dnorm(r, n);
        rel = beta / r0;
        if (beta <= target || (happy && fabs(g[j]) <= target)) { status = G_CONVERGED; goto done; }
        if (happy) { status = G_STAGNATED; goto done; }
        if (beta >= cycle_start * (1.0 - 1e-12)) { status = G_STAGNATED; goto done; }
    }
    status = G_MAX_ITERS;
#undef RESID
done:
    *iters_out = total;
    *status_out = status;
    *rel_out = rel;
    free(r); free(tmp); free(V); free(w); free(H); free(cs); free(sn); free(g); free(y); free(dx);
    return rc;
}

int orc_gmres_jv(orc_case* h, const double* u, const double* r_u, const double* b, double* x,
                 int restart, double rel_reduction, int max_iters, int right, int* iters, int* status,
                 double* rel_residual) {
    jv_op op = {h, u, r_u, xcalloc(h->nc, sizeof(v3)), xcalloc(h->nc, sizeof(v3))};
    const int rc = gmres(&op, b, x, 3 * h->nc, restart, rel_reduction, max_iters, right, iters, status,
                         rel_residual);
    free(op.s1);
    free(op.s2);
    return rc;
}

/* ------------------------------------------------------------------ JFNK */

static double field_norm(const v3* v, int nc) { /* nonlinear.cpp:19-24 */
    double s = 0.0;
    for (int c = 0; c < nc; ++c) {
        s += v[c].x * v[c].x;
        s += v[c].y * v[c].y;
        s += v[c].z * v[c].z;
    }
    return sqrt(s);
}

static void push_record(sfv_solve_report* rep, int iter, double r_norm, int kry, double s) {
    const int cap = (int)(sizeof rep->records / sizeof rep->records[0]);
    if (rep->n_records < cap)
        rep->records[rep->n_records] = (sfv_iteration_record){0, iter, r_norm, kry, s};
    ++rep->n_records;
}

static double now_s(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

/* jfnk_solve (nonlinear.cpp:173-266) with line_search (:140-163) and
 * check_convergence (:97-103).  Returns an error code only for errors the
 * reference lets escape (e.g. GradientFailure); statuses go in rep. */
static int jfnk(orc_case* h, v3* u, const sfv_solver_cfg* cfg, sfv_solve_report* rep) {
    const double t0 = now_s();
    const int nc = h->nc, n = 3 * nc;
    const int max_outer = cfg->max_outer > 0 ? cfg->max_outer : 50;
    const double inner = cfg->inner_reduction > 0.0 ? cfg->inner_reduction : 1e-3;
    memset(rep, 0, sizeof *rep);
    rep->status = SFV_MAX_ITERS;
    v3* r = xcalloc(nc, sizeof(v3));
    v3* cand = xcalloc(nc, sizeof(v3));
    v3* rc_s = xcalloc(nc, sizeof(v3));
    double* uflat = xcalloc(n, sizeof(double));
    double* rflat = xcalloc(n, sizeof(double));
    double* rhs = xcalloc(n, sizeof(double));
    double* x = xcalloc(n, sizeof(double));
    jv_op op = {h, uflat, rflat, xcalloc(nc, sizeof(v3)), xcalloc(nc, sizeof(v3))};
    int err = residual(h, u, r);
    if (err) goto out;
    double r_norm = field_norm(r, nc);
    const double r_norm0 = r_norm;
    rep->initial_residual = r_norm0;
    rep->final_residual = r_norm;
    push_record(rep, 0, r_norm, 0, 0.0);
    if (r_norm <= cfg->a_tol || r_norm <= cfg->r_tol * r_norm0) {
        rep->status = SFV_CONVERGED;
        goto out;
    }
    int stag = 0;
    for (int k = 0; k < max_outer; ++k) {
        store_cells(rflat, r, nc);
        store_cells(uflat, u, nc);
        for (int i = 0; i < n; ++i) { rhs[i] = -rflat[i]; x[i] = 0.0; }
        int iters = 0, status = 0;
        double rel = 0.0;
        err = gmres(&op, rhs, x, n, cfg->restart, inner, cfg->max_krylov, cfg->right_preconditioned, &iters,
                    &status, &rel);
        if (err == SFV_ERR_JVP_NAN) {
            rep->status = SFV_DIVERGED;
            snprintf(rep->detail, SFV_DETAIL_LEN, "%s", h->err.msg);
            err = SFV_OK;
            break;
        }
        if (err) goto out;
        rep->krylov_iters += iters;
        if (status == G_STAGNATED) {
            if (++stag >= 2) {
                rep->status = SFV_DIVERGED;
                snprintf(rep->detail, SFV_DETAIL_LEN, "gmres stagnated on two consecutive outer iterations");
                break;
            }
        } else {
            stag = 0;
        }
        double s = 1.0;
        if (cfg->line_search) {
            int ok = 0;
            double ss = 1.0, rn = 0.0;
            for (int attempt = 0; attempt < 6; ++attempt, ss *= 0.5) {
                for (int c = 0; c < nc; ++c)
                    cand[c] = vadd(u[c], vscale((v3){x[3 * c], x[3 * c + 1], x[3 * c + 2]}, ss));
                if (residual(h, cand, rc_s)) continue;
                rn = field_norm(rc_s, nc);
                if (rn < r_norm) { ok = 1; break; }
            }
            if (!ok) {
                rep->status = SFV_DIVERGED;
                snprintf(rep->detail, SFV_DETAIL_LEN, "line search found no residual decrease");
                break;
            }
            s = ss;
            memcpy(r, rc_s, sizeof(v3) * nc);
            r_norm = rn;
            for (int c = 0; c < nc; ++c)
                u[c] = vadd(u[c], vscale((v3){x[3 * c], x[3 * c + 1], x[3 * c + 2]}, s));
        } else {
            for (int c = 0; c < nc; ++c) u[c] = vadd(u[c], (v3){x[3 * c], x[3 * c + 1], x[3 * c + 2]});
            if (residual(h, u, r)) {
                rep->status = SFV_DIVERGED;
                snprintf(rep->detail, SFV_DETAIL_LEN, "%s", h->err.msg);
                rep->outer_iters = k + 1;
                break;
            }
            r_norm = field_norm(r, nc);
        }
        rep->outer_iters = k + 1;
        push_record(rep, k + 1, r_norm, iters, s);
        rep->final_residual = r_norm;
        /* du_norm = s * field_norm(du); s_tol branch */
        double du_norm = 0.0;
        if (cfg->s_tol > 0.0) {
            double acc = 0.0;
            for (int i = 0; i < n; ++i) acc += x[i] * x[i];
            du_norm = s * sqrt(acc);
        }
        if (r_norm <= cfg->a_tol || r_norm <= cfg->r_tol * r_norm0 ||
            (cfg->s_tol > 0.0 && du_norm <= cfg->s_tol * field_norm(u, nc))) {
            rep->status = SFV_CONVERGED;
            break;
        }
    }
    if (rep->status == SFV_MAX_ITERS && rep->outer_iters == max_outer)
        snprintf(rep->detail, SFV_DETAIL_LEN, "outer iteration limit reached");
out:
    rep->wall_seconds = now_s() - t0;
    free(r); free(cand); free(rc_s); free(uflat); free(rflat); free(rhs); free(x);
    free(op.s1); free(op.s2);
    return err;
}

/* ------------------------------------------------------------------ segregated solver */

/* Ic0Precond (linalg.cpp:174-221): L on the lower pattern of A, row-oriented; 0 or -1 on a
 * breakdown (missing diagonal / non-positive pivot, IluBreakdown) */
static int ic0_factor(const csr* a, csr* L) {
    const int n = a->n;
    L->n = n;
    L->row_ptr = xcalloc(n + 1, sizeof(int));
    int nnz = 0;
    for (int i = 0; i < n; ++i)
        for (int p = a->row_ptr[i]; p < a->row_ptr[i + 1]; ++p)
            if (a->col[p] <= i) ++nnz;
    L->nnz = nnz;
    L->col = xcalloc(nnz > 0 ? nnz : 1, sizeof(int));
    L->val = xcalloc(nnz > 0 ? nnz : 1, sizeof(double));
    int q = 0;
    for (int i = 0; i < n; ++i) {
        for (int p = a->row_ptr[i]; p < a->row_ptr[i + 1]; ++p)
            if (a->col[p] <= i) {
                L->col[q] = a->col[p];
                L->val[q++] = a->val[p];
            }
        L->row_ptr[i + 1] = q;
    }
    const int* rp = L->row_ptr;
    const int* col = L->col;
    double* val = L->val;
    for (int i = 0; i < n; ++i) {
        const int diag_p = rp[i + 1] - 1;
        if (diag_p < rp[i] || col[diag_p] != i) return -1;
        for (int p = rp[i]; p < diag_p; ++p) {
            const int j = col[p];
            double s = val[p];
            int pi = rp[i], pj = rp[j];
            while (pi < p && pj < rp[j + 1] - 1) {
                if (col[pi] == col[pj]) s -= val[pi++] * val[pj++];
                else if (col[pi] < col[pj]) ++pi;
                else ++pj;
            }
            val[p] = s / val[rp[j + 1] - 1];
        }
        double s = val[diag_p];
        for (int p = rp[i]; p < diag_p; ++p) s -= val[p] * val[p];
        if (!(s > 0.0)) return -1;
        val[diag_p] = sqrt(s);
    }
    return 0;
}

/* Ic0Precond::solve: forward L y = r, then backward L^T z = y in saxpy form */
static void ic0_solve(const csr* L, const double* r, double* z) {
    const int n = L->n;
    memcpy(z, r, sizeof(double) * n);
    for (int i = 0; i < n; ++i) {
        for (int p = L->row_ptr[i]; p < L->row_ptr[i + 1] - 1; ++p) z[i] -= L->val[p] * z[L->col[p]];
        z[i] /= L->val[L->row_ptr[i + 1] - 1];
    }
    for (int j = n - 1; j >= 0; --j) {
        z[j] /= L->val[L->row_ptr[j + 1] - 1];
        for (int p = L->row_ptr[j]; p < L->row_ptr[j + 1] - 1; ++p) z[L->col[p]] -= L->val[p] * z[j];
    }
}

static void csr_apply(const csr* a, const double* x, double* y) { /* ScalarCsrMatrix::apply */
    for (int i = 0; i < a->n; ++i) {
        double s = 0.0;
        for (int p = a->row_ptr[i]; p < a->row_ptr[i + 1]; ++p) s += a->val[p] * x[a->col[p]];
        y[i] = s;
    }
}

/* cg_solve (linalg.cpp:380-421): IC(0)-preconditioned CG, Jacobi on an IC(0) breakdown;
 * x holds x0 on entry.  Returns the iteration count; *fallback set on the Jacobi fallback. */
static int cg_solve(const csr* a, const double* b, double* x, double rel, int max_iters, int* fallback) {
    const int n = a->n;
    csr L;
    memset(&L, 0, sizeof L);
    double* inv_diag = NULL;
    if (ic0_factor(a, &L) != 0) {
        csr_free(&L);
        *fallback = 1;
        inv_diag = xcalloc(n, sizeof(double));
        for (int i = 0; i < n; ++i) {
            inv_diag[i] = 1.0;
            for (int p = a->row_ptr[i]; p < a->row_ptr[i + 1]; ++p)
                if (a->col[p] == i && a->val[p] != 0.0) inv_diag[i] = 1.0 / a->val[p];
        }
    }
    double* r = xcalloc(n, sizeof(double));
    double* z = xcalloc(n, sizeof(double));
    double* p = xcalloc(n, sizeof(double));
    double* ap = xcalloc(n, sizeof(double));
    int iters = 0;
    csr_apply(a, x, r);
    for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
    const double r0 = dnorm(r, n);
    if (r0 != 0.0) {
#define PRECOND(in, out)                                               \
    do {                                                               \
        if (inv_diag)                                                  \
            for (int i_ = 0; i_ < n; ++i_) out[i_] = inv_diag[i_] * in[i_]; \
        else                                                           \
            ic0_solve(&L, in, out);                                    \
    } while (0)
        PRECOND(r, z);
        memcpy(p, z, sizeof(double) * n);
        double rz = ddot(r, z, n);
        for (int it = 0; it < max_iters; ++it) {
            csr_apply(a, p, ap);
            const double pap = ddot(p, ap, n);
            if (!(pap > 0.0)) break;
            const double alpha = rz / pap;
            daxpy(alpha, p, x, n);
            daxpy(-alpha, ap, r, n);
            iters = it + 1;
            if (dnorm(r, n) <= rel * r0) break;
            PRECOND(r, z);
            const double rz_new = ddot(r, z, n);
            const double beta = rz_new / rz;
            rz = rz_new;
            for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        }
#undef PRECOND
    }
    free(r); free(z); free(p); free(ap); free(inv_diag);
    if (!inv_diag) csr_free(&L);
    return iters;
}

static int check_conv(double r_norm, double r0, double du_norm, double u_norm, const sfv_solver_cfg* cfg) {
    if (r_norm <= cfg->a_tol) return 1; /* nonlinear.cpp:97-103 */
    if (r_norm <= cfg->r_tol * r0) return 1;
    if (cfg->s_tol > 0.0 && du_norm <= cfg->s_tol * u_norm) return 1;
    return 0;
}

/* segregated_solve (nonlinear.cpp:268-351): per component, A u_next = A u + R_c(u) by CG */
static int segregated(orc_case* h, v3* u, const sfv_solver_cfg* cfg, const csr comps[3], sfv_solve_report* rep) {
    const double t0 = now_s();
    const int nc = h->nc;
    const int max_outer = cfg->max_outer > 0 ? cfg->max_outer : 2000;
    const double inner = cfg->inner_reduction > 0.0 ? cfg->inner_reduction : 0.9;
    const double relax = cfg->relaxation > 0.0 ? cfg->relaxation : 1.0;
    memset(rep, 0, sizeof *rep);
    rep->status = SFV_MAX_ITERS;
    v3* r = xcalloc(nc, sizeof(v3));
    v3* un = xcalloc(nc, sizeof(v3));
    double *uc = xcalloc(nc, sizeof(double)), *rc_ = xcalloc(nc, sizeof(double)), *b = xcalloc(nc, sizeof(double));
    int rc = residual(h, u, r);
    if (rc) goto out;
    double r_norm = field_norm(r, nc);
    const double r0 = r_norm;
    rep->initial_residual = r0;
    rep->final_residual = r_norm;
    push_record(rep, 0, r_norm, 0, 0.0);
    if (check_conv(r_norm, r0, 0.0, 0.0, cfg)) {
        rep->status = SFV_CONVERGED;
        goto out;
    }
    for (int k = 0; k < max_outer; ++k) {
        int krylov = 0;
        for (int c = 0; c < 3; ++c) {
            for (int i = 0; i < nc; ++i) {
                uc[i] = vget(u[i], c);
                rc_[i] = vget(r[i], c);
            }
            csr_apply(&comps[c], uc, b);
            for (int i = 0; i < nc; ++i) b[i] += rc_[i];
            krylov += cg_solve(&comps[c], b, uc, inner, nc > 50 ? nc : 50, &rep->cg_diag_fallback);
            for (int i = 0; i < nc; ++i) vset(&un[i], c, uc[i]);
        }
        rep->krylov_iters += krylov;
        double du_norm = 0.0;
        for (int i = 0; i < nc; ++i) {
            const v3 du = vscale(vsub(un[i], u[i]), relax);
            du_norm += du.x * du.x;
            du_norm += du.y * du.y;
            du_norm += du.z * du.z;
            u[i] = vadd(u[i], du);
        }
        du_norm = sqrt(du_norm);
        if (residual(h, u, r)) {
            rep->status = SFV_DIVERGED;
            snprintf(rep->detail, SFV_DETAIL_LEN, "%s", h->err.msg);
            rep->outer_iters = k + 1;
            break;
        }
        r_norm = field_norm(r, nc);
        rep->outer_iters = k + 1;
        push_record(rep, k + 1, r_norm, krylov, 1.0);
        rep->final_residual = r_norm;
        if (!isfinite(r_norm)) {
            rep->status = SFV_DIVERGED;
            snprintf(rep->detail, SFV_DETAIL_LEN, "residual norm overflow");
            break;
        }
        if (check_conv(r_norm, r0, du_norm, field_norm(u, nc), cfg)) {
            rep->status = SFV_CONVERGED;
            break;
        }
    }
    if (rep->status == SFV_MAX_ITERS) snprintf(rep->detail, SFV_DETAIL_LEN, "outer iteration limit reached");
out:
    rep->wall_seconds = now_s() - t0;
    free(r); free(un); free(uc); free(rc_); free(b);
    return rc;
}

int orc_jfnk_solve(orc_case* h, double* uf, const sfv_solver_cfg* cfg, sfv_solve_report* rep) {
    v3* u = xcalloc(h->nc, sizeof(v3));
    load_cells(u, uf, h->nc);
    const int rc = jfnk(h, u, cfg, rep);
    store_cells(uf, u, h->nc);
    free(u);
    return rc;
}

/* run_steps (nonlinear.cpp:382-446) with predict_step_start (:165-171) */
int orc_run_steps(orc_case* h, double* field, const sfv_solver_cfg* cfg, int n_steps,
                  sfv_solve_report* reports, int cap, int* n_reports, double* wall) {
    const double t0 = now_s();
    const int nc = h->nc;
    if (n_steps < 1) return fail(&h->err, SFV_ERR_INVALID_ARGUMENT, -1, "run_steps: need at least one step");
    *n_reports = 0;
    const int seg = cfg->algorithm == SFV_ALG_SEGREGATED;
    csr comps[3];
    memset(comps, 0, sizeof comps);
    int rc = 0;
    if (seg) { /* scalar_component_matrices instead of a preconditioner (nonlinear.cpp:397-400) */
        if (negated_components(h, comps) != 0) {
            for (int c = 0; c < 3; ++c) csr_free(&comps[c]);
            return fail(&h->err, SFV_ERR_INVALID_ARGUMENT, -1, "scalar_component: blocks are not diagonal");
        }
    } else {
        rc = orc_precond_create(h, cfg->preconditioner);
        if (rc) return rc;
    }
    v3* fu = xcalloc(nc, sizeof(v3));
    v3* fuo = xcalloc(nc, sizeof(v3));
    v3* fuoo = xcalloc(nc, sizeof(v3));
    v3* fvo = xcalloc(nc, sizeof(v3));
    v3* fvoo = xcalloc(nc, sizeof(v3));
    v3* fao = xcalloc(nc, sizeof(v3));
    v3* u = xcalloc(nc, sizeof(v3));
    load_cells(fu, field, nc);
    load_cells(fuo, field + 3 * nc, nc);
    load_cells(fuoo, field + 6 * nc, nc);
    load_cells(fvo, field + 9 * nc, nc);
    load_cells(fvoo, field + 12 * nc, nc);
    load_cells(fao, field + 15 * nc, nc);
    const double dt = h->dt;
    for (int step = 1; step <= n_steps; ++step) {
        h->time = h->transient ? step * dt : (double)step / n_steps;
        if (h->transient) {
            memcpy(h->u_old, fuo, sizeof(v3) * nc);
            memcpy(h->u_old_old, fuoo, sizeof(v3) * nc);
            memcpy(h->v_old, fvo, sizeof(v3) * nc);
            memcpy(h->v_old_old, fvoo, sizeof(v3) * nc);
            for (int c = 0; c < nc; ++c)
                u[c] = vadd(vadd(fuo[c], vscale(fvo[c], dt)), vscale(fao[c], 0.5 * dt * dt));
        } else {
            memcpy(u, fu, sizeof(v3) * nc);
        }
        sfv_solve_report rep;
        const int e = seg ? segregated(h, u, cfg, comps, &rep) : jfnk(h, u, cfg, &rep);
        if (e) {
            memset(&rep, 0, sizeof rep);
            rep.status = SFV_DIVERGED;
            snprintf(rep.detail, SFV_DETAIL_LEN, "%s", h->err.msg);
        }
        rep.step = step;
        for (int i = 0; i < rep.n_records && i < 64; ++i) rep.records[i].step = step;
        if (*n_reports < cap) reports[*n_reports] = rep;
        ++*n_reports;
        if (rep.status != SFV_CONVERGED) break;
        if ((rc = commit_state(h, u)) != SFV_OK) break; /* eval.commit(u) (nonlinear.cpp:426) */
        if (h->transient) {
            for (int c = 0; c < nc; ++c) {
                const v3 vn = bdf2_vel(u[c], fuo[c], fuoo[c], dt);
                const v3 an = bdf2_acc(u[c], fuo[c], fuoo[c], fvo[c], fvoo[c], dt);
                fuoo[c] = fuo[c];
                fuo[c] = u[c];
                fvoo[c] = fvo[c];
                fvo[c] = vn;
                fao[c] = an;
            }
        } else {
            memcpy(fuo, u, sizeof(v3) * nc);
        }
        memcpy(fu, u, sizeof(v3) * nc);
    }
    if (*n_reports > cap) *n_reports = cap;
    store_cells(field, fu, nc);
    store_cells(field + 3 * nc, fuo, nc);
    store_cells(field + 6 * nc, fuoo, nc);
    store_cells(field + 9 * nc, fvo, nc);
    store_cells(field + 12 * nc, fvoo, nc);
    store_cells(field + 15 * nc, fao, nc);
    free(fu); free(fuo); free(fuoo); free(fvo); free(fvoo); free(fao); free(u);
    for (int c = 0; c < 3; ++c) csr_free(&comps[c]);
    *wall = now_s() - t0;
    return rc;
}

/* DiscretisationConfig::body_force (discretisation.hpp:24): f = body_force(centroid_c) per
   cell (3 nc, interleaved; NULL clears); the residual adds volume_c * f_c (discretisation.cpp:160-161) */
int orc_set_body_force(orc_case* h, const double* f) {
    free(h->body_vol);
    h->body_vol = NULL;
    if (!f) return SFV_OK;
    h->body_vol = xcalloc(h->nc, sizeof(v3));
    for (int c = 0; c < h->nc; ++c) {
        const v3 fc = {f[3 * c], f[3 * c + 1], f[3 * c + 2]};
        h->body_vol[c] = vscale(fc, h->volume[c]);
    }
    return SFV_OK;
}

/* per boundary face values (3 (nf - nint), face nint + i; NULL = per patch): the sampled
   BoundaryCondition::value(face_centroid, t) of the current time */
int orc_set_face_bc(orc_case* h, const double* v) {
    free(h->face_bc);
    h->face_bc = NULL;
    if (!v) return SFV_OK;
    const int nb = h->nf - h->nint;
    h->face_bc = xcalloc(nb > 0 ? nb : 1, sizeof(v3));
    for (int i = 0; i < nb; ++i) h->face_bc[i] = (v3){v[3 * i], v[3 * i + 1], v[3 * i + 2]};
    return SFV_OK;
}
