// face_math.cuh — the per-cell / per-face arithmetic of the residual, shared by the
// device kernels.  Every helper performs exactly the operations (and operation order) of
// the reference's small-matrix code (/root/reference/proj/src/laws.cpp,
// discretisation.cpp:33-106), so kernels built on them are bit-identical to
// ResidualEvaluator::residual when compiled with -fmad=false.
#pragma once

#include <cmath>

#include "device.h"
#include "sfv_case.h"

namespace sfv {
namespace fm {

struct d3 {
    double x, y, z;
};
struct dm3 {
    double a[3][3];
};

__device__ __forceinline__ d3 add(d3 a, d3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ d3 sub(d3 a, d3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ d3 scl(d3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ d3 neg(d3 a) { return {-a.x, -a.y, -a.z}; }
__device__ __forceinline__ double dot(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ double nrm(d3 a) { return sqrt(dot(a, a)); }
__device__ __forceinline__ double cmp(d3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

__device__ __forceinline__ dm3 madd(const dm3& a, const dm3& b) {
    dm3 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) r.a[i][j] = a.a[i][j] + b.a[i][j];
    return r;
}
__device__ __forceinline__ dm3 mscl(const dm3& a, double s) {
    dm3 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) r.a[i][j] = a.a[i][j] * s;
    return r;
}
__device__ __forceinline__ dm3 mmul(const dm3& a, const dm3& b) {
    dm3 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 3; ++k) s += a.a[i][k] * b.a[k][j];
            r.a[i][j] = s;
        }
    return r;
}
__device__ __forceinline__ dm3 mtr(const dm3& a) {
    dm3 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) r.a[i][j] = a.a[j][i];
    return r;
}
__device__ __forceinline__ d3 mv(const dm3& a, d3 v) {
    return {a.a[0][0] * v.x + a.a[0][1] * v.y + a.a[0][2] * v.z, a.a[1][0] * v.x + a.a[1][1] * v.y + a.a[1][2] * v.z,
            a.a[2][0] * v.x + a.a[2][1] * v.y + a.a[2][2] * v.z};
}
// v . A (row vector times matrix)
__device__ __forceinline__ d3 dot_left(d3 v, const dm3& a) {
    return {v.x * a.a[0][0] + v.y * a.a[1][0] + v.z * a.a[2][0], v.x * a.a[0][1] + v.y * a.a[1][1] + v.z * a.a[2][1],
            v.x * a.a[0][2] + v.y * a.a[1][2] + v.z * a.a[2][2]};
}
__device__ __forceinline__ double det(const dm3& a) {
    return a.a[0][0] * (a.a[1][1] * a.a[2][2] - a.a[1][2] * a.a[2][1]) -
           a.a[0][1] * (a.a[1][0] * a.a[2][2] - a.a[1][2] * a.a[2][0]) +
           a.a[0][2] * (a.a[1][0] * a.a[2][1] - a.a[1][1] * a.a[2][0]);
}
__device__ __forceinline__ dm3 inverse(const dm3& a) {
    const double id = 1.0 / det(a);
    dm3 r;
    r.a[0][0] = (a.a[1][1] * a.a[2][2] - a.a[1][2] * a.a[2][1]) * id;
    r.a[0][1] = (a.a[0][2] * a.a[2][1] - a.a[0][1] * a.a[2][2]) * id;
    r.a[0][2] = (a.a[0][1] * a.a[1][2] - a.a[0][2] * a.a[1][1]) * id;
    r.a[1][0] = (a.a[1][2] * a.a[2][0] - a.a[1][0] * a.a[2][2]) * id;
    r.a[1][1] = (a.a[0][0] * a.a[2][2] - a.a[0][2] * a.a[2][0]) * id;
    r.a[1][2] = (a.a[0][2] * a.a[1][0] - a.a[0][0] * a.a[1][2]) * id;
    r.a[2][0] = (a.a[1][0] * a.a[2][1] - a.a[1][1] * a.a[2][0]) * id;
    r.a[2][1] = (a.a[0][1] * a.a[2][0] - a.a[0][0] * a.a[2][1]) * id;
    r.a[2][2] = (a.a[0][0] * a.a[1][1] - a.a[0][1] * a.a[1][0]) * id;
    return r;
}
// w P + (1 - w) N (discretisation.cpp:33)
__device__ __forceinline__ dm3 interp(const dm3& p, const dm3& n, double w) { return madd(mscl(p, w), mscl(n, 1.0 - w)); }
// F = I + grad(u)^T (laws.cpp:5-9)
__device__ __forceinline__ dm3 defgrad(const dm3& g) {
    dm3 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) r.a[i][j] = (i == j ? 1.0 : 0.0) + g.a[j][i];
    return r;
}
// I - 2 n n^T (discretisation.cpp:60-66)
__device__ __forceinline__ dm3 reflection(d3 gamma) {
    const d3 n = scl(gamma, 1.0 / nrm(gamma));
    dm3 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) r.a[i][j] = (i == j ? 1.0 : 0.0) - (cmp(n, i) * cmp(n, j)) * 2.0;
    return r;
}
__device__ __forceinline__ dm3 mirror_avg(const dm3& a, const dm3& R) { return mscl(madd(a, mmul(mmul(R, a), R)), 0.5); }
// linear elastic (laws.cpp:21-27)
__device__ __forceinline__ dm3 hooke(const dm3& g, double mu, double lam) {
    dm3 s;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) s.a[i][j] = (g.a[i][j] + g.a[j][i]) * mu;
    const double t = lam * ((g.a[0][0] + g.a[1][1]) + g.a[2][2]);
    s.a[0][0] += t;
    s.a[1][1] += t;
    s.a[2][2] += t;
    return s;
}
// compressible neo-Hookean, Cauchy stress (laws.cpp:29-45)
__device__ __forceinline__ dm3 neo_hookean(const dm3& g, double mu, double kappa, bool& ok) {
    const dm3 F = defgrad(g);
    const double J = det(F);
    ok = J > 0.0;
    const dm3 bb = mscl(mmul(F, mtr(F)), pow(J, -2.0 / 3.0));
    const double t = ((bb.a[0][0] + bb.a[1][1]) + bb.a[2][2]) / 3.0;
    dm3 dv = bb;
    dv.a[0][0] -= t;
    dv.a[1][1] -= t;
    dv.a[2][2] -= t;
    dm3 s = mscl(dv, mu / J);
    const double p = 0.5 * kappa * (J * J - 1.0) / J;
    s.a[0][0] += p;
    s.a[1][1] += p;
    s.a[2][2] += p;
    return s;
}
// Green-Lagrange strain of kinematics() (laws.cpp:9-18): 0.5 ((G + G^T) + G G^T)
__device__ __forceinline__ dm3 green_strain(const dm3& g) { return mscl(madd(madd(g, mtr(g)), mmul(g, mtr(g))), 0.5); }
__device__ __forceinline__ double trc(const dm3& a) { return (a.a[0][0] + a.a[1][1]) + a.a[2][2]; }
// A : B, row by row (types.hpp ddot)
__device__ __forceinline__ double ddot(const dm3& a, const dm3& b) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) s += a.a[i][j] * b.a[i][j];
    return s;
}
// St. Venant-Kirchhoff, Cauchy stress (laws.cpp:29-37): (1/J) F S F^T, S = 2 mu E + lambda tr(E) I
__device__ __forceinline__ dm3 stvk(const dm3& g, double mu, double lam, bool& ok) {
    const dm3 F = defgrad(g);
    const double J = det(F);
    ok = J > 0.0;
    const dm3 E = green_strain(g);
    dm3 S = mscl(E, 2.0 * mu);
    const double t = lam * trc(E);
    S.a[0][0] += t;
    S.a[1][1] += t;
    S.a[2][2] += t;
    return mscl(mmul(mmul(F, S), mtr(F)), 1.0 / J);
}
// Guccione (laws.cpp:49-77); gc = C, c_f, c_t, c_fs, kappa, f0 xyz.  code: 0 ok, 1 det F <= 0,
// 2 exponent overflow (Q > 500 or not finite, LawOverflow)
__device__ __forceinline__ dm3 guccione(const dm3& g, const double* gc, int& code) {
    const dm3 F = defgrad(g);
    const double J = det(F);
    code = J > 0.0 ? 0 : 1;
    const dm3 E = green_strain(g);
    const double C = gc[0], cf = gc[1], ct = gc[2], cfs = gc[3], kappa = gc[4];
    const double f0[3] = {gc[5], gc[6], gc[7]};
    dm3 ff;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) ff.a[i][j] = f0[i] * f0[j];
    const dm3 EE = mmul(E, E);
    const double i1 = trc(E);
    const double i2 = 0.5 * (i1 * i1 - trc(EE));
    const double i4 = ddot(E, ff);
    const double i5 = ddot(EE, ff);
    const double cq = (cf - 2.0 * cfs) + ct;
    const double Q = (((ct * i1) * i1 - (2.0 * ct) * i2) + (cq * i4) * i4) + (2.0 * (cfs - ct)) * i5;
    if (code == 0 && (Q > 500.0 || !isfinite(Q))) code = 2;
    // guccione_dQ_dE: 2 c_t E + (2 cq i4) ff + 2 (c_fs - c_t) (E ff + ff E)
    const dm3 dq = madd(madd(mscl(E, 2.0 * ct), mscl(ff, (2.0 * cq) * i4)),
                        mscl(madd(mmul(E, ff), mmul(ff, E)), 2.0 * (cfs - ct)));
    dm3 S = mscl(dq, (0.5 * C) * exp(Q));
    const double pen = ((0.5 * kappa) * (J * J - 1.0)) / J;
    S.a[0][0] += pen;
    S.a[1][1] += pen;
    S.a[2][2] += pen;
    return mscl(mmul(mmul(F, S), mtr(F)), 1.0 / J);
}
// HardeningCurve::value / slope (laws.cpp:79-102): table (piecewise linear) or saturation
__device__ __forceinline__ double hard_value(const Physics& ph, double e) {
    if (ph.jn > 0) {
        if (e <= ph.jt[0]) return ph.jt[1];
        for (int i = 1; i < ph.jn; ++i)
            if (e <= ph.jt[2 * i]) {
                const double e0 = ph.jt[2 * i - 2], s0 = ph.jt[2 * i - 1], e1 = ph.jt[2 * i], s1 = ph.jt[2 * i + 1];
                return s0 + (s1 - s0) * (e - e0) / (e1 - e0);
            }
        return ph.jt[2 * ph.jn - 1];
    }
    return ph.ja + ph.jb * e + (ph.jc - ph.ja) * (1.0 - exp(-ph.jd * e));
}
__device__ __forceinline__ double hard_slope(const Physics& ph, double e) {
    if (ph.jn > 0) {
        if (e <= ph.jt[0] || e >= ph.jt[2 * ph.jn - 2]) return 0.0;
        for (int i = 1; i < ph.jn; ++i)
            if (e <= ph.jt[2 * i]) return (ph.jt[2 * i + 1] - ph.jt[2 * i - 1]) / (ph.jt[2 * i] - ph.jt[2 * i - 2]);
        return 0.0;
    }
    return ph.jb + (ph.jc - ph.ja) * ph.jd * exp(-ph.jd * e);
}
__device__ __forceinline__ double frob(const dm3& a) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) s += a.a[i][j] * a.a[i][j];
    return sqrt(s);
}
// j2_radial_return (laws.cpp:104-168) on the committed state st = b_bar (9), eps_p, F (9);
// the trial state goes to nst.  code: 0 ok, 1 det F <= 0 or inverted increment
// (InvertedElement), 3 hardening Newton did not converge (ReturnMapFailure).
__device__ __forceinline__ dm3 j2_return(const dm3& g, const double* st, const Physics& ph, int& code, double* nst) {
    const double mu = ph.mu, kappa = ph.lam;
    const dm3 Fn = defgrad(g);
    const double J = det(Fn);
    code = 0;
    dm3 bc, Fc;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        bc.a[q / 3][q % 3] = st[q];
        Fc.a[q / 3][q % 3] = st[10 + q];
    }
    const double epc = st[9];
    if (!(J > 0.0)) {
        code = 1;
        return Fn;
    }
    const dm3 frel = mmul(Fn, inverse(Fc));
    const double detf = det(frel);
    if (!(detf > 0.0)) {
        code = 1;
        return Fn;
    }
    const dm3 fbar = mscl(frel, pow(detf, -1.0 / 3.0));
    const dm3 bt0 = mmul(mmul(fbar, bc), mtr(fbar));
    const dm3 btr = mscl(madd(bt0, mtr(bt0)), 0.5);  // sym()
    const double t = ((btr.a[0][0] + btr.a[1][1]) + btr.a[2][2]) / 3.0;
    dm3 dv = btr;
    dv.a[0][0] -= t;
    dv.a[1][1] -= t;
    dv.a[2][2] -= t;
    const dm3 strial = mscl(dv, mu / J);
    const double snorm = frob(strial);
    const double sq23 = sqrt(2.0 / 3.0);
    const double fy = snorm - sq23 * hard_value(ph, epc);
    dm3 s = strial;
    dm3 bnew = btr;
    double epn = epc;
    if (!(fy <= 0.0)) {  // plastic (laws.cpp:128: elastic iff f_yield <= 0)
        const double trb = (btr.a[0][0] + btr.a[1][1]) + btr.a[2][2];
        const double mub = mu * trb / (3.0 * J);
        double dg = 0.0;
        bool done = false;
        const double tol = 1e-12 * fmax(snorm, hard_value(ph, 0.0));
        for (int it = 0; it < 50; ++it) {
            const double eps = epc + sq23 * dg;
            const double gg = snorm - 2.0 * mub * dg - sq23 * hard_value(ph, eps);
            if (fabs(gg) <= tol) {
                done = true;
                break;
            }
            const double gp = -2.0 * mub - (2.0 / 3.0) * hard_slope(ph, eps);
            const double next = dg - gg / gp;
            dg = next > 0.0 ? next : 0.5 * dg;
        }
        if (!done) code = 3;
        const dm3 ndir = mscl(strial, 1.0 / snorm);
        const double k = 2.0 * mub * dg;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) s.a[i][j] = strial.a[i][j] - ndir.a[i][j] * k;
        epn = epc + sq23 * dg;
        bnew = mscl(s, J / mu);
        const double iso = trb / 3.0;
        bnew.a[0][0] += iso;
        bnew.a[1][1] += iso;
        bnew.a[2][2] += iso;
    }
    if (nst) {
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            nst[q] = bnew.a[q / 3][q % 3];
            nst[10 + q] = Fn.a[q / 3][q % 3];
        }
        nst[9] = epn;
    }
    const double p = 0.5 * kappa * (J * J - 1.0) / J;
    s.a[0][0] += p;
    s.a[1][1] += p;
    s.a[2][2] += p;
    return s;
}
// the law's Cauchy stress; code 0 ok, 1 inverted (det F <= 0), 2 exponent overflow
__device__ __forceinline__ dm3 stress_code(const Physics& ph, const dm3& g, int& code) {
    bool ok = true;
    dm3 s;
    code = 0;
    switch (ph.law) {
        case SFV_LAW_NEO_HOOKEAN: s = neo_hookean(g, ph.mu, ph.lam, ok); break;
        case SFV_LAW_STVK: s = stvk(g, ph.mu, ph.lam, ok); break;
        case SFV_LAW_GUCCIONE: return guccione(g, ph.gc, code);
        default: return hooke(g, ph.mu, ph.lam);
    }
    code = ok ? 0 : 1;
    return s;
}
__device__ __forceinline__ dm3 stress(const Physics& ph, const dm3& g, bool& ok) {
    int code;
    const dm3 s = stress_code(ph, g, code);
    ok = code == 0;
    return s;
}
// Rhie-Chow term (discretisation.cpp:176-208)
__device__ __forceinline__ d3 rhie_chow(d3 up, d3 uo, const dm3& gf, d3 delta, double d_mag, double area_mag,
                                        double alpha, double kbar) {
    const d3 compact = scl(sub(uo, up), nrm(delta) / d_mag);
    return scl(sub(compact, dot_left(delta, gf)), alpha * kbar * area_mag);
}
// Nanson: J Gamma . F^{-1} (discretisation.cpp:96-106)
__device__ __forceinline__ d3 transform_area(d3 gamma, const dm3& ff, bool& ok) {
    const double j = det(ff);
    ok = j > 0.0;
    return scl(dot_left(gamma, inverse(ff)), j);
}

// Hooke, small strain: flux = Gamma . interp(sigma_P, sigma_N, w) and the Rhie-Chow term
// with grad_f = interp(G_P, G_N, w), element by element with exactly the operations of
// hooke(), interp(), dot_left() and rhie_chow() (bit-identical) but without materialising
// the four 3x3 matrices.  gp, gn: row-major 3x3 gradients.
// cfac = |Delta| / |d| and gmag = |Gamma| are the per-face constants of rhie_chow().
__device__ __forceinline__ void hooke_face(const double* gp, const double* gn, double w, double mu, double lam, d3 gam,
                                           d3 del, d3 up, d3 un, double cfac, double gmag, double alpha, double kbar,
                                           d3& flux, d3& st) {
    const double tp = lam * ((gp[0] + gp[4]) + gp[8]);
    const double tn = lam * ((gn[0] + gn[4]) + gn[8]);
    const double wn = 1.0 - w;
    // interp(sigma_P, sigma_N, w) is symmetric bit for bit ((g_ij + g_ji) == (g_ji + g_ij) in
    // IEEE arithmetic), so its 6 distinct entries are evaluated once each
    double a[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = i; j < 3; ++j) {
            double sp = (gp[3 * i + j] + gp[3 * j + i]) * mu;
            double sn = (gn[3 * i + j] + gn[3 * j + i]) * mu;
            if (i == j) {
                sp += tp;
                sn += tn;
            }
            a[i][j] = sp * w + sn * wn;
            a[j][i] = a[i][j];
        }
    double f[3], dg[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        double g[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) g[i] = gp[3 * i + j] * w + gn[3 * i + j] * wn;
        f[j] = gam.x * a[0][j] + gam.y * a[1][j] + gam.z * a[2][j];
        dg[j] = del.x * g[0] + del.y * g[1] + del.z * g[2];
    }
    flux = {f[0], f[1], f[2]};
    const d3 compact = scl(sub(un, up), cfac);
    st = scl(sub(compact, d3{dg[0], dg[1], dg[2]}), alpha * kbar * gmag);
}

}  // namespace fm
}  // namespace sfv
