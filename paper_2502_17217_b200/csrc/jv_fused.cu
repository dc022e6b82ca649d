// jv_fused.cu — the fused residual / J.v kernel for sm_100a (one persistent launch).
//
// Same arithmetic as residual.cu (bit-identical to ResidualEvaluator::residual,
// /root/reference/proj/src/discretisation.cpp:108-174), restructured as a three-stage
// wavefront over tiles of kTile consecutive cells, so that nothing but the compulsory
// inputs and the output touches HBM:
//
//   A(t)  gradient of tile t (u + eps v fused on load) -> G ring      (discretisation.cpp:10-31)
//   B1(s) every face whose lower cell lies in tile s, computed ONCE:  (discretisation.cpp:121-156,
//         interpolated-stress flux and Rhie-Chow term, written to the   :176-208)
//         face-result ring at both of its cells' slots (negated on the neighbour side)
//   B2(s) per cell of tile s, the ring entries in ascending face order: sum of fluxes, then
//         sum of stabilisation terms, BDF2 inertia, NaN scan, J.v epilogue
//
// with s = t - lag, lag = ceil(bandwidth / kTile) + 1 (the largest owner/neighbour index gap
// decides how far ahead the gradients must be).  Both rings are sized to the pipeline depth
// (a few MB at 1M cells) and stay resident in the 126 MB L2; ring traffic goes through L2
// only (ld/st .cg).  Tiles are claimed from an atomic ticket by a persistent grid whose
// CTAs are all resident, and stages hand over through per-tile epoch flags (release /
// acquire); every wait points at an earlier ticket, so the pipeline cannot deadlock.
//
// Compiled with -fmad=false (see residual.cu).
#include <cfloat>

#include "device.h"
#include "sfv_case.h"

// timing probes (scripts/probes): -DSFV_FPROBE=m drops 1: stage waits, 2: face stage, 4: gradient
// stage, 8: per-cell sums.  Results are then wrong; production builds use 0.
#ifndef SFV_FPROBE
#define SFV_FPROBE 0
#endif
#define FPROBE(b) (!(SFV_FPROBE & (b)))

namespace sfv {
namespace {

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
__device__ __forceinline__ bool fin(d3 a) { return isfinite(a.x) && isfinite(a.y) && isfinite(a.z); }

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
__device__ __forceinline__ dm3 interp(const dm3& p, const dm3& n, double w) { return madd(mscl(p, w), mscl(n, 1.0 - w)); }
__device__ __forceinline__ dm3 defgrad(const dm3& g) {
    dm3 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) r.a[i][j] = (i == j ? 1.0 : 0.0) + g.a[j][i];
    return r;
}
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
__device__ __forceinline__ dm3 stress(const Physics& ph, const dm3& g, bool& ok) {
    if (ph.law == SFV_LAW_NEO_HOOKEAN) return neo_hookean(g, ph.mu, ph.lam, ok);
    ok = true;
    return hooke(g, ph.mu, ph.lam);
}
__device__ __forceinline__ d3 rhie_chow(d3 up, d3 uo, const dm3& gf, d3 delta, double d_mag, double area_mag,
                                        double alpha, double kbar) {
    const d3 compact = scl(sub(uo, up), nrm(delta) / d_mag);
    return scl(sub(compact, dot_left(delta, gf)), alpha * kbar * area_mag);
}
__device__ __forceinline__ d3 transform_area(d3 gamma, const dm3& ff, bool& ok) {
    const double j = det(ff);
    ok = j > 0.0;
    return scl(dot_left(gamma, inverse(ff)), j);
}

template <bool PERT>
__device__ __forceinline__ d3 load_u(const double* __restrict__ u, const double* __restrict__ v, double eps, int c) {
    if (PERT)
        return {u[3 * c] + eps * v[3 * c], u[3 * c + 1] + eps * v[3 * c + 1], u[3 * c + 2] + eps * v[3 * c + 2]};
    return {u[3 * c], u[3 * c + 1], u[3 * c + 2]};
}
__device__ __forceinline__ d3 ld3(const double* __restrict__ p, int c) { return {p[3 * c], p[3 * c + 1], p[3 * c + 2]}; }

__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Flag polls are relaxed on purpose: an acquire load compiles to LDG.STRONG + CCTL.IVALL,
// i.e. it invalidates the whole SM's L1 on every poll and destroys the neighbour reuse
// of every co-resident CTA.  The data a stage hands over (the two rings) is only ever read
// with ld.global.cg (LDG.STRONG.GPU, served by L2, the coherence point) and only after the
// poll loop has observed the flag; the producer publishes with st.release.gpu
// (MEMBAR.ALL.GPU before the flag store), so the ring lines are in L2 before the flag.
__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// every thread polls a share of flags[lo..hi] until all equal epoch, then the CTA syncs
__device__ __forceinline__ void wait_range(const int* flags, int lo, int hi, int epoch) {
    if (lo < 0) lo = 0;
    for (int i = lo + static_cast<int>(threadIdx.x); i <= hi; i += blockDim.x)
        while (FPROBE(1) && ld_relaxed(&flags[i]) != epoch) __nanosleep(32);
    __syncthreads();
}

// bar.sync orders the CTA's writes before thread 0's gpu-scope fence (cumulativity),
// so one fence + release store publishes the whole tile
__device__ __forceinline__ void publish(int* flag, int epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        st_release(flag, epoch);
    }
}

// Hooke, small strain: flux = Gamma . interp(sigma_P, sigma_N, w) and the Rhie-Chow term
// with grad_f = interp(G_P, G_N, w), evaluated element by element with exactly the
// operations of hooke(), interp() and dot_left() (so the result is bit-identical) but
// without materialising the four 3x3 matrices — about half the live registers.
__device__ __forceinline__ void hooke_face(const double* gp, const double* gn, double w, double mu, double lam,
                                           d3 gam, d3 del, d3 up, d3 un, double dmag, double alpha, double kbar,
                                           d3& flux, d3& st) {
    const double tp = lam * ((gp[0] + gp[4]) + gp[8]);
    const double tn = lam * ((gn[0] + gn[4]) + gn[8]);
    const double wn = 1.0 - w;
    double f[3], dg[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        double a[3], g[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            double sp = (gp[3 * i + j] + gp[3 * j + i]) * mu;
            double sn = (gn[3 * i + j] + gn[3 * j + i]) * mu;
            if (i == j) {
                sp += tp;
                sn += tn;
            }
            a[i] = sp * w + sn * wn;
            g[i] = gp[3 * i + j] * w + gn[3 * i + j] * wn;
        }
        f[j] = gam.x * a[0] + gam.y * a[1] + gam.z * a[2];
        dg[j] = del.x * g[0] + del.y * g[1] + del.z * g[2];
    }
    flux = {f[0], f[1], f[2]};
    const d3 compact = scl(sub(un, up), nrm(del) / dmag);
    st = scl(sub(compact, d3{dg[0], dg[1], dg[2]}), alpha * kbar * nrm(gam));
}

__device__ __forceinline__ dm3 ring_ldG(const double* ring, int rc, int slot) {
    dm3 g;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) g.a[i][j] = __ldcg(&ring[static_cast<size_t>(3 * i + j) * rc + slot]);
    return g;
}

template <bool PERT, int S, bool GEN>
__global__ void __launch_bounds__(kTile, GEN ? 2 : 3) fused_kernel(FusedArgs a) {
    __shared__ int s_ticket;
    const DevMesh& m = a.m;
    const FusedLayout& L = a.L;
    const Physics& ph = a.ph;
    const int tid = threadIdx.x;
    const double eps = PERT ? *a.eps : 0.0;
    const bool zero = PERT && eps == 0.0;  // |v| = 0 (nonlinear.cpp:110)
    const int RC = L.ring_cells;
    for (;;) {
        if (tid == 0) s_ticket = atomicAdd(a.ticket, 1);
        __syncthreads();
        const int k = s_ticket;
        __syncthreads();
        if (k >= L.ntiles + L.lag) break;
        // ---------------- A(k): gradients of tile k into the G ring
        if (k < L.ntiles) {
            // the ring slots of tile k last held tile k - RT, read by B1/B2 of [k-RT-lag+1, k-RT]
            wait_range(a.b2_done, k - L.ring_tiles - L.lag + 1, k - L.ring_tiles, a.epoch);
            const int c = k * kTile + tid;
            if (c < m.nc && !zero && FPROBE(4)) {
                const d3 uc = load_u<PERT>(a.u, a.v, eps, c);
                dm3 g;
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j) g.a[i][j] = 0.0;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    if (s >= m.slots) break;
                    const size_t si = static_cast<size_t>(s) * m.nc + c;
                    const int o = m.slot_other[si];
                    d3 du;
                    if (o >= 0) {
                        du = sub(load_u<PERT>(a.u, a.v, eps, o), uc);
                    } else if (o <= -2 && a.pt.kind[-o - 2] == SFV_PATCH_SYMMETRY) {
                        const int f = m.slot_face[si] & 0x7fffffff;
                        const dm3 R = reflection({m.gam[f], m.gam[m.nf + f], m.gam[2 * static_cast<size_t>(m.nf) + f]});
                        du = sub(mv(R, uc), uc);
                    } else {
                        continue;
                    }
                    const d3 ls = {m.slot_ls[(3 * static_cast<size_t>(s)) * m.nc + c],
                                   m.slot_ls[(3 * static_cast<size_t>(s) + 1) * m.nc + c],
                                   m.slot_ls[(3 * static_cast<size_t>(s) + 2) * m.nc + c]};
#pragma unroll
                    for (int i = 0; i < 3; ++i)
#pragma unroll
                        for (int j = 0; j < 3; ++j) g.a[i][j] += cmp(ls, i) * cmp(du, j);
                }
                const int rs = c % RC;
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j) __stcg(&L.gring[static_cast<size_t>(3 * i + j) * RC + rs], g.a[i][j]);
            }
            publish(&a.a_done[k], a.epoch);
        }
        const int t = k - L.lag;
        if (t < 0 || t >= L.ntiles) continue;
        // ---------------- B1(t): faces whose lower cell is in tile t, each computed once
        wait_range(a.a_done, t, min(t + L.lag - 1, L.ntiles - 1), a.epoch);
        wait_range(a.b2_done, t - L.ring_tiles, t + L.lag - 1 - L.ring_tiles, a.epoch);
        if (!zero && FPROBE(2)) {
            const int fend = L.tile_face_ptr[t + 1];
            for (int fi = L.tile_face_ptr[t] + tid; fi < fend; fi += kTile) {
                const int p = L.f_owner[fi], o = L.f_other[fi];
                const int sl = L.f_slots[fi];
                const int sp = sl & 0xff, sn = (sl >> 8) & 0xff;
                const d3 gam = {L.f_geo[fi], L.f_geo[static_cast<size_t>(L.nfl) + fi],
                                L.f_geo[2 * static_cast<size_t>(L.nfl) + fi]};
                const d3 del = {L.f_geo[3 * static_cast<size_t>(L.nfl) + fi], L.f_geo[4 * static_cast<size_t>(L.nfl) + fi],
                                L.f_geo[5 * static_cast<size_t>(L.nfl) + fi]};
                const double dmag = L.f_geo[6 * static_cast<size_t>(L.nfl) + fi];
                const d3 up = load_u<PERT>(a.u, a.v, eps, p);
                d3 flux, st;
                if (!GEN && o >= 0) {  // Hooke, small strain: register-light, same arithmetic
                    double gp[9], gn[9];
                    const int rp0 = p % RC, rn0 = o % RC;
#pragma unroll
                    for (int q = 0; q < 9; ++q) {
                        gp[q] = __ldcg(&L.gring[static_cast<size_t>(q) * RC + rp0]);
                        gn[q] = __ldcg(&L.gring[static_cast<size_t>(q) * RC + rn0]);
                    }
                    const double w = L.f_geo[7 * static_cast<size_t>(L.nfl) + fi];
                    const d3 un = load_u<PERT>(a.u, a.v, eps, o);
                    hooke_face(gp, gn, w, ph.mu, ph.lam, gam, del, up, un, dmag, ph.alpha, ph.kbar, flux, st);
                    const d3 nf = ph.stab_only ? d3{0.0, 0.0, 0.0} : neg(flux), ns = neg(st);
                    double* fr = L.fring + static_cast<size_t>(sn) * 6 * RC + rn0;
                    __stcg(fr, nf.x);
                    __stcg(fr + RC, nf.y);
                    __stcg(fr + 2 * static_cast<size_t>(RC), nf.z);
                    __stcg(fr + 3 * static_cast<size_t>(RC), ns.x);
                    __stcg(fr + 4 * static_cast<size_t>(RC), ns.y);
                    __stcg(fr + 5 * static_cast<size_t>(RC), ns.z);
                    if (ph.stab_only) flux = {0.0, 0.0, 0.0};
                    double* fo = L.fring + static_cast<size_t>(sp) * 6 * RC + rp0;
                    __stcg(fo, flux.x);
                    __stcg(fo + RC, flux.y);
                    __stcg(fo + 2 * static_cast<size_t>(RC), flux.z);
                    __stcg(fo + 3 * static_cast<size_t>(RC), st.x);
                    __stcg(fo + 4 * static_cast<size_t>(RC), st.y);
                    __stcg(fo + 5 * static_cast<size_t>(RC), st.z);
                    continue;
                }
                const dm3 gp = ring_ldG(L.gring, RC, p % RC);
                bool okp;
                const dm3 sp3 = stress(ph, gp, okp);
                if (!okp) atomicMin(&a.err->inverted_cell, p);
                if (GEN && o >= 0) {
                    const double w = L.f_geo[7 * static_cast<size_t>(L.nfl) + fi];
                    const dm3 gn = ring_ldG(L.gring, RC, o % RC);
                    bool okn;
                    const dm3 sn3 = stress(ph, gn, okn);
                    if (!okn) atomicMin(&a.err->inverted_cell, o);
                    d3 gm = gam;
                    if (ph.tl) {
                        bool ok;
                        gm = transform_area(gam, interp(defgrad(gp), defgrad(gn), w), ok);
                        if (!ok) atomicMin(&a.err->inverted_face, L.f_index[fi]);
                    }
                    flux = dot_left(gm, interp(sp3, sn3, w));
                    const d3 un = load_u<PERT>(a.u, a.v, eps, o);
                    st = rhie_chow(up, un, interp(gp, gn, w), del, dmag, nrm(gam), ph.alpha, ph.kbar);
                    const int rn = o % RC;
                    const d3 nf = ph.stab_only ? d3{0.0, 0.0, 0.0} : neg(flux), ns = neg(st);
                    __stcg(&L.fring[(static_cast<size_t>(sn) * 6 + 0) * RC + rn], nf.x);
                    __stcg(&L.fring[(static_cast<size_t>(sn) * 6 + 1) * RC + rn], nf.y);
                    __stcg(&L.fring[(static_cast<size_t>(sn) * 6 + 2) * RC + rn], nf.z);
                    __stcg(&L.fring[(static_cast<size_t>(sn) * 6 + 3) * RC + rn], ns.x);
                    __stcg(&L.fring[(static_cast<size_t>(sn) * 6 + 4) * RC + rn], ns.y);
                    __stcg(&L.fring[(static_cast<size_t>(sn) * 6 + 5) * RC + rn], ns.z);
                } else {
                    const int patch = -o - 2;
                    const int kind = a.pt.kind[patch];
                    const d3 bc = {a.pt.value[patch][0], a.pt.value[patch][1], a.pt.value[patch][2]};
                    if (kind == SFV_PATCH_DISPLACEMENT) {
                        d3 gm = gam;
                        if (ph.tl) {
                            bool ok;
                            gm = transform_area(gam, defgrad(gp), ok);
                            if (!ok) atomicMin(&a.err->inverted_face, L.f_index[fi]);
                        }
                        flux = dot_left(gm, sp3);
                        st = rhie_chow(up, bc, gp, del, dmag, nrm(gam), ph.alpha, ph.kbar);
                    } else if (kind == SFV_PATCH_SYMMETRY) {
                        const dm3 R = reflection(gam);
                        d3 gm = gam;
                        if (ph.tl) {
                            bool ok;
                            gm = transform_area(gam, mirror_avg(defgrad(gp), R), ok);
                            if (!ok) atomicMin(&a.err->inverted_face, L.f_index[fi]);
                        }
                        flux = dot_left(gm, mirror_avg(sp3, R));
                        st = rhie_chow(up, mv(R, up), mirror_avg(gp, R), del, dmag, nrm(gam), ph.alpha, ph.kbar);
                    } else {  // traction: no stabilisation term (discretisation.cpp:204-205)
                        flux = scl(bc, nrm(gam));
                        st = {0.0, 0.0, 0.0};
                    }
                }
                if (ph.stab_only) flux = {0.0, 0.0, 0.0};
                const int rp = p % RC;
                __stcg(&L.fring[(static_cast<size_t>(sp) * 6 + 0) * RC + rp], flux.x);
                __stcg(&L.fring[(static_cast<size_t>(sp) * 6 + 1) * RC + rp], flux.y);
                __stcg(&L.fring[(static_cast<size_t>(sp) * 6 + 2) * RC + rp], flux.z);
                __stcg(&L.fring[(static_cast<size_t>(sp) * 6 + 3) * RC + rp], st.x);
                __stcg(&L.fring[(static_cast<size_t>(sp) * 6 + 4) * RC + rp], st.y);
                __stcg(&L.fring[(static_cast<size_t>(sp) * 6 + 5) * RC + rp], st.z);
            }
        }
        publish(&a.b1_done[t], a.epoch);
        // ---------------- B2(t): ordered per-cell sums
        wait_range(a.b1_done, t - L.lag + 1, t - 1, a.epoch);
        {
            const int c = t * kTile + tid;
            if (c < m.nc && FPROBE(8)) {
                if (zero) {
                    a.out[3 * c] = 0.0;
                    a.out[3 * c + 1] = 0.0;
                    a.out[3 * c + 2] = 0.0;
                } else {
                    const int rc = c % RC;
                    d3 r = {0.0, 0.0, 0.0};
                    int other[S];
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        other[s] = s < m.slots ? m.slot_other[static_cast<size_t>(s) * m.nc + c] : -1;
                        if (other[s] == -1) continue;  // padding
                        const d3 f = {__ldcg(&L.fring[(static_cast<size_t>(s) * 6 + 0) * RC + rc]),
                                      __ldcg(&L.fring[(static_cast<size_t>(s) * 6 + 1) * RC + rc]),
                                      __ldcg(&L.fring[(static_cast<size_t>(s) * 6 + 2) * RC + rc])};
                        if (!ph.stab_only) r = add(r, f);
                    }
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        const int o = other[s];
                        if (o == -1) continue;
                        if (o <= -2 && a.pt.kind[-o - 2] == SFV_PATCH_TRACTION) continue;
                        const d3 st = {__ldcg(&L.fring[(static_cast<size_t>(s) * 6 + 3) * RC + rc]),
                                       __ldcg(&L.fring[(static_cast<size_t>(s) * 6 + 4) * RC + rc]),
                                       __ldcg(&L.fring[(static_cast<size_t>(s) * 6 + 5) * RC + rc])};
                        r = add(r, st);
                    }
                    if (ph.law == SFV_LAW_NEO_HOOKEAN) {  // the stress loop visits every cell
                        bool ok;
                        (void)stress(ph, ring_ldG(L.gring, RC, rc), ok);
                        if (!ok) atomicMin(&a.err->inverted_cell, c);
                    }
                    if (ph.transient && !ph.stab_only) {
                        const d3 uc = load_u<PERT>(a.u, a.v, eps, c);
                        const double idt = 1.0 / (2.0 * ph.dt);
                        const d3 ut = ld3(a.hist.u_old, c), utm1 = ld3(a.hist.u_old_old, c);
                        const d3 vt = ld3(a.hist.v_old, c), vtm1 = ld3(a.hist.v_old_old, c);
                        const d3 vn = scl(add(sub(scl(uc, 3.0), scl(ut, 4.0)), utm1), idt);
                        const d3 ac = scl(add(sub(scl(vn, 3.0), scl(vt, 4.0)), vtm1), idt);
                        r = sub(r, scl(ac, ph.rho * m.volume[c]));
                    }
                    if (!ph.stab_only && !fin(r)) atomicMin(&a.err->nan_cell, c);
                    if constexpr (PERT) {
                        const double o0 = (r.x - a.r_u[3 * c]) / eps, o1 = (r.y - a.r_u[3 * c + 1]) / eps,
                                     o2 = (r.z - a.r_u[3 * c + 2]) / eps;
                        if (!(isfinite(o0) && isfinite(o1) && isfinite(o2))) atomicMin(&a.err->nan_jv, c);
                        a.out[3 * c] = o0;
                        a.out[3 * c + 1] = o1;
                        a.out[3 * c + 2] = o2;
                    } else {
                        a.out[3 * c] = r.x;
                        a.out[3 * c + 1] = r.y;
                        a.out[3 * c + 2] = r.z;
                    }
                }
            }
        }
        publish(&a.b2_done[t], a.epoch);
    }
}

template <bool PERT, int S, bool GEN>
int max_ctas() {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_kernel<PERT, S, GEN>, kTile, 0);
    return per_sm;
}

template <bool PERT, int S>
void launch_s(const FusedArgs& a, int grid, cudaStream_t s) {
    const bool gen = a.ph.law != SFV_LAW_HOOKE || a.ph.tl;
    if (gen) fused_kernel<PERT, S, true><<<grid, kTile, 0, s>>>(a);
    else fused_kernel<PERT, S, false><<<grid, kTile, 0, s>>>(a);
}

}  // namespace

int fused_resident_ctas(bool general) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per_sm = general ? min(max_ctas<true, 6, true>(), max_ctas<false, 6, true>())
                         : min(max_ctas<true, 6, false>(), max_ctas<false, 6, false>());
    per_sm = min(per_sm, general ? max_ctas<true, 8, true>() : max_ctas<true, 8, false>());
    per_sm = min(per_sm, general ? max_ctas<true, 4, true>() : max_ctas<true, 4, false>());
    return max(1, per_sm) * sms;
}

void launch_fused(const FusedArgs& a, int grid, cudaStream_t s) {
    const bool pert = a.eps != nullptr;
    const int S = a.m.slots;
    if (S <= 4) {
        if (pert) launch_s<true, 4>(a, grid, s);
        else launch_s<false, 4>(a, grid, s);
    } else if (S <= 6) {
        if (pert) launch_s<true, 6>(a, grid, s);
        else launch_s<false, 6>(a, grid, s);
    } else {
        if (pert) launch_s<true, 8>(a, grid, s);
        else launch_s<false, 8>(a, grid, s);
    }
}

}  // namespace sfv
