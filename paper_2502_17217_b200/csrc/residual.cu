// residual.cu — fused FP64 residual / J.v kernels for sm_100a.
//
// Restates ResidualEvaluator::residual (/root/reference/proj/src/discretisation.cpp:108-174)
// and jacobian_vector_product (nonlinear.cpp:105-138) as two cell-centric passes:
//
//   grad_kernel  : LS gradient of u (+ eps v, the perturbation fused on load so u+eps v
//                  is never materialised) — cell_gradients, discretisation.cpp:10-31;
//   flux_kernel  : per cell, walk its faces in ascending face index (the order the
//                  reference's face loops reach that cell): interpolated-stress flux,
//                  Rhie-Chow term, boundary fluxes, BDF2 inertia, NaN scan and the J.v
//                  difference-quotient epilogue.  Internal faces are evaluated with the
//                  owner/neighbour operands in the reference's order and negated on the
//                  neighbour side, so every cell sums exactly the terms the reference
//                  adds, in the same order: bit-identical R(u) (no atomics, deterministic).
//
// This translation unit is compiled with -fmad=false: the reference build has no FMA
// (baseline x86-64), and contraction would change the rounding of every term.
#include <algorithm>
#include <cfloat>
#include <cstdint>
#include <climits>

#include "device.h"
#include "sfv_case.h"

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
__device__ __forceinline__ dm3 mmul(const dm3& a, const dm3& b) {  // types.hpp:72-81
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
__device__ __forceinline__ d3 dot_left(d3 v, const dm3& a) {  // types.hpp:91-96
    return {v.x * a.a[0][0] + v.y * a.a[1][0] + v.z * a.a[2][0], v.x * a.a[0][1] + v.y * a.a[1][1] + v.z * a.a[2][1],
            v.x * a.a[0][2] + v.y * a.a[1][2] + v.z * a.a[2][2]};
}
__device__ __forceinline__ double det(const dm3& a) {  // types.hpp:127-131
    return a.a[0][0] * (a.a[1][1] * a.a[2][2] - a.a[1][2] * a.a[2][1]) -
           a.a[0][1] * (a.a[1][0] * a.a[2][2] - a.a[1][2] * a.a[2][0]) +
           a.a[0][2] * (a.a[1][0] * a.a[2][1] - a.a[1][1] * a.a[2][0]);
}
__device__ __forceinline__ dm3 inverse(const dm3& a) {  // types.hpp:133-148
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
__device__ __forceinline__ dm3 interp(const dm3& p, const dm3& n, double w) {  // fields.hpp:49-52
    return madd(mscl(p, w), mscl(n, 1.0 - w));
}
__device__ __forceinline__ dm3 defgrad(const dm3& g) {  // F = I + grad^T
    dm3 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) r.a[i][j] = (i == j ? 1.0 : 0.0) + g.a[j][i];
    return r;
}
__device__ __forceinline__ dm3 reflection(d3 gamma) {  // reflection(normal), mesh.cpp:389, :450
    const d3 n = scl(gamma, 1.0 / nrm(gamma));
    dm3 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) r.a[i][j] = (i == j ? 1.0 : 0.0) - (cmp(n, i) * cmp(n, j)) * 2.0;
    return r;
}
__device__ __forceinline__ dm3 mirror_avg(const dm3& a, const dm3& R) {  // 0.5 (A + R A R)
    return mscl(madd(a, mmul(mmul(R, a), R)), 0.5);
}

// hooke_stress (laws.cpp:20-27)
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

// neo_hookean_stress via kinematics (laws.cpp:9-18, :39-47); ok=false when det F <= 0
__device__ __forceinline__ dm3 neo_hookean(const dm3& g, double mu, double kappa, bool& ok) {
    const dm3 F = defgrad(g);
    const double J = det(F);
    ok = J > 0.0;
    const dm3 bb = mscl(mmul(F, mtr(F)), pow(J, -2.0 / 3.0));
    const double t = ((bb.a[0][0] + bb.a[1][1]) + bb.a[2][2]) / 3.0;  // dev (types.hpp:118-125)
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

// rhie_chow_face (discretisation.cpp:33-37)
__device__ __forceinline__ d3 rhie_chow(d3 up, d3 uo, const dm3& gf, d3 delta, double d_mag, double area_mag,
                                        double alpha, double kbar) {
    const d3 compact = scl(sub(uo, up), nrm(delta) / d_mag);
    return scl(sub(compact, dot_left(delta, gf)), alpha * kbar * area_mag);
}

// transform_area (discretisation.cpp:100-104)
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
__device__ __forceinline__ d3 ldsoa(const double* __restrict__ p, int n, int i) {
    return {p[i], p[n + i], p[2 * n + i]};
}
__device__ __forceinline__ dm3 ldG(const double* __restrict__ G, int nc, int c) {
    dm3 g;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) g.a[i][j] = G[(3 * i + j) * static_cast<size_t>(nc) + c];
    return g;
}

constexpr int kSign = 0x80000000;

// ---------------------------------------------------------------- gradient pass
template <bool PERT>
__global__ void __launch_bounds__(256) grad_kernel(DevMesh m, PatchTable pt, const double* __restrict__ u,
                                                   const double* __restrict__ v, const double* __restrict__ eps_p,
                                                   double* __restrict__ G) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= m.nc) return;
    const double eps = PERT ? *eps_p : 0.0;
    const d3 uc = load_u<PERT>(u, v, eps, c);
    dm3 g;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) g.a[i][j] = 0.0;
    for (int s = 0; s < m.slots; ++s) {
        const size_t si = static_cast<size_t>(s) * m.nc + c;
        const int o = m.slot_other[si];
        d3 du;
        if (o >= 0) {
            du = sub(load_u<PERT>(u, v, eps, o), uc);
        } else if (o <= -2 && pt.kind[-o - 2] == SFV_PATCH_SYMMETRY) {
            const int f = m.slot_face[si] & ~kSign;
            const dm3 R = reflection(ldsoa(m.gam, m.nf, f));
            du = sub(mv(R, uc), uc);
        } else {
            continue;  // traction / displacement faces are not in the stencil; padding
        }
        const d3 ls = {m.slot_ls[(3 * static_cast<size_t>(s)) * m.nc + c],
                       m.slot_ls[(3 * static_cast<size_t>(s) + 1) * m.nc + c],
                       m.slot_ls[(3 * static_cast<size_t>(s) + 2) * m.nc + c]};
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) g.a[i][j] += cmp(ls, i) * cmp(du, j);
    }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) G[(3 * i + j) * static_cast<size_t>(m.nc) + c] = g.a[i][j];
}

// ---------------------------------------------------------------- flux pass
template <bool PERT, int S>
__global__ void __launch_bounds__(128) flux_kernel(DevMesh m, Physics ph, PatchTable pt, History hist,
                                                   const double* __restrict__ u, const double* __restrict__ v,
                                                   const double* __restrict__ eps_p, const double* __restrict__ G,
                                                   const double* __restrict__ r_u, double* __restrict__ out,
                                                   ErrWords* __restrict__ err) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= m.nc) return;
    const double eps = PERT ? *eps_p : 0.0;
    if (PERT && eps == 0.0) {  // |v| = 0 short-circuit (nonlinear.cpp:110)
        out[3 * c] = 0.0;
        out[3 * c + 1] = 0.0;
        out[3 * c + 2] = 0.0;
        return;
    }
    const d3 uc = load_u<PERT>(u, v, eps, c);
    const dm3 gc = ldG(G, m.nc, c);
    bool ok_c;
    const dm3 sc = stress(ph, gc, ok_c);
    if (!ok_c) atomicMin(&err->inverted_cell, c);
    d3 r = {0.0, 0.0, 0.0};
    d3 st[S];
    bool has_st[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        has_st[s] = false;
        st[s] = {0.0, 0.0, 0.0};
        if (s >= m.slots) continue;
        const size_t si = static_cast<size_t>(s) * m.nc + c;
        const int fr = m.slot_face[si];
        if (fr == -1) continue;
        const int f = fr & ~kSign;
        const int o = m.slot_other[si];
        const d3 gam = ldsoa(m.gam, m.nf, f);
        if (o >= 0) {
            // internal face: operands in owner/neighbour order, negated on the neighbour side
            const bool is_nb = (fr & kSign) != 0;
            const double w = m.w[f];
            const dm3 go = ldG(G, m.nc, o);
            bool ok_o;
            const dm3 so = stress(ph, go, ok_o);
            const dm3& sP = is_nb ? so : sc;
            const dm3& sN = is_nb ? sc : so;
            d3 gm = gam;
            if (ph.tl) {
                bool ok;
                const dm3 fP = defgrad(is_nb ? go : gc), fN = defgrad(is_nb ? gc : go);
                gm = transform_area(gam, interp(fP, fN, w), ok);
                if (!ok) atomicMin(&err->inverted_face, f);
            }
            const d3 flux = dot_left(gm, interp(sP, sN, w));
            if (!ph.stab_only) r = is_nb ? sub(r, flux) : add(r, flux);
            const d3 uo = load_u<PERT>(u, v, eps, o);
            const dm3 gf = is_nb ? interp(go, gc, w) : interp(gc, go, w);
            const d3 dp = is_nb ? rhie_chow(uo, uc, gf, ldsoa(m.del, m.nf, f), m.dmag[f], nrm(gam), ph.alpha, ph.kbar)
                                : rhie_chow(uc, uo, gf, ldsoa(m.del, m.nf, f), m.dmag[f], nrm(gam), ph.alpha, ph.kbar);
            st[s] = is_nb ? neg(dp) : dp;
            has_st[s] = true;
            continue;
        }
        const int patch = -o - 2;
        const int kind = pt.kind[patch];
        const d3 bc = {pt.value[patch][0], pt.value[patch][1], pt.value[patch][2]};
        if (kind == SFV_PATCH_DISPLACEMENT) {
            d3 gm = gam;
            if (ph.tl) {
                bool ok;
                gm = transform_area(gam, defgrad(gc), ok);
                if (!ok) atomicMin(&err->inverted_face, f);
            }
            if (!ph.stab_only) r = add(r, dot_left(gm, sc));
            st[s] = rhie_chow(uc, bc, gc, ldsoa(m.del, m.nf, f), m.dmag[f], nrm(gam), ph.alpha, ph.kbar);
            has_st[s] = true;
        } else if (kind == SFV_PATCH_SYMMETRY) {
            const dm3 R = reflection(gam);
            d3 gm = gam;
            if (ph.tl) {
                bool ok;
                gm = transform_area(gam, mirror_avg(defgrad(gc), R), ok);
                if (!ok) atomicMin(&err->inverted_face, f);
            }
            if (!ph.stab_only) r = add(r, dot_left(gm, mirror_avg(sc, R)));
            st[s] = rhie_chow(uc, mv(R, uc), mirror_avg(gc, R), ldsoa(m.del, m.nf, f), m.dmag[f], nrm(gam), ph.alpha,
                              ph.kbar);
            has_st[s] = true;
        } else if (!ph.stab_only) {  // traction: nominal load |Gamma| T (discretisation.cpp:151-154)
            r = add(r, scl(bc, nrm(gam)));
        }
    }
    // add_stabilisation runs after the whole flux loop (discretisation.cpp:158)
#pragma unroll
    for (int s = 0; s < S; ++s)
        if (has_st[s]) r = add(r, st[s]);
    if (ph.transient && !ph.stab_only) {  // BDF2 inertia (discretisation.cpp:48-57, :163-169)
        const double idt = 1.0 / (2.0 * ph.dt);
        const d3 ut = ld3(hist.u_old, c), utm1 = ld3(hist.u_old_old, c);
        const d3 vt = ld3(hist.v_old, c), vtm1 = ld3(hist.v_old_old, c);
        const d3 vn = scl(add(sub(scl(uc, 3.0), scl(ut, 4.0)), utm1), idt);
        const d3 a = scl(add(sub(scl(vn, 3.0), scl(vt, 4.0)), vtm1), idt);
        r = sub(r, scl(a, ph.rho * m.volume[c]));
    }
    if (!ph.stab_only && !fin(r)) atomicMin(&err->nan_cell, c);
    if constexpr (PERT) {  // (R(u + eps v) - R(u)) / eps (nonlinear.cpp:132-136)
        const double o0 = (r.x - r_u[3 * c]) / eps, o1 = (r.y - r_u[3 * c + 1]) / eps,
                     o2 = (r.z - r_u[3 * c + 2]) / eps;
        if (!(isfinite(o0) && isfinite(o1) && isfinite(o2))) atomicMin(&err->nan_jv, c);
        out[3 * c] = o0;
        out[3 * c + 1] = o1;
        out[3 * c + 2] = o2;
    } else {
        out[3 * c] = r.x;
        out[3 * c + 1] = r.y;
        out[3 * c + 2] = r.z;
    }
}

// |u|^2 and |v|^2 with a fixed-order two-level reduction, then eps (nonlinear.cpp:109-115).
// 16-byte loads, 8 of them in flight per thread, warp-shuffle block sums; the last block
// to finish (one atomic per block) sums the block partials in block order.
constexpr int kRedThreads = 512;

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    return x;
}
// fixed-order block sum of two values (lane 0 of warp 0 holds the result)
__device__ __forceinline__ void block_sum2(double& a, double& b, double* sh) {
    a = warp_sum(a);
    b = warp_sum(b);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sh[2 * w] = a;
        sh[2 * w + 1] = b;
    }
    __syncthreads();
    if (w == 0) {
        a = l < kRedThreads / 32 ? sh[2 * l] : 0.0;
        b = l < kRedThreads / 32 ? sh[2 * l + 1] : 0.0;
        a = warp_sum(a);
        b = warp_sum(b);
    }
}

// VEC: both vectors 16-byte aligned (a GMRES basis vector V + j n is not when n is odd)
template <bool VEC>
__global__ void __launch_bounds__(kRedThreads) jv_eps_kernel(const double* __restrict__ u, const double* __restrict__ v,
                                                            int n, double* __restrict__ partial,
                                                            unsigned* __restrict__ counter, double* __restrict__ eps_out,
                                                            double* __restrict__ u_norm, bool cached) {
    __shared__ double sh[2 * kRedThreads / 32];
    __shared__ bool last;
    double au = 0.0, av = 0.0;
    const int st = gridDim.x * blockDim.x;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (!VEC) {
        for (; i + 7 * st < n; i += 8 * st) {  // 8 iterations' loads together
            double x[8], y[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                y[k] = v[i + k * st];
                x[k] = cached ? 0.0 : u[i + k * st];
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                av += y[k] * y[k];
                if (!cached) au += x[k] * x[k];
            }
        }
        for (; i < n; i += st) {
            av += v[i] * v[i];
            if (!cached) au += u[i] * u[i];
        }
    }
    const int n2 = VEC ? n / 2 : 0;  // double2 elements
    const double2* u2 = reinterpret_cast<const double2*>(u);
    const double2* v2 = reinterpret_cast<const double2*>(v);
    for (; i + 3 * st < n2; i += 4 * st) {
        double2 x[4], y[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            y[k] = v2[i + k * st];
            x[k] = cached ? make_double2(0.0, 0.0) : u2[i + k * st];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            av += y[k].x * y[k].x;
            av += y[k].y * y[k].y;
            if (!cached) {
                au += x[k].x * x[k].x;
                au += x[k].y * x[k].y;
            }
        }
    }
    for (; i < n2; i += st) {
        const double2 y = v2[i];
        av += y.x * y.x;
        av += y.y * y.y;
        if (!cached) {
            const double2 x = u2[i];
            au += x.x * x.x;
            au += x.y * x.y;
        }
    }
    if (VEC && blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) {  // odd tail
        av += v[n - 1] * v[n - 1];
        if (!cached) au += u[n - 1] * u[n - 1];
    }
    block_sum2(au, av, sh);
    if (threadIdx.x == 0) {
        partial[2 * blockIdx.x] = au;
        partial[2 * blockIdx.x + 1] = av;
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double tu = 0.0, tv = 0.0;
    for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
        tu += __ldcg(&partial[2 * b]);
        tv += __ldcg(&partial[2 * b + 1]);
    }
    __syncthreads();
    block_sum2(tu, tv, sh);
    if (threadIdx.x == 0) {
        const double vn = sqrt(tv);
        const double un = cached ? *u_norm : sqrt(tu);
        if (!cached) *u_norm = un;
        *eps_out = vn == 0.0 ? 0.0 : sqrt(DBL_EPSILON) * sqrt(1.0 + un) / vn;
        *counter = 0u;
    }
}

// |u|^2, |v|^2 block partials only (the jv_pair.cu perturb pass finishes the reduction)
template <bool VEC>
__global__ void __launch_bounds__(kRedThreads) norm_partials_kernel(const double* __restrict__ u,
                                                                   const double* __restrict__ v, int n,
                                                                   double* __restrict__ partial, bool cached) {
    __shared__ double sh[2 * kRedThreads / 32];
    double au = 0.0, av = 0.0;
    const int st = gridDim.x * blockDim.x;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (!VEC) {
        for (; i + 7 * st < n; i += 8 * st) {
            double x[8], y[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                y[k] = v[i + k * st];
                x[k] = cached ? 0.0 : u[i + k * st];
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                av += y[k] * y[k];
                if (!cached) au += x[k] * x[k];
            }
        }
        for (; i < n; i += st) {
            av += v[i] * v[i];
            if (!cached) au += u[i] * u[i];
        }
    }
    const int n2 = VEC ? n / 2 : 0;
    const double2* u2 = reinterpret_cast<const double2*>(u);
    const double2* v2 = reinterpret_cast<const double2*>(v);
    for (; i + 3 * st < n2; i += 4 * st) {
        double2 x[4], y[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            y[k] = v2[i + k * st];
            x[k] = cached ? make_double2(0.0, 0.0) : u2[i + k * st];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            av += y[k].x * y[k].x;
            av += y[k].y * y[k].y;
            if (!cached) {
                au += x[k].x * x[k].x;
                au += x[k].y * x[k].y;
            }
        }
    }
    for (; i < n2; i += st) {
        const double2 y = v2[i];
        av += y.x * y.x;
        av += y.y * y.y;
        if (!cached) {
            const double2 x = u2[i];
            au += x.x * x.x;
            au += x.y * x.y;
        }
    }
    if (VEC && blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) {
        av += v[n - 1] * v[n - 1];
        if (!cached) au += u[n - 1] * u[n - 1];
    }
    block_sum2(au, av, sh);
    if (threadIdx.x == 0) {
        partial[2 * blockIdx.x] = au;
        partial[2 * blockIdx.x + 1] = av;
    }
}

}  // namespace

void launch_residual(const DevMesh& m, const Physics& ph, const PatchTable& pt, const History& hist, const double* u,
                     const double* v, const double* jv_eps, const double* r_u, double* out, double* grad_scratch,
                     ErrWords* err, cudaStream_t s) {
    const int tg = 256, tf = 128;
    const int bg = (m.nc + tg - 1) / tg, bf = (m.nc + tf - 1) / tf;
    const bool pert = jv_eps != nullptr;
    if (pert)
        grad_kernel<true><<<bg, tg, 0, s>>>(m, pt, u, v, jv_eps, grad_scratch);
    else
        grad_kernel<false><<<bg, tg, 0, s>>>(m, pt, u, v, jv_eps, grad_scratch);
#define SFV_FLUX(S)                                                                                              \
    do {                                                                                                         \
        if (pert)                                                                                                \
            flux_kernel<true, S><<<bf, tf, 0, s>>>(m, ph, pt, hist, u, v, jv_eps, grad_scratch, r_u, out, err);  \
        else                                                                                                     \
            flux_kernel<false, S><<<bf, tf, 0, s>>>(m, ph, pt, hist, u, v, jv_eps, grad_scratch, r_u, out, err); \
    } while (0)
    if (m.slots <= 4)
        SFV_FLUX(4);
    else if (m.slots <= 6)
        SFV_FLUX(6);
    else
        SFV_FLUX(8);
#undef SFV_FLUX
}

void launch_gradients(const DevMesh& m, const PatchTable& pt, const double* u, double* G, cudaStream_t s) {
    grad_kernel<false><<<(m.nc + 255) / 256, 256, 0, s>>>(m, pt, u, nullptr, nullptr, G);
}

int launch_norm_partials(const double* u, const double* v, int n, double* partial, bool u_norm_cached,
                         cudaStream_t s) {
    static const int sms = [] {
        int dev = 0, x = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&x, cudaDevAttrMultiProcessorCount, dev);
        return std::max(1, std::min(x, 148 * 2));
    }();
    const int blocks = std::max(1, std::min(4 * sms, (n / 2 + kRedThreads - 1) / kRedThreads));
    const bool vec = ((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
    if (vec) norm_partials_kernel<true><<<blocks, kRedThreads, 0, s>>>(u, v, n, partial, u_norm_cached);
    else norm_partials_kernel<false><<<blocks, kRedThreads, 0, s>>>(u, v, n, partial, u_norm_cached);
    return blocks;
}

void launch_jv_eps(const double* u, const double* v, int n, double* scratch, unsigned* counter, double* eps_out,
                   double* u_norm_inout, bool u_norm_cached, cudaStream_t s) {
    static const int sms = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return std::max(1, std::min(v, 148 * 2));
    }();
    const int blocks = std::max(1, std::min(4 * sms, (n / 2 + kRedThreads - 1) / kRedThreads));
    const bool vec = ((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
    if (vec)
        jv_eps_kernel<true><<<blocks, kRedThreads, 0, s>>>(u, v, n, scratch, counter, eps_out, u_norm_inout,
                                                           u_norm_cached);
    else
        jv_eps_kernel<false><<<blocks, kRedThreads, 0, s>>>(u, v, n, scratch, counter, eps_out, u_norm_inout,
                                                            u_norm_cached);
}

}  // namespace sfv
