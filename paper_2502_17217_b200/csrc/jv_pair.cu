// jv_pair.cu — residual / J.v as two sync-free kernels with one thread per (cell, face slot).
//
// The reference evaluates R(u) cell by cell: gradients (discretisation.cpp:10-31), then
// for every face the interpolated-stress flux (:121-156) and, after the whole face loop,
// the Rhie-Chow terms (:158, :176-208), then the BDF2 inertia and the NaN scan
// (:163-172).  Here a CTA owns kCells consecutive cells and runs one warp per face slot:
// lane l of warp s evaluates slot s of cell (base + l).  Every per-face load of a thread
// is independent of the others (only the slot's face index and other cell come first),
// so a warp keeps ~40 loads in flight with no cross-CTA synchronisation at all.  The
// per-face results go to shared memory and the ordered per-cell sums — fluxes in
// ascending face order, then stabilisation terms in the same order, exactly the
// reference's summation order — are done by 3 x kCells threads, one per (component,
// cell), whose output stores are fully coalesced.
//
// Internal faces are evaluated from both sides with the operands in (owner, neighbour)
// order and the result negated on the neighbour side, which is bit-identical to the
// reference's r[N] -= flux.  Compiled with -fmad=false (see residual.cu).
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdlib>

#include <cooperative_groups.h>

#include "device.h"
#include "face_math.cuh"
#include "sfv_case.h"

namespace sfv {
namespace {

namespace cg = cooperative_groups;

using namespace fm;

constexpr int kCells = 32;  // cells per CTA (one warp-width); CTA = kCells x S threads
constexpr int kSign = static_cast<int>(0x80000000u);

// Tiled tables (device.h): entry q of cell (face) c at tiled(c, nq) + 32 q.  One base
// address per gathered record, the field offsets are immediates (no per-load IMADs).
__device__ __forceinline__ d3 ld3(const double* __restrict__ p) { return {p[0], p[32], p[64]}; }
// face record of face f: Gamma (rows 0-2), Delta (3-5), |Delta|/|d|, |Gamma|, w
__device__ __forceinline__ const double* face_rec(const DevMesh& m, int f) { return m.tf9 + tiled(f, 9); }
// Streams read once per pass (slot tables, least-squares vectors, r_u) are loaded with
// evict-first (ld.global.cs) so that the gathered w and G (~96 MB at 1M cells) stay in L2.
// The 32 lanes of a warp (32 consecutive cells, one face slot) load 32 consecutive values
// per instruction: the L1 wavefront queue, not DRAM, limits a gather kernel whose loads
// each touch many 128-byte lines.
// w and G are written with an L2 evict-last policy: their consumers gather them within
// the next two kernels, after ~170 MB of streamed least-squares vectors and slot tables.
__device__ __forceinline__ unsigned long long evict_last_policy() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_keep(double* a, double v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
// [w | G] record of cell c: w xyz (rows 0-2), G row-major (rows 3-11, q = 3 i + j)
__device__ __forceinline__ const double* wg_rec(const double* __restrict__ wg, int c) { return wg + tiled(c, kWG); }
__device__ __forceinline__ void ldg9(const double* __restrict__ r, double* g) {
#pragma unroll
    for (int q = 0; q < 9; ++q) g[q] = r[32 * (3 + q)];
}
__device__ __forceinline__ dm3 ldG(const double* __restrict__ r) {
    dm3 a;
#pragma unroll
    for (int q = 0; q < 9; ++q) a.a[q / 3][q % 3] = r[32 * (3 + q)];
    return a;
}

#ifndef SFV_HOOKE_CTAS
#define SFV_HOOKE_CTAS 4  // resident 6-warp CTAs per SM the Hooke face pass is compiled for
#endif
#ifndef SFV_OWN_ASYNC
#define SFV_OWN_ASYNC 0  // 1: a tile's own [w | G] records staged in shared memory (measured slower on hexes)
#endif
#ifndef SFV_GEN_CTAS
#define SFV_GEN_CTAS 2  // resident 6-warp CTAs per SM the non-Hooke / TL face pass is compiled for
#endif

// programmatic dependent launch (see launch_win)
__device__ __forceinline__ void wait_predecessor() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#ifndef SFV_PDL_EARLY
#define SFV_PDL_EARLY 0  // 1: trigger dependents at kernel entry, 0: after the CTA's stores (measured better)
#endif
__device__ __forceinline__ void release_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void release_early() {
    if (SFV_PDL_EARLY) release_dependents();
}
__device__ __forceinline__ void release_late() {
    if (!SFV_PDL_EARLY) release_dependents();
}

// cell stress, all 9 entries (grad_cell_kernel<S, true>), tiled record: F S F^T of St.
// Venant-Kirchhoff / Guccione is symmetric only up to rounding, so nothing is mirrored
__device__ __forceinline__ dm3 ld_sig(const double* __restrict__ r) {
    dm3 a;
#pragma unroll
    for (int q = 0; q < 9; ++q) a.a[q / 3][q % 3] = r[32 * q];
    return a;
}

// ---------------------------------------------------------------- perturbed state
// w = u + eps v, formed once per J.v exactly as the reference forms u_pert
// (nonlinear.cpp:116-118); plain residual: w = u.
// ε from the block partials of ‖u‖², ‖v‖² (launch_norm_partials): every block sums them in
// the same fixed order, so all blocks hold the same bits; block 0 publishes ε (and ‖u‖).
// Replaces a last-block finalisation (atomics and a serial tail) on the J·v critical path.
__device__ __forceinline__ double eps_from_partials(const double* __restrict__ part, int np, double* __restrict__ u_norm,
                                                    bool cached, double* sh, int nthr = 0) {
    double tu = 0.0, tv = 0.0;
    const int nt = nthr ? nthr : blockDim.x;
    if (threadIdx.x < nt)
    for (int b = threadIdx.x; b < np; b += nt) {
        tu += __ldcg(&part[2 * b]);
        tv += __ldcg(&part[2 * b + 1]);
    }
    // fixed-order block sums (warp shuffles, then warps in order)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        tu += __shfl_down_sync(0xffffffffu, tu, o);
        tv += __shfl_down_sync(0xffffffffu, tv, o);
    }
    const int wi = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (l == 0) {
        sh[2 * wi] = tu;
        sh[2 * wi + 1] = tv;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double su = 0.0, sv = 0.0;
        for (int k = 0; k < nw; ++k) {
            su += sh[2 * k];
            sv += sh[2 * k + 1];
        }
        const double vn = sqrt(sv);
        const double un = cached ? *u_norm : sqrt(su);
        sh[2 * nw] = vn == 0.0 ? 0.0 : sqrt(DBL_EPSILON) * sqrt(1.0 + un) / vn;  // nonlinear.cpp:109-115
        sh[2 * nw + 1] = un;
    }
    __syncthreads();
    return sh[2 * nw];
}

template <bool PERT>
__global__ void __launch_bounds__(256) perturb_kernel(int nc, const double* __restrict__ u, const double* __restrict__ v,
                                                      double* __restrict__ eps_p, double* __restrict__ wg,
                                                      const double* __restrict__ part, int np,
                                                      double* __restrict__ u_norm, bool cached) {
    __shared__ double sh[2 * 8 + 2];
    release_early();
    wait_predecessor();  // ‖u‖² / ‖v‖² partials (or a given ε), and the previous pass that read w
    double eps = 0.0;
    if (PERT) {
        if (part) {
            eps = eps_from_partials(part, np, u_norm, cached, sh);
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                *eps_p = eps;
                if (!cached) *u_norm = sh[2 * (blockDim.x >> 5) + 1];
            }
        } else {
            eps = *eps_p;
        }
    }
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x) {
        double x = u[3 * c], y = u[3 * c + 1], z = u[3 * c + 2];
        if (PERT) {
            x = x + eps * v[3 * c];
            y = y + eps * v[3 * c + 1];
            z = z + eps * v[3 * c + 2];
        }
        const unsigned long long pol = evict_last_policy();
        double* r = wg + tiled(c, kWG);
        st_keep(r, x, pol);
        st_keep(r + 32, y, pol);
        st_keep(r + 64, z, pol);
    }
    release_late();
}

// ε and w = u + εv in one launch: the grid (all CTAs resident) reduces ‖u‖², ‖v‖² to fixed-order
// block partials, meets at a grid barrier, and every block finishes ε from the partials in
// the same order (so all hold the same bits) and forms w.  u and v are read from HBM once;
// the second read hits L2 (48 MB at 1M cells).  Replaces launch_norm_partials + perturb.
// The reduction is the one of launch_norm_partials + perturb_kernel operation for operation
// (same grid, per-thread strides, block trees and final partial sum), so ε — and with it
// every Krylov and Newton decision — is bitwise what the two-launch path computes.
constexpr int kEpT = 512;
template <bool VEC>  // VEC: u and v 16-byte aligned (double2 loads)
__global__ void __launch_bounds__(kEpT, 4) eps_perturb_kernel(int nc, const double* __restrict__ u,
                                                          const double* __restrict__ v, double* __restrict__ eps_p,
                                                          double* __restrict__ wg, double* __restrict__ part,
                                                          double* __restrict__ u_norm, bool cached,
                                                          const int* __restrict__ vj, long long vstride) {
    __shared__ double sh[2 * (kEpT / 32) + 2];
    release_early();
    wait_predecessor();  // u, v, and the previous pass that read w
    if (vj) v += static_cast<size_t>(*vj) * vstride;  // v = V[j], j on the device (GMRES cycle graph)
    const int n2 = VEC ? 3 * nc / 2 : 0;  // double2 elements of u and v (3 nc is even, or the tail below)
    const double2* u2 = reinterpret_cast<const double2*>(u);
    const double2* v2 = reinterpret_cast<const double2*>(v);
    const int st = gridDim.x * blockDim.x;
    double au = 0.0, av = 0.0;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (!VEC) {
        for (; i < 3 * nc; i += st) {
            av += v[i] * v[i];
            if (!cached) au += u[i] * u[i];
        }
    }
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
    if (VEC && (3 * nc) % 2 != 0 && blockIdx.x == 0 && threadIdx.x == 0) {  // odd length: last entry
        const double y = v[3 * nc - 1];
        av += y * y;
        if (!cached) au += u[3 * nc - 1] * u[3 * nc - 1];
    }
    // block tree of norm_partials_kernel (residual.cu block_sum2): warp shuffles, then warp 0
    // shuffles the 16 warp sums
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        au += __shfl_down_sync(0xffffffffu, au, o);
        av += __shfl_down_sync(0xffffffffu, av, o);
    }
    const int wi = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sh[2 * wi] = au;
        sh[2 * wi + 1] = av;
    }
    __syncthreads();
    if (wi == 0) {
        au = l < kEpT / 32 ? sh[2 * l] : 0.0;
        av = l < kEpT / 32 ? sh[2 * l + 1] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            au += __shfl_down_sync(0xffffffffu, au, o);
            av += __shfl_down_sync(0xffffffffu, av, o);
        }
    }
    __syncthreads();  // sh is reused below
    if (threadIdx.x == 0) {
        __stcg(&part[2 * blockIdx.x], au);
        __stcg(&part[2 * blockIdx.x + 1], av);
    }
    // grid barrier: the launch is cooperative (launch_eps_perturb), so every CTA is resident
    // or the launch is refused; the barrier state is the runtime's, per launch
    cg::this_grid().sync();
    // perturb_kernel's final sum ran on 256-thread blocks: threads >= 256 contribute +0.0
    // after the 8 warp sums, which leaves every value unchanged
    const double eps = eps_from_partials(part, gridDim.x, u_norm, cached, sh, 256);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *eps_p = eps;
        if (!cached) *u_norm = sh[2 * (kEpT >> 5) + 1];
    }
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += st) {
        const double x = u[3 * c] + eps * v[3 * c];
        const double y = u[3 * c + 1] + eps * v[3 * c + 1];
        const double z = u[3 * c + 2] + eps * v[3 * c + 2];
        const unsigned long long pol = evict_last_policy();
        double* r = wg + tiled(c, kWG);
        st_keep(r, x, pol);
        st_keep(r + 32, y, pol);
        st_keep(r + 64, z, pol);
    }
    release_late();
}

// launch_norm_partials' grid, or 0 when it cannot be co-resident (then the two-launch path runs)
int eps_perturb_grid(int nc) {
    static int sms = -1, resident = 0;
    if (sms < 0) {
        int dev = 0, a = 0, b = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, eps_perturb_kernel<true>, kEpT, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, eps_perturb_kernel<false>, kEpT, 0);
        resident = std::min(a, b) * sms;
    }
    const int n = 3 * nc;
    const int want = std::max(1, std::min(4 * std::max(1, std::min(sms, 148 * 2)), (n / 2 + kEpT - 1) / kEpT));
    return want <= resident ? want : 0;
}

// ---------------------------------------------------------------- gradients
// one thread per cell, slots unrolled so the neighbour loads are all in flight together
// (discretisation.cpp:10-31: g += ls_f (x) (u_N - u_P), faces in cell order)
// GEN (non-Hooke law or total Lagrangian): the cell's stress sigma(G_c) is evaluated here
// once (laws.cpp; the stress loop of discretisation.cpp:116-119, which also reports an
// inverted cell, or the Guccione exponent overflow) and stored, instead of twice per face
// in the flux pass — same function on the same G, so the same bits.
// J2: the stress is the radial return from the cell's committed state (J2PlasticLaw::stress,
// laws.cpp:201-212); with ph.commit set the trial state replaces it (ResidualEvaluator::commit,
// discretisation.cpp:91-95 — each cell reads and writes only its own record).
// HOIST (every law but J2): the least-squares vectors — the largest stream of the pass,
// independent of the predecessor — are loaded together with the slot indices before
// griddepcontrol.wait, so all 18 are in flight with the 6 neighbour gathers (110 instead of
// 76 registers, 16 instead of 24 resident warps; J.v at C2 0.193-0.210 -> 0.180 ms, C3
// 0.166 -> 0.150, C4 0.234 -> 0.204).
template <int S, bool GEN, bool J2 = false, bool HOIST = false>
__global__ void __launch_bounds__(256) grad_cell_kernel(DevMesh m, PatchTable pt, Physics ph, double* __restrict__ wg,
                                                        double* __restrict__ sig, double* __restrict__ lawst,
                                                        ErrWords* __restrict__ err) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= m.nc) return;
    release_early();
    const int* ts = m.tslot + tiled(c, 2 * S);
    const double* tl = m.tls + tiled(c, 3 * S);
    int o[S];
#pragma unroll
    for (int s = 0; s < S; ++s) o[s] = __ldcs(ts + 32 * (S + s));  // padding slots hold -1
    d3 lsv[HOIST ? S : 1];
    if constexpr (HOIST) {
#pragma unroll
        for (int s = 0; s < S; ++s)
            lsv[s] = {__ldcs(tl + 32 * (3 * s)), __ldcs(tl + 32 * (3 * s + 1)), __ldcs(tl + 32 * (3 * s + 2))};
    }
    wait_predecessor();  // w
    double* rc = wg + tiled(c, kWG);
    const d3 wc = ld3(rc);
    d3 wn[S];
#pragma unroll
    for (int s = 0; s < S; ++s) wn[s] = o[s] >= 0 ? ld3(wg_rec(wg, o[s])) : d3{0.0, 0.0, 0.0};
    double g[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) g[q] = 0.0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        d3 du;
        if (o[s] >= 0) {
            du = sub(wn[s], wc);
        } else if (o[s] <= -2 && pt.kind[-o[s] - 2] == SFV_PATCH_SYMMETRY) {
            const dm3 R = reflection(ld3(face_rec(m, ts[32 * s] & ~kSign)));
            du = sub(mv(R, wc), wc);
        } else {
            continue;  // traction / displacement faces are not in the stencil; padding
        }
        d3 ls;
        if constexpr (HOIST) ls = lsv[s];
        else ls = {__ldcs(tl + 32 * (3 * s)), __ldcs(tl + 32 * (3 * s + 1)), __ldcs(tl + 32 * (3 * s + 2))};
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) g[3 * i + j] += cmp(ls, i) * cmp(du, j);
    }
    const unsigned long long pol = evict_last_policy();
#pragma unroll
    for (int q = 0; q < 9; ++q) st_keep(rc + 32 * (3 + q), g[q], pol);
    if (GEN) {
        dm3 gm;
#pragma unroll
        for (int q = 0; q < 9; ++q) gm.a[q / 3][q % 3] = g[q];
        int code;
        dm3 sc;
        if constexpr (J2) {
            double* rst = lawst + tiled(c, kJ2);
            double st[kJ2], nst[kJ2];
#pragma unroll
            for (int q = 0; q < kJ2; ++q) st[q] = rst[32 * q];
            sc = j2_return(gm, st, ph, code, nst);
            if (ph.commit && code == 0)
#pragma unroll
                for (int q = 0; q < kJ2; ++q) rst[32 * q] = nst[q];
        } else {
            sc = stress_code(ph, gm, code);
        }
        if (code == 1) atomicMin(&err->inverted_cell, c);
        if (code == 2) atomicMin(&err->overflow_cell, c);
        if (code == 3) atomicMin(&err->retmap_cell, c);
        double* rs = sig + tiled(c, kSig);
#pragma unroll
        for (int q = 0; q < 9; ++q) st_keep(rs + 32 * q, sc.a[q / 3][q % 3], pol);
    }
    release_late();
}

// One cell's gradient with exactly grad_cell_kernel's operations (slots in face order), for
// the boundary pass, which then needs w only and can run beside the gradient pass.
__device__ __forceinline__ dm3 cell_gradient_at(const DevMesh& m, const PatchTable& pt, const double* __restrict__ wg,
                                                int c) {
    const int* ts = m.tslot + tiled(c, 2 * m.spad);
    const double* tl = m.tls + tiled(c, 3 * m.spad);
    const d3 wc = ld3(wg_rec(wg, c));
    double g[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) g[q] = 0.0;
    for (int s = 0; s < m.slots; ++s) {
        const int o = ts[32 * (m.spad + s)];
        d3 du;
        if (o >= 0) {
            du = sub(ld3(wg_rec(wg, o)), wc);
        } else if (o <= -2 && pt.kind[-o - 2] == SFV_PATCH_SYMMETRY) {
            const dm3 R = reflection(ld3(face_rec(m, ts[32 * s] & ~kSign)));
            du = sub(mv(R, wc), wc);
        } else {
            continue;
        }
        const d3 ls = {tl[32 * (3 * s)], tl[32 * (3 * s + 1)], tl[32 * (3 * s + 2)]};
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) g[3 * i + j] += cmp(ls, i) * cmp(du, j);
    }
    dm3 r;
#pragma unroll
    for (int q = 0; q < 9; ++q) r.a[q / 3][q % 3] = g[q];
    return r;
}

// ---------------------------------------------------------------- boundary faces
// One thread per boundary face (face f = nint + fb, bnd_cs[fb] = cell * 8 + slot):
// flux and stabilisation term into bres[q * nbf + fb] (discretisation.cpp:128-154, :186-205).
// Kept out of the per-slot kernel so its register budget is set by the internal faces.
// with_g: G is read from wg (else each cell's gradient is recomputed from w).
__global__ void __launch_bounds__(128) boundary_kernel(DevMesh m, Physics ph, PatchTable pt,
                                                       const int* __restrict__ bnd_cs, const double* __restrict__ wg,
                                                       const double* __restrict__ eps_p, bool with_g,
                                                       const double* __restrict__ sig, double* __restrict__ bres,
                                                       ErrWords* __restrict__ err) {
    release_early();
    const int nbf = m.nf - m.nint;
    const int fb = blockIdx.x * blockDim.x + threadIdx.x;
    wait_predecessor();  // w (and G when it is read)
    if (fb >= nbf) return;
    if (eps_p && *eps_p == 0.0) return;
    const int cs = bnd_cs[fb];
    const int c = cs >> 3, s = cs & 7;
    const int f = m.nint + fb;
    const int patch = -m.tslot[tiled(c, 2 * m.spad) + 32 * (m.spad + s)] - 2;
    const int pk = pt.kind[patch];
    double bv[3];
    bc_of(pt, patch, f, m.nint, bv);
    const d3 bc = {bv[0], bv[1], bv[2]};
    const double* fr = face_rec(m, f);
    const d3 gam = ld3(fr);
    // rhie_chow()'s per-face constants |Delta| / |d| and |Gamma|, precomputed on the host with
    // the reference's operations (see flux_pair_kernel)
    const double cfac = fr[32 * 6], gmag = fr[32 * 7];
    auto rc = [&](d3 up, d3 uo, const dm3& gf, d3 delta) {
        const d3 compact = scl(sub(uo, up), cfac);
        return scl(sub(compact, dot_left(delta, gf)), ph.alpha * ph.kbar * gmag);
    };
    d3 flux, st{0.0, 0.0, 0.0};
    if (pk == SFV_PATCH_TRACTION) {  // nominal load |Gamma| T (discretisation.cpp:151-154)
        flux = scl(bc, gmag);
    } else {
        const double* rcell = wg_rec(wg, c);
        const dm3 gc = with_g ? ldG(rcell) : cell_gradient_at(m, pt, wg, c);
        const d3 uc = ld3(rcell);
        const d3 del = ld3(fr + 32 * 3);
        // the cell stress of the gradient pass (J2 needs its committed state), else the law
        bool okc;
        const dm3 sc = with_g && sig ? ld_sig(sig + tiled(c, kSig)) : stress(ph, gc, okc);
        if (pk == SFV_PATCH_DISPLACEMENT) {
            d3 gm = gam;
            if (ph.tl) {
                bool ok;
                gm = transform_area(gam, defgrad(gc), ok);
                if (!ok) atomicMin(&err->inverted_face, f);
            }
            flux = dot_left(gm, sc);
            st = rc(uc, bc, gc, del);
        } else {  // symmetry plane (discretisation.cpp:138-150, :194-203)
            const dm3 R = reflection(gam);
            d3 gm = gam;
            if (ph.tl) {
                bool ok;
                gm = transform_area(gam, mirror_avg(defgrad(gc), R), ok);
                if (!ok) atomicMin(&err->inverted_face, f);
            }
            flux = dot_left(gm, mirror_avg(sc, R));
            st = rc(uc, mv(R, uc), mirror_avg(gc, R), del);
        }
    }
    bres[fb] = flux.x;
    bres[nbf + fb] = flux.y;
    bres[2 * static_cast<size_t>(nbf) + fb] = flux.z;
    bres[3 * static_cast<size_t>(nbf) + fb] = st.x;
    bres[4 * static_cast<size_t>(nbf) + fb] = st.y;
    bres[5 * static_cast<size_t>(nbf) + fb] = st.z;
    release_late();
}

// ---------------------------------------------------------------- fluxes + epilogue
// Face records (m.tf9): Gamma xyz, Delta xyz, |Delta| / |d|, |Gamma|, w (the two ratios are
// the per-face constants of rhie_chow(), precomputed with the same IEEE operations).
// kind of a slot's contribution: 0 none (padding), 1 flux only (traction), 2 flux + stabilisation
// INLB (Hooke, small strain, no symmetry patch): boundary faces are evaluated here, from the
// cell's own gradient, instead of by boundary_kernel.
template <bool PERT, int S, bool GEN, bool INLB>
__global__ void __launch_bounds__(kCells* S, GEN ? SFV_GEN_CTAS * 6 / S : SFV_HOOKE_CTAS * 6 / S)
    flux_pair_kernel(DevMesh m, Physics ph, PatchTable pt, History hist, const double* __restrict__ wg,
                     const double* __restrict__ eps_p, const double* __restrict__ sig,
                     const double* __restrict__ bres, const double* __restrict__ r_u, double* __restrict__ out,
                     ErrWords* __restrict__ err, int tile0, int tile1) {
    // double-buffered per-slot results: one barrier per tile; the sums of tile i (warps
    // s < 3) overlap the face work of tile i + 1, and the barrier of tile i + 1 orders
    // them before buffer i & 1 is rewritten by tile i + 2
    __shared__ double res_buf[2][S][6][kCells];
    // slot kinds lane-major, 8 bytes per cell: the summing thread reads them in one 64-bit load
    __shared__ __align__(8) unsigned char kind_buf[2][kCells][8];
    // Hooke: the tile's own [w | G] records — one contiguous 3072-byte block of the tiled table —
    // are copied to shared memory one tile ahead (cp.async.cg, 16 bytes per thread, past L1), so
    // the six slot warps read them from there instead of gathering them six times through L1
    constexpr bool OWN = !GEN && SFV_OWN_ASYNC;
    __shared__ __align__(16) double own_buf[OWN ? 2 : 1][OWN ? kWG : 1][kCells];
    const int lane = threadIdx.x % kCells, s = threadIdx.x / kCells;
    const int ntiles = tile1;  // this launch covers tiles [tile0, tile1) (the host-buffer J.v runs chunks)
    auto stage_own = [&](int t, int b) {
        if (!OWN || t >= ntiles) return;
        const char* src = reinterpret_cast<const char*>(wg + static_cast<size_t>(t) * (kWG * kCells));
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&own_buf[b][0][0]));
        for (int x = threadIdx.x; x < kWG * kCells / 2; x += kCells * S)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * x), "l"(src + 16 * x) : "memory");
    };
    // Persistent grid-stride loop over tiles of kCells cells (= the tiles of the tables).
    // The slot indices of a tile and the epilogue operand r_u of (component s, cell) —
    // threads s < 3 do the per-cell sums — are loaded one iteration ahead, so a tile's
    // dependent chain is one gather.
    auto fetch = [&](int t, int& fr, int& o, double& ru) {
        const int cc = t * kCells + lane;
        fr = -1;
        o = -1;
        ru = 0.0;
        if (t < ntiles) {  // padding cells of the last tile hold fr = o = -1
            const int* ts = m.tslot + static_cast<size_t>(t) * (2 * S * kCells) + lane;
            fr = __ldcs(ts + kCells * s);
            o = __ldcs(ts + kCells * (S + s));
            if (PERT && s < 3 && cc < m.nc) ru = __ldcs(&r_u[3 * cc + s]);
        }
    };
    int fr_next, o_next;
    double ru_next;
    fetch(tile0 + blockIdx.x, fr_next, o_next, ru_next);
    wait_predecessor();  // bres (and through it G, w, eps)
    if (OWN) {
        stage_own(tile0 + blockIdx.x, 0);
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
    }
    const double eps = PERT ? *eps_p : 0.0;
    const bool zero = PERT && eps == 0.0;  // |v| = 0 short-circuit (nonlinear.cpp:110)
    int it = 0;
    for (int tile = tile0 + blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        double(*res)[6][kCells] = res_buf[it & 1];
        unsigned char(*kind)[8] = kind_buf[it & 1];
        const double(*own)[kCells] = own_buf[OWN ? it & 1 : 0];
        (void)own;
        const int fr = fr_next, o = o_next;
        const double ru = ru_next;
        fetch(tile + gridDim.x, fr_next, o_next, ru_next);
        // buffer (it + 1) & 1 was last read in iteration it - 1, before that iteration's barrier
        stage_own(tile + gridDim.x, (it + 1) & 1);
        const int c = tile * kCells + lane;
        unsigned char kd = 0;
        if (fr != -1 && !zero) {
            const int f = fr & ~kSign;
            d3 flux, st;
            if (o >= 0) {
                const bool nb = (fr & kSign) != 0;
                const int ip = nb ? o : c, in = nb ? c : o;  // reference owner / neighbour
                const double* rf = face_rec(m, f);
                const double* rp = wg_rec(wg, ip);
                const double* rn = wg_rec(wg, in);
                const d3 gam = ld3(rf), del = ld3(rf + 96);
                const double cfac = rf[192], gmag = rf[224], wf = rf[256];
                if (OWN) {
                    // the other cell's record gathered, this cell's from the staged tile
                    const double* rx = wg_rec(wg, o);
                    const d3 ux = ld3(rx);
                    double gx[9], gp[9], gn[9];
                    ldg9(rx, gx);
                    const d3 uo = {own[0][lane], own[1][lane], own[2][lane]};
                    const d3 up = nb ? ux : uo, un = nb ? uo : ux;
#pragma unroll
                    for (int q = 0; q < 9; ++q) {
                        const double go = own[3 + q][lane];
                        gp[q] = nb ? gx[q] : go;
                        gn[q] = nb ? go : gx[q];
                    }
                    hooke_face(gp, gn, wf, ph.mu, ph.lam, gam, del, up, un, cfac, gmag, ph.alpha, ph.kbar, flux, st);
                } else if (!GEN) {
                    const d3 up = ld3(rp), un = ld3(rn);
                    double gp[9], gn[9];
                    ldg9(rp, gp);
                    ldg9(rn, gn);
                    hooke_face(gp, gn, wf, ph.mu, ph.lam, gam, del, up, un, cfac, gmag, ph.alpha, ph.kbar, flux, st);
                } else {
                    const d3 up = ld3(rp), un = ld3(rn);
                    const dm3 gp = ldG(rp), gn = ldG(rn);
                    const dm3 sp = ld_sig(sig + tiled(ip, kSig)), sn = ld_sig(sig + tiled(in, kSig));
                    d3 gm = gam;
                    if (ph.tl) {
                        bool ok;
                        gm = transform_area(gam, interp(defgrad(gp), defgrad(gn), wf), ok);
                        if (!ok) atomicMin(&err->inverted_face, f);
                    }
                    flux = dot_left(gm, interp(sp, sn, wf));
                    // rhie_chow() with its per-face constants precomputed
                    const d3 compact = scl(sub(un, up), cfac);
                    st = scl(sub(compact, dot_left(del, interp(gp, gn, wf))), ph.alpha * ph.kbar * gmag);
                }
                if (nb) {
                    flux = neg(flux);
                    st = neg(st);
                }
                kd = 2;
            } else if (INLB) {
                // boundary face (boundary_kernel's operations): traction |Gamma| T
                // (discretisation.cpp:151-154, no stabilisation term, :204-205), displacement
                // Gamma . sigma_P and the Rhie-Chow term towards the prescribed value (:136-140, :189-193)
                const int patch = -o - 2;
                double bv[3];
                bc_of(pt, patch, f, m.nint, bv);
                const d3 bc = {bv[0], bv[1], bv[2]};
                const double* rf = face_rec(m, f);
                const double gmag = rf[224];
                if (pt.kind[patch] == SFV_PATCH_TRACTION) {
                    flux = scl(bc, gmag);
                    st = {0.0, 0.0, 0.0};
                    kd = 1;
                } else {
                    const double* rc = wg_rec(wg, c);
                    dm3 gc;
                    d3 uc;
                    if (OWN) {
#pragma unroll
                        for (int q = 0; q < 9; ++q) gc.a[q / 3][q % 3] = own[3 + q][lane];
                        uc = {own[0][lane], own[1][lane], own[2][lane]};
                    } else {
                        gc = ldG(rc);
                        uc = ld3(rc);
                    }
                    flux = dot_left(ld3(rf), hooke(gc, ph.mu, ph.lam));
                    const d3 compact = scl(sub(bc, uc), rf[192]);
                    st = scl(sub(compact, dot_left(ld3(rf + 96), gc)), ph.alpha * ph.kbar * gmag);
                    kd = 2;
                }
            } else {
                // boundary face: evaluated by boundary_kernel; traction faces carry no
                // stabilisation term (discretisation.cpp:204-205)
                const int fb = f - m.nint;
                const int nbf = m.nf - m.nint;
                flux = {bres[fb], bres[nbf + fb], bres[2 * nbf + fb]};
                st = {bres[3 * nbf + fb], bres[4 * nbf + fb], bres[5 * nbf + fb]};
                kd = pt.kind[-o - 2] == SFV_PATCH_TRACTION ? 1 : 2;
            }
            res[s][0][lane] = flux.x;
            res[s][1][lane] = flux.y;
            res[s][2][lane] = flux.z;
            res[s][3][lane] = st.x;
            res[s][4][lane] = st.y;
            res[s][5][lane] = st.z;
        }
        kind[lane][s] = kd;
        if (OWN) asm volatile("cp.async.wait_all;" ::: "memory");  // the next tile's records (issued a tile ago)
        __syncthreads();
        // (component k = s, cell c): the reference's per-cell summation order
        if (s < 3 && c < m.nc) {
            const int k = s;
            const int ik = 3 * c + k;
            if (zero) {
                out[ik] = 0.0;
            } else {
                double r = 0.0;
                const unsigned long long kw = *reinterpret_cast<const unsigned long long*>(kind[lane]);
                if (!ph.stab_only) {
#pragma unroll
                    for (int t = 0; t < S; ++t)
                        if ((kw >> (8 * t)) & 0xff) r += res[t][k][lane];
                }
#pragma unroll
                for (int t = 0; t < S; ++t)
                    if (((kw >> (8 * t)) & 0xff) == 2) r += res[t][3 + k][lane];
                if (hist.body && !ph.stab_only) r = r + hist.body[ik];  // body force (discretisation.cpp:160-161)
                if (ph.transient && !ph.stab_only) {  // BDF2 inertia (discretisation.cpp:48-57, :163-169)
                    const double uc = wg[tiled(c, kWG) + 32 * k];
                    const double idt = 1.0 / (2.0 * ph.dt);
                    const double vn = ((uc * 3.0 - hist.u_old[ik] * 4.0) + hist.u_old_old[ik]) * idt;
                    const double ac = ((vn * 3.0 - hist.v_old[ik] * 4.0) + hist.v_old_old[ik]) * idt;
                    r = r - ac * (ph.rho * m.volume[c]);
                }
                if (!ph.stab_only && !isfinite(r)) atomicMin(&err->nan_cell, c);
                if constexpr (PERT) {  // (R(u + eps v) - R(u)) / eps (nonlinear.cpp:132-136)
                    const double q = (r - ru) / eps;
                    if (!isfinite(q)) atomicMin(&err->nan_jv, c);
                    out[ik] = q;
                } else {
                    out[ik] = r;
                }
            }
        }
    }
}

// G (tiled rows 3-11 of wg) -> SoA [q * nc + c] (sfv_gradients)
__global__ void untile_grad_kernel(int nc, const double* __restrict__ wg, double* __restrict__ G) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
#pragma unroll
    for (int q = 0; q < 9; ++q) G[static_cast<size_t>(q) * nc + c] = wg[tiled(c, kWG) + 32 * (3 + q)];
}

template <bool PERT, int S, bool GEN, bool INLB>
int flux_grid(int ntiles) {
    static int per_sm = -1;
    static int sms = 0;
    if (per_sm < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, flux_pair_kernel<PERT, S, GEN, INLB>, kCells * S, 0);
        per_sm = per_sm < 1 ? 1 : per_sm;
    }
    const int g = per_sm * sms;
    return ntiles < g ? ntiles : g;
}

// Every pass is launched as a programmatic dependent of the previous one (PDL): its CTAs
// are scheduled while the predecessor drains, load what does not depend on it (slot
// tables, least-squares vectors, r_u), and block in griddepcontrol.wait — which returns
// once the predecessor grid has completed and its writes are visible — before the first
// read of the predecessor's output.  Optionally the [w | G] L2 persisting window.

template <typename... KArgs, typename... Args>
void launch_win(void (*kern)(KArgs...), int grid, int block, cudaStream_t st, const PairScratch& ps, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
    if (ps.win_bytes) {
        attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[na].val.accessPolicyWindow.base_ptr = ps.win_base;
        attr[na].val.accessPolicyWindow.num_bytes = ps.win_bytes;
        attr[na].val.accessPolicyWindow.hitRatio = ps.win_hit;
        attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// The fused ε + perturb pass: a cooperative launch (co-residency guaranteed, or the launch is
// refused) chained to its predecessor by PDL.  Returns false — with the launch error cleared —
// when the runtime refuses it; the caller then runs the two-launch path.
template <typename... KArgs, typename... Args>
bool launch_eps_perturb(void (*kern)(KArgs...), int grid, cudaStream_t st, Args... args) {
    static int mode = [] {
        const char* e = std::getenv("SFV_EPS_COOP");  // 0: never fused, 1: cooperative without PDL
        return e ? std::atoi(e) : 2;
    }();
    while (mode > 0) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kEpT);
        cfg.stream = st;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = mode == 2 ? 2 : 1;
        if (cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...) == cudaSuccess) return true;
        cudaGetLastError();
        --mode;  // PDL + cooperative refused: cooperative alone; then never
    }
    return false;
}

template <int S>
void launch_grad(const DevMesh& m, const Physics& ph, const PatchTable& pt, const PairScratch& ps, ErrWords* err,
                 cudaStream_t st) {
    const int cb = (m.nc + 255) / 256;
    const bool gen = ph.law != SFV_LAW_HOOKE || ph.tl;
    if (ph.law == SFV_LAW_J2)
        launch_win(grad_cell_kernel<S, true, true>, cb, 256, st, ps, m, pt, ph, ps.wg, ps.sig, ps.lawst, err);
    else if (gen)
        launch_win(grad_cell_kernel<S, true, false, true>, cb, 256, st, ps, m, pt, ph, ps.wg, ps.sig, ps.lawst, err);
    else
        launch_win(grad_cell_kernel<S, false, false, true>, cb, 256, st, ps, m, pt, ph, ps.wg, ps.sig, ps.lawst, err);
}

template <bool PERT, int S>
void launch_s(const DevMesh& m, const Physics& ph, const PatchTable& pt, const History& hist, const double* u,
              const double* v, const double* eps, const double* r_u, double* out, const PairScratch& ps,
              ErrWords* err, cudaStream_t st) {
    double* wg = ps.wg;
    const int cb = (m.nc + 255) / 256;
    const int epg = PERT && ps.partials && ps.bar ? eps_perturb_grid(m.nc) : 0;
    bool fused = false;
    if (epg > 0) {  // ε reduction and w in one launch
        const bool vec = ((reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(v)) & 15) == 0 &&
                         (!ps.vsel_j || ps.vsel_stride % 2 == 0);
        fused = launch_eps_perturb(vec ? eps_perturb_kernel<true> : eps_perturb_kernel<false>, epg, st, m.nc, u, v,
                                   const_cast<double*>(eps), wg, const_cast<double*>(ps.partials), ps.u_norm,
                                   ps.u_norm_cached, ps.vsel_j, static_cast<long long>(ps.vsel_stride));
    }
    if (!fused && ps.vsel_j) {  // only the fused pass reads v through the device index
        if (ps.vsel_failed) *ps.vsel_failed = true;
        return;
    }
    if (!fused) {
        int np = ps.npart;
        if (PERT && ps.partials && ps.bar)  // the fused launch was refused: the two-launch path
            np = launch_norm_partials(u, v, 3 * m.nc, const_cast<double*>(ps.partials), ps.u_norm_cached, st);
        // with the ε reduction folded in, a grid of a few waves keeps the per-block partial sums cheap
        const int pgrid = ps.partials ? std::min(cb, 148 * 8) : cb;
        launch_win(perturb_kernel<PERT>, pgrid, 256, st, ps, m.nc, u, v, const_cast<double*>(eps), wg, ps.partials,
                   np, ps.u_norm, ps.u_norm_cached);
    }
    if (ps.marks) cudaEventRecord(ps.marks[0], st);
    const int nbf = m.nf - m.nint;
    if (nbf > 0 && ps.side) cudaEventRecord(ps.ev_w, st);  // w ready: the boundary pass may start
    const bool gen = ph.law != SFV_LAW_HOOKE || ph.tl;
    launch_grad<S>(m, ph, pt, ps, err, st);
    if (ps.marks) cudaEventRecord(ps.marks[1], st);
    const double* no_eps = nullptr;
    const bool inlb = !gen && !ps.sym && !ps.side;  // boundary faces inside the flux pass
    if (nbf > 0 && !inlb) {
        if (ps.side) {  // beside the gradient pass: the boundary pass computes its own cells' gradients
            cudaStreamWaitEvent(ps.side, ps.ev_w, 0);
            boundary_kernel<<<(nbf + 127) / 128, 128, 0, ps.side>>>(m, ph, pt, ps.bnd_cs, wg, PERT ? eps : no_eps,
                                                                   false, no_eps, ps.bres, err);
            cudaEventRecord(ps.ev_b, ps.side);
            cudaStreamWaitEvent(st, ps.ev_b, 0);
        } else {
            launch_win(boundary_kernel, (nbf + 127) / 128, 128, st, ps, m, ph, pt, ps.bnd_cs, wg, PERT ? eps : no_eps,
                       true, static_cast<const double*>(ps.sig), ps.bres, err);
        }
    }
    if (ps.marks) cudaEventRecord(ps.marks[2], st);
    const int ntiles = (m.nc + kCells - 1) / kCells;
    if (ps.ru_ready) cudaStreamWaitEvent(st, ps.ru_ready, 0);
    const double* cwg = wg;
    const double* sg = ps.sig;
    const double* br = ps.bres;
    // one launch, or (host-buffer J.v) one per chunk of tiles, each after its share of r_u has
    // arrived and followed by an event for the copy of its share of the result
    const int nk = ps.nchunk > 1 ? ps.nchunk : 1;
    for (int k = 0; k < nk; ++k) {
        const int t0 = static_cast<int>(static_cast<long long>(ntiles) * k / nk);
        const int t1 = static_cast<int>(static_cast<long long>(ntiles) * (k + 1) / nk);
        if (nk > 1 && ps.ru_chunk) cudaStreamWaitEvent(st, ps.ru_chunk[k], 0);
        if (gen)
            launch_win(flux_pair_kernel<PERT, S, true, false>, flux_grid<PERT, S, true, false>(t1 - t0), kCells * S,
                       st, ps, m, ph, pt, hist, cwg, eps, sg, br, r_u, out, err, t0, t1);
        else if (inlb)
            launch_win(flux_pair_kernel<PERT, S, false, true>, flux_grid<PERT, S, false, true>(t1 - t0), kCells * S,
                       st, ps, m, ph, pt, hist, cwg, eps, sg, br, r_u, out, err, t0, t1);
        else
            launch_win(flux_pair_kernel<PERT, S, false, false>, flux_grid<PERT, S, false, false>(t1 - t0), kCells * S,
                       st, ps, m, ph, pt, hist, cwg, eps, sg, br, r_u, out, err, t0, t1);
        if (nk > 1 && ps.out_chunk) cudaEventRecord(ps.out_chunk[k], st);
    }
}

}  // namespace

void launch_residual_pair(const DevMesh& m, const Physics& ph, const PatchTable& pt, const History& hist,
                          const double* u, const double* v, const double* jv_eps, const double* r_u, double* out,
                          const PairScratch& ps, ErrWords* err, cudaStream_t s) {
    const bool pert = jv_eps != nullptr;
    if (m.spad == 4) {
        if (pert) launch_s<true, 4>(m, ph, pt, hist, u, v, jv_eps, r_u, out, ps, err, s);
        else launch_s<false, 4>(m, ph, pt, hist, u, v, jv_eps, r_u, out, ps, err, s);
    } else if (m.spad == 6) {
        if (pert) launch_s<true, 6>(m, ph, pt, hist, u, v, jv_eps, r_u, out, ps, err, s);
        else launch_s<false, 6>(m, ph, pt, hist, u, v, jv_eps, r_u, out, ps, err, s);
    } else {
        if (pert) launch_s<true, 8>(m, ph, pt, hist, u, v, jv_eps, r_u, out, ps, err, s);
        else launch_s<false, 8>(m, ph, pt, hist, u, v, jv_eps, r_u, out, ps, err, s);
    }
}

int eps_perturb_grid_for(int nc) { return eps_perturb_grid(nc); }

void launch_gradients_pair(const DevMesh& m, const PatchTable& pt, const Physics& ph, const double* u, double* G,
                           const PairScratch& ps, ErrWords* err, cudaStream_t s) {
    Physics hp = ph;  // gradients only: no stress evaluation (except a J2 commit pass)
    if (!ph.commit) {
        hp.law = SFV_LAW_HOOKE;
        hp.tl = 0;
    }
    const int cb = (m.nc + 255) / 256;
    launch_win(perturb_kernel<false>, cb, 256, s, ps, m.nc, u, u, static_cast<double*>(nullptr), ps.wg,
               static_cast<const double*>(nullptr), 0, static_cast<double*>(nullptr), false);
    if (m.spad == 4) launch_grad<4>(m, hp, pt, ps, err, s);
    else if (m.spad == 6) launch_grad<6>(m, hp, pt, ps, err, s);
    else launch_grad<8>(m, hp, pt, ps, err, s);
    if (G) untile_grad_kernel<<<cb, 256, 0, s>>>(m.nc, ps.wg, G);
}

}  // namespace sfv
