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

#include "device.h"
#include "face_math.cuh"
#include "sfv_case.h"

namespace sfv {
namespace {

using namespace fm;

constexpr int kCells = 32;  // cells per CTA (one warp-width); CTA = kCells x S threads
constexpr int kSign = static_cast<int>(0x80000000u);

__device__ __forceinline__ d3 ldsoa(const double* __restrict__ p, int n, int i) {
    return {p[i], p[n + i], p[2 * static_cast<size_t>(n) + i]};
}
// Streams read once per pass (slot tables, least-squares vectors, r_u) are loaded with
// evict-first (ld.global.cs) so that the gathered w and G (~96 MB at 1M cells) stay in L2.
// All gathered arrays are SoA so that the 32 lanes of a warp (32 consecutive cells, one
// face slot) load 32 consecutive doubles per instruction: the L1 wavefront queue, not DRAM,
// limits a gather kernel whose loads each touch many 128-byte lines.
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
// perturbed state w[k * nc + c] = u + eps v
__device__ __forceinline__ d3 ldw(const double* __restrict__ w, int nc, int c) {
    return {w[c], w[nc + c], w[2 * nc + c]};
}
// cell gradient G[q * nc + c], q = 3 i + j (row-major)
__device__ __forceinline__ void ldg9(const double* __restrict__ G, int nc, int c, double* g) {
#pragma unroll
    for (int q = 0; q < 9; ++q) g[q] = G[q * nc + c];
}
__device__ __forceinline__ dm3 ldG(const double* __restrict__ G, int nc, int c) {
    dm3 r;
#pragma unroll
    for (int q = 0; q < 9; ++q) r.a[q / 3][q % 3] = G[q * nc + c];
    return r;
}

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

// symmetric cell stress from its 6 stored entries (grad_cell_kernel<S, true>)
__device__ __forceinline__ dm3 ld_sig(const double* __restrict__ sig, int nc, int c) {
    dm3 r;
    r.a[0][0] = sig[c];
    r.a[0][1] = r.a[1][0] = sig[nc + c];
    r.a[0][2] = r.a[2][0] = sig[2 * nc + c];
    r.a[1][1] = sig[3 * nc + c];
    r.a[1][2] = r.a[2][1] = sig[4 * nc + c];
    r.a[2][2] = sig[5 * nc + c];
    return r;
}

// ---------------------------------------------------------------- perturbed state
// w = u + eps v, formed once per J.v exactly as the reference forms u_pert
// (nonlinear.cpp:116-118); plain residual: w = u.
// ε from the block partials of ‖u‖², ‖v‖² (launch_norm_partials): every block sums them in
// the same fixed order, so all blocks hold the same bits; block 0 publishes ε (and ‖u‖).
// Replaces a last-block finalisation (atomics and a serial tail) on the J·v critical path.
__device__ __forceinline__ double eps_from_partials(const double* __restrict__ part, int np, double* __restrict__ u_norm,
                                                    bool cached, double* sh) {
    double tu = 0.0, tv = 0.0;
    for (int b = threadIdx.x; b < np; b += blockDim.x) {
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
                                                      double* __restrict__ eps_p, double* __restrict__ w,
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
        st_keep(&w[c], x, pol);
        st_keep(&w[nc + c], y, pol);
        st_keep(&w[2 * nc + c], z, pol);
    }
    release_late();
}

// ---------------------------------------------------------------- gradients
// one thread per cell, slots unrolled so the neighbour loads are all in flight together
// (discretisation.cpp:10-31: g += ls_f (x) (u_N - u_P), faces in cell order)
// GEN (non-Hooke law or total Lagrangian): the cell's stress sigma(G_c) is evaluated here
// once (laws.cpp; the stress loop of discretisation.cpp:116-119, which also reports an
// inverted cell) and stored as its 6 independent entries, instead of twice per face in
// the flux pass — same function on the same G, so the same bits (sigma is symmetric
// bitwise: every entry pair is a product sum of the same factors).
template <int S, bool GEN>
__global__ void __launch_bounds__(256) grad_cell_kernel(DevMesh m, PatchTable pt, Physics ph,
                                                        const double* __restrict__ w, double* __restrict__ G,
                                                        double* __restrict__ sig, ErrWords* __restrict__ err) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= m.nc) return;
    release_early();
    int o[S];
#pragma unroll
    for (int s = 0; s < S; ++s) o[s] = s < m.slots ? __ldcs(&m.slot_other[s * m.nc + c]) : -1;
    wait_predecessor();  // w
    const d3 wc = ldw(w, m.nc, c);
    d3 wn[S];
#pragma unroll
    for (int s = 0; s < S; ++s) wn[s] = o[s] >= 0 ? ldw(w, m.nc, o[s]) : d3{0.0, 0.0, 0.0};
    double g[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) g[q] = 0.0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        d3 du;
        if (o[s] >= 0) {
            du = sub(wn[s], wc);
        } else if (o[s] <= -2 && pt.kind[-o[s] - 2] == SFV_PATCH_SYMMETRY) {
            const dm3 R = reflection(ldsoa(m.gam, m.nf, m.slot_face[s * m.nc + c] & ~kSign));
            du = sub(mv(R, wc), wc);
        } else {
            continue;  // traction / displacement faces are not in the stencil; padding
        }
        const d3 ls = {__ldcs(&m.slot_ls[(3 * s) * m.nc + c]), __ldcs(&m.slot_ls[(3 * s + 1) * m.nc + c]),
                       __ldcs(&m.slot_ls[(3 * s + 2) * m.nc + c])};
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) g[3 * i + j] += cmp(ls, i) * cmp(du, j);
    }
    const unsigned long long pol = evict_last_policy();
#pragma unroll
    for (int q = 0; q < 9; ++q) st_keep(&G[q * m.nc + c], g[q], pol);
    if (GEN) {
        dm3 gm;
#pragma unroll
        for (int q = 0; q < 9; ++q) gm.a[q / 3][q % 3] = g[q];
        bool ok;
        const dm3 sc = stress(ph, gm, ok);
        if (!ok) atomicMin(&err->inverted_cell, c);
        st_keep(&sig[c], sc.a[0][0], pol);
        st_keep(&sig[m.nc + c], sc.a[0][1], pol);
        st_keep(&sig[2 * m.nc + c], sc.a[0][2], pol);
        st_keep(&sig[3 * m.nc + c], sc.a[1][1], pol);
        st_keep(&sig[4 * m.nc + c], sc.a[1][2], pol);
        st_keep(&sig[5 * m.nc + c], sc.a[2][2], pol);
    }
    release_late();
}

// One cell's gradient with exactly grad_cell_kernel's operations (slots in face order), for
// the boundary pass, which then needs w only and can run beside the gradient pass.
__device__ __forceinline__ dm3 cell_gradient_at(const DevMesh& m, const PatchTable& pt, const double* __restrict__ w,
                                                int c) {
    const d3 wc = ldw(w, m.nc, c);
    double g[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) g[q] = 0.0;
    for (int s = 0; s < m.slots; ++s) {
        const int o = m.slot_other[s * m.nc + c];
        d3 du;
        if (o >= 0) {
            du = sub(ldw(w, m.nc, o), wc);
        } else if (o <= -2 && pt.kind[-o - 2] == SFV_PATCH_SYMMETRY) {
            const dm3 R = reflection(ldsoa(m.gam, m.nf, m.slot_face[s * m.nc + c] & ~kSign));
            du = sub(mv(R, wc), wc);
        } else {
            continue;
        }
        const d3 ls = {m.slot_ls[(3 * s) * m.nc + c], m.slot_ls[(3 * s + 1) * m.nc + c],
                       m.slot_ls[(3 * s + 2) * m.nc + c]};
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
// One thread per boundary face (face f = nint + fb, slot index bnd_si[fb] = s * nc + cell):
// flux and stabilisation term into bres[q * nbf + fb] (discretisation.cpp:128-154, :186-205).
// Kept out of the per-slot kernel so its register budget is set by the internal faces.
__global__ void __launch_bounds__(128) boundary_kernel(DevMesh m, Physics ph, PatchTable pt,
                                                       const int* __restrict__ bnd_si, const double* __restrict__ face9,
                                                       const double* __restrict__ w,
                                                       const double* __restrict__ eps_p,
                                                       const double* __restrict__ G, double* __restrict__ bres,
                                                       ErrWords* __restrict__ err) {
    release_early();
    const int nbf = m.nf - m.nint;
    const int fb = blockIdx.x * blockDim.x + threadIdx.x;
    wait_predecessor();  // w (and G when it is read)
    if (fb >= nbf) return;
    if (eps_p && *eps_p == 0.0) return;
    const int si = bnd_si[fb];
    const int c = si % m.nc;
    const int f = m.nint + fb;
    const int patch = -m.slot_other[si] - 2;
    const int pk = pt.kind[patch];
    const d3 bc = {pt.value[patch][0], pt.value[patch][1], pt.value[patch][2]};
    const d3 gam = ldsoa(face9, m.nf, f);
    // rhie_chow()'s per-face constants |Delta| / |d| and |Gamma|, precomputed on the host with
    // the reference's operations (see flux_pair_kernel)
    const double cfac = face9[6 * static_cast<size_t>(m.nf) + f], gmag = face9[7 * static_cast<size_t>(m.nf) + f];
    auto rc = [&](d3 up, d3 uo, const dm3& gf, d3 delta) {
        const d3 compact = scl(sub(uo, up), cfac);
        return scl(sub(compact, dot_left(delta, gf)), ph.alpha * ph.kbar * gmag);
    };
    d3 flux, st{0.0, 0.0, 0.0};
    if (pk == SFV_PATCH_TRACTION) {  // nominal load |Gamma| T (discretisation.cpp:151-154)
        flux = scl(bc, gmag);
    } else {
        const dm3 gc = G ? ldG(G, m.nc, c) : cell_gradient_at(m, pt, w, c);
        const d3 uc = ldw(w, m.nc, c);
        const d3 del = ldsoa(face9 + 3 * static_cast<size_t>(m.nf), m.nf, f);
        bool okc;
        const dm3 sc = stress(ph, gc, okc);
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
// face9[q * nf + f], q = Gamma xyz, Delta xyz, |Delta| / |d|, |Gamma|, w (the two ratios are
// the per-face constants of rhie_chow(), precomputed with the same IEEE operations).
// kind of a slot's contribution: 0 none (padding), 1 flux only (traction), 2 flux + stabilisation
template <bool PERT, int S, bool GEN>
__global__ void __launch_bounds__(kCells* S, GEN ? 12 / S : 24 / S)
    flux_pair_kernel(DevMesh m, Physics ph, PatchTable pt, History hist, const double* __restrict__ w,
                     const double* __restrict__ eps_p, const double* __restrict__ G, const double* __restrict__ sig,
                     const double* __restrict__ face9, const double* __restrict__ bres,
                     const double* __restrict__ r_u, double* __restrict__ out, ErrWords* __restrict__ err) {
    // double-buffered per-slot results: one barrier per tile; the sums of tile i (warps
    // s < 3) overlap the face work of tile i + 1, and the barrier of tile i + 1 orders
    // them before buffer i & 1 is rewritten by tile i + 2
    __shared__ double res_buf[2][S][6][kCells];
    __shared__ unsigned char kind_buf[2][S][kCells];
    const int lane = threadIdx.x % kCells, s = threadIdx.x / kCells;
    const int ntiles = (m.nc + kCells - 1) / kCells;
    // Persistent grid-stride loop over tiles of kCells cells.  The slot indices of a tile
    // and the epilogue operand r_u of (component s, cell) — threads s < 3 do the per-cell
    // sums — are loaded one iteration ahead, so a tile's dependent chain is one gather.
    auto fetch = [&](int t, int& fr, int& o, double& ru) {
        const int cc = t * kCells + lane;
        fr = -1;
        o = -1;
        ru = 0.0;
        if (t < ntiles && cc < m.nc) {
            if (s < m.slots) {
                fr = __ldcs(&m.slot_face[s * m.nc + cc]);
                o = __ldcs(&m.slot_other[s * m.nc + cc]);
            }
            if (PERT && s < 3) ru = __ldcs(&r_u[3 * cc + s]);
        }
    };
    int fr_next, o_next;
    double ru_next;
    fetch(blockIdx.x, fr_next, o_next, ru_next);
    wait_predecessor();  // bres (and through it G, w, eps)
    const double eps = PERT ? *eps_p : 0.0;
    const bool zero = PERT && eps == 0.0;  // |v| = 0 short-circuit (nonlinear.cpp:110)
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        double(*res)[6][kCells] = res_buf[it & 1];
        unsigned char(*kind)[kCells] = kind_buf[it & 1];
        const int fr = fr_next, o = o_next;
        const double ru = ru_next;
        fetch(tile + gridDim.x, fr_next, o_next, ru_next);
        const int c = tile * kCells + lane;
        unsigned char kd = 0;
        if (fr != -1 && !zero) {
            const int f = fr & ~kSign;
            d3 flux, st;
            if (o >= 0) {
                const bool nb = (fr & kSign) != 0;
                const int ip = nb ? o : c, in = nb ? c : o;  // reference owner / neighbour
                const int nf = m.nf;
                const d3 gam = {face9[f], face9[nf + f], face9[2 * nf + f]};
                const d3 del = {face9[3 * nf + f], face9[4 * nf + f], face9[5 * nf + f]};
                const double cfac = face9[6 * nf + f], gmag = face9[7 * nf + f], wf = face9[8 * nf + f];
                const d3 up = ldw(w, m.nc, ip), un = ldw(w, m.nc, in);
                if (!GEN) {
                    double gp[9], gn[9];
                    ldg9(G, m.nc, ip, gp);
                    ldg9(G, m.nc, in, gn);
                    hooke_face(gp, gn, wf, ph.mu, ph.lam, gam, del, up, un, cfac, gmag, ph.alpha, ph.kbar, flux, st);
                } else {
                    const dm3 gp = ldG(G, m.nc, ip), gn = ldG(G, m.nc, in);
                    const dm3 sp = ld_sig(sig, m.nc, ip), sn = ld_sig(sig, m.nc, in);
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
        kind[s][lane] = kd;
        __syncthreads();
        // (component k = s, cell c): the reference's per-cell summation order
        if (s < 3 && c < m.nc) {
            const int k = s;
            const int ik = 3 * c + k;
            if (zero) {
                out[ik] = 0.0;
            } else {
                double r = 0.0;
                if (!ph.stab_only) {
#pragma unroll
                    for (int t = 0; t < S; ++t)
                        if (kind[t][lane] != 0) r += res[t][k][lane];
                }
#pragma unroll
                for (int t = 0; t < S; ++t)
                    if (kind[t][lane] == 2) r += res[t][3 + k][lane];
                if (ph.transient && !ph.stab_only) {  // BDF2 inertia (discretisation.cpp:48-57, :163-169)
                    const double uc = w[k * m.nc + c];
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

template <bool PERT, int S, bool GEN>
int flux_grid(int ntiles) {
    static int per_sm = -1;
    static int sms = 0;
    if (per_sm < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, flux_pair_kernel<PERT, S, GEN>, kCells * S, 0);
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

template <bool PERT, int S>
void launch_s(const DevMesh& m, const Physics& ph, const PatchTable& pt, const History& hist, const double* u,
              const double* v, const double* eps, const double* r_u, double* out, const PairScratch& ps,
              ErrWords* err, cudaStream_t st) {
    double* w = ps.w;
    double* G = ps.G;
    const int cb = (m.nc + 255) / 256;
    // with the ε reduction folded in, a grid of a few waves keeps the per-block partial sums cheap
    const int pgrid = ps.partials ? std::min(cb, 148 * 8) : cb;
    launch_win(perturb_kernel<PERT>, pgrid, 256, st, ps, m.nc, u, v, const_cast<double*>(eps), w, ps.partials,
               ps.npart, ps.u_norm, ps.u_norm_cached);
    if (ps.marks) cudaEventRecord(ps.marks[0], st);
    const int nbf = m.nf - m.nint;
    if (nbf > 0 && ps.side) cudaEventRecord(ps.ev_w, st);  // w ready: the boundary pass may start
    const bool gen = ph.law != SFV_LAW_HOOKE || ph.tl;
    if (gen) launch_win(grad_cell_kernel<S, true>, cb, 256, st, ps, m, pt, ph, w, G, ps.sig, err);
    else launch_win(grad_cell_kernel<S, false>, cb, 256, st, ps, m, pt, ph, w, G, ps.sig, err);
    if (ps.marks) cudaEventRecord(ps.marks[1], st);
    if (nbf > 0) {
        if (ps.side) {  // beside the gradient pass: the boundary pass computes its own cells' gradients
            cudaStreamWaitEvent(ps.side, ps.ev_w, 0);
            boundary_kernel<<<(nbf + 127) / 128, 128, 0, ps.side>>>(
                m, ph, pt, ps.bnd_si, ps.face9, w, PERT ? eps : static_cast<const double*>(nullptr), nullptr, ps.bres, err);
            cudaEventRecord(ps.ev_b, ps.side);
            cudaStreamWaitEvent(st, ps.ev_b, 0);
        } else {
            launch_win(boundary_kernel, (nbf + 127) / 128, 128, st, ps, m, ph, pt, ps.bnd_si, ps.face9, w,
                       PERT ? eps : static_cast<const double*>(nullptr), G, ps.bres, err);
        }
    }
    if (ps.marks) cudaEventRecord(ps.marks[2], st);
    const int ntiles = (m.nc + kCells - 1) / kCells;
    const double* f9 = ps.face9;
    if (gen)
        launch_win(flux_pair_kernel<PERT, S, true>, flux_grid<PERT, S, true>(ntiles), kCells * S, st, ps, m, ph, pt,
                   hist, w, eps, G, static_cast<const double*>(ps.sig), f9, ps.bres, r_u, out, err);
    else
        launch_win(flux_pair_kernel<PERT, S, false>, flux_grid<PERT, S, false>(ntiles), kCells * S, st, ps, m, ph,
                   pt, hist, w, eps, G, static_cast<const double*>(ps.sig), f9, ps.bres, r_u, out, err);
}

}  // namespace

void launch_residual_pair(const DevMesh& m, const Physics& ph, const PatchTable& pt, const History& hist,
                          const double* u, const double* v, const double* jv_eps, const double* r_u, double* out,
                          const PairScratch& ps, ErrWords* err, cudaStream_t s) {
    const bool pert = jv_eps != nullptr;
    if (m.slots <= 4) {
        if (pert) launch_s<true, 4>(m, ph, pt, hist, u, v, jv_eps, r_u, out, ps, err, s);
        else launch_s<false, 4>(m, ph, pt, hist, u, v, jv_eps, r_u, out, ps, err, s);
    } else if (m.slots <= 6) {
        if (pert) launch_s<true, 6>(m, ph, pt, hist, u, v, jv_eps, r_u, out, ps, err, s);
        else launch_s<false, 6>(m, ph, pt, hist, u, v, jv_eps, r_u, out, ps, err, s);
    } else {
        if (pert) launch_s<true, 8>(m, ph, pt, hist, u, v, jv_eps, r_u, out, ps, err, s);
        else launch_s<false, 8>(m, ph, pt, hist, u, v, jv_eps, r_u, out, ps, err, s);
    }
}

}  // namespace sfv
