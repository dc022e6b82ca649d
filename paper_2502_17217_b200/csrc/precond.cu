// precond.cu — the reference's preconditioner actions on the GPU (FP64, sm_100a).
//
// ILU(k) apply (IlukPrecond::solve, /root/reference/proj/src/linalg.cpp:302-316).  The
// reference factors the 3n x 3n scalar expansion of the c*I-block approximate Jacobian;
// with c*I blocks that factor is, entry for entry, the n x n cell-graph ILU(k) applied to
// each displacement component (SURVEY.md finding 4), so the device solves the cell graph
// with three interleaved right-hand sides.  Each row keeps the reference's arithmetic
// order (ascending columns forward, descending columns backward, then the pivot divide),
// compiled without FMA, so the apply is bit-identical to the reference's.
//
// Scheduling is sync-free: rows are visited in dependency-level order (levels padded to
// whole warps, so a warp never waits on itself) by a persistent grid whose CTAs are all
// resident; a row polls its dependencies' values through L2 against an sNaN sentinel and
// publishes its own with plain stores.  No grid-wide barrier and no flag array; the
// critical path is the dependency-level count.
//
// Dense apply: exact A^{-1} for the small-system "lu" path (make_preconditioner picks LU
// at <= 30000 rows, nonlinear.cpp:355-356), a warp per row over 3 interleaved RHS.
#include <cooperative_groups.h>

#include <algorithm>

#include <cusolverDn.h>

#include <string>

#include "device.h"

namespace cg = cooperative_groups;

// Timing probes (scripts/probes): build with -DSFV_PROBE_MASK=m to drop parts of the DSMEM
// sweep (1: dependency loads, 2: pivot divide, 4: HBM copies).  Results are then wrong;
// production builds use 0.
#ifndef SFV_PROBE_MASK
#define SFV_PROBE_MASK 0
#endif
#define SFV_PROBE(b) (!(SFV_PROBE_MASK & (b)))
#ifndef SFV_DS_MODE
#define SFV_DS_MODE 0
#endif

namespace sfv {
namespace {

// Sentinel protocol: before a sweep the output vector is filled with an sNaN bit
// pattern no FP operation can produce (arithmetic only ever yields quiet NaNs).  A row
// polls the three values of each dependency directly — one L2 round trip per
// dependency level, no flag array and no fence — and publishes by plain 8-byte stores
// (each single-copy atomic).  A computed value that happens to equal the sentinel is
// canonicalised to the quiet NaN so it can never be mistaken for "not ready".
constexpr unsigned long long kSentinel = 0x7ff4dead0000beefULL;

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double publish(double x) {
    return __double_as_longlong(x) == static_cast<long long>(kSentinel) ? __longlong_as_double(0x7ff8000000000000LL)
                                                                         : x;
}

__global__ void fill_sentinel_kernel(double* z, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        z[i] = __longlong_as_double(static_cast<long long>(kSentinel));
}

// One triangular sweep.  Positions are in dependency-level order, each level padded to
// whole warps, so a warp never waits on one of its own lanes; the grid is persistent
// (all CTAs resident), so every awaited row is owned by a running thread.
// NRHS = 3: one factor shared by the three interleaved components (c*I blocks);
// NRHS = 1: per-component factors (axis-aligned symmetry planes), component = blockIdx.y.
// RS = 1 (with NRHS = 1): one scalar factor over all 3n unknowns — the expanded matrix of a
// symmetry plane that is not axis-aligned, whose blocks couple the components.
template <bool UPPER, int NRHS, int RS = 3>
__global__ void __launch_bounds__(256) tri_kernel(TriSet set, const double* __restrict__ src, double* dst,
                                                  int sleep_ns) {
    const int comp = NRHS == 3 ? 0 : static_cast<int>(blockIdx.y);
    const DevTri& t = set.t[comp];
    const int stride = gridDim.x * blockDim.x;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < t.n; p += stride) {
        const int i = t.order[p];
        if (i < 0) continue;  // level padding
        const int b = t.rp[p], e = t.rp[p + 1];
        double z[NRHS];
#pragma unroll
        for (int k = 0; k < NRHS; ++k) z[k] = src[RS * i + comp + k];
        for (int q = b; q < e; ++q) {
            const int j = t.col[q];
            const double a = t.val[q];
            unsigned long long wv[NRHS];
            for (;;) {
                bool ready = true;
#pragma unroll
                for (int k = 0; k < NRHS; ++k) {
                    wv[k] = ld_relaxed_u64(&dst[RS * j + comp + k]);
                    ready &= wv[k] != kSentinel;
                }
                if (ready) break;
                if (sleep_ns) __nanosleep(sleep_ns);
            }
#pragma unroll
            for (int k = 0; k < NRHS; ++k) z[k] -= a * __longlong_as_double(static_cast<long long>(wv[k]));
        }
        if (UPPER) {
            const double d = t.diag[p];
#pragma unroll
            for (int k = 0; k < NRHS; ++k) z[k] /= d;
        }
#pragma unroll
        for (int k = 0; k < NRHS; ++k) __stcg(&dst[RS * i + comp + k], publish(z[k]));
    }
}

// Level-synchronous sweep in POSITION space, run by one thread-block cluster (or one CTA):
// rows are renumbered in dependency-level order at setup (columns too), the right-hand
// side is gathered into that order once, and the result scattered back once, so every
// load a row needs except its dependency values is contiguous, coalesced and independent
// of the sweep.  The next level's rows are loaded into registers between the arrive and
// the wait of a split-phase barrier.cluster (release/acquire at cluster scope); the only
// loads on the critical path are the dependency values (one L2 round trip per level).
constexpr int kLvlChunk = 1024;

template <bool UPPER, int NRHS, int MAXD, bool SOLO>
__global__ void __launch_bounds__(SOLO ? 1024 : 512) tri_cluster_kernel(TriSet set, const double* __restrict__ src,
                                                                         double* dst) {
    int comp, nthr, tid;
    if (SOLO) {  // one CTA per component
        comp = NRHS == 3 ? 0 : static_cast<int>(blockIdx.x);
        nthr = blockDim.x;
        tid = threadIdx.x;
    } else {
        cg::cluster_group cluster = cg::this_cluster();
        comp = NRHS == 3 ? 0 : static_cast<int>(blockIdx.x / cluster.dim_blocks().x);
        nthr = static_cast<int>(cluster.num_threads());
        tid = static_cast<int>(cluster.block_rank()) * blockDim.x + threadIdx.x;
    }
    const DevTri& t = set.t[comp];
    const int np = t.n;
    // the prefetched row (this thread's first position in the upcoming level)
    int pp = -1;
    int pc[MAXD];
    double pv[MAXD], pz[NRHS], pd = 1.0;
    auto fetch = [&](int p) {
        pp = p;
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
            pc[k] = k < t.maxd ? t.ell_pcol[static_cast<size_t>(k) * np + p] : -1;
            pv[k] = k < t.maxd ? t.ell_val[static_cast<size_t>(k) * np + p] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < NRHS; ++k) pz[k] = src[3 * static_cast<size_t>(p) + comp + k];
        if (UPPER) pd = t.diag[p];
    };
    auto solve = [&]() {
        double z[NRHS];
#pragma unroll
        for (int k = 0; k < NRHS; ++k) z[k] = pz[k];
        double dv[MAXD][NRHS];
#pragma unroll
        for (int q = 0; q < MAXD; ++q)  // all dependency loads in flight together
            if (pc[q] >= 0)
#pragma unroll
                for (int k = 0; k < NRHS; ++k) {
                    const size_t a = 3 * static_cast<size_t>(pc[q]) + comp + k;
                    dv[q][k] = SOLO ? dst[a] : __ldcg(&dst[a]);
                }
#pragma unroll
        for (int q = 0; q < MAXD; ++q)  // then the reference's order of subtraction
            if (pc[q] >= 0)
#pragma unroll
                for (int k = 0; k < NRHS; ++k) z[k] -= pv[q] * dv[q][k];
        if (UPPER)
#pragma unroll
            for (int k = 0; k < NRHS; ++k) z[k] /= pd;
#pragma unroll
        for (int k = 0; k < NRHS; ++k) {
            const size_t a = 3 * static_cast<size_t>(pp) + comp + k;
            if (SOLO) dst[a] = z[k];
            else __stcg(&dst[a], z[k]);
        }
    };
    // level boundaries staged in shared memory (chunks of kLvlChunk levels)
    __shared__ int lp[kLvlChunk + 2];
    auto stage_levels = [&](int base) {
        __syncthreads();
        for (int x = threadIdx.x; x < kLvlChunk + 2; x += blockDim.x)
            lp[x] = base + x <= t.n_levels ? t.level_ptr[base + x] : t.level_ptr[t.n_levels];
        __syncthreads();
    };
    stage_levels(0);
    if (t.n_levels > 0 && lp[0] + tid < lp[1]) fetch(lp[0] + tid);
    for (int l = 0; l < t.n_levels; ++l) {
        const int ll = l % kLvlChunk;
        const int p0 = lp[ll] + tid, pend = lp[ll + 1];
        if (p0 < pend && pp >= 0) solve();
        for (int p = p0 + nthr; p < pend; p += nthr) {  // levels wider than the cluster
            fetch(p);
            solve();
        }
        pp = -1;
        const int q0 = lp[ll + 1] + tid;
        const bool more = l + 1 < t.n_levels && q0 < lp[ll + 2];
        if (SOLO) {
            if (more) fetch(q0);
            __syncthreads();  // one CTA: bar.sync orders its global writes for all its threads
        } else {
            asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
            if (more) fetch(q0);
            asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        }
        if (ll == kLvlChunk - 1) stage_levels(l + 1);
    }
}

// DSMEM sweep: the same position-space level sweep, but the values the next levels read
// live in a ring in the cluster's distributed shared memory.  Positions are dealt to the
// cluster's CTAs in warp-sized chunks (chunk c -> CTA c % CS); each CTA keeps its chunks'
// values in a ring of kRingPerCta 32-byte slots, so a dependency is one or two
// ld.shared::cluster (~200 cycles) instead of an L2 round trip, and the split-phase
// barrier.cluster per level only orders shared-memory writes.  Each thread keeps the
// matrix rows of the next TWO levels in registers (two register sets used alternately,
// refilled right after each arrive), so the HBM latency of the streamed factor is hidden behind two
// barrier periods.  Results go to HBM with plain stores issued after the arrive, so the
// release never waits for them.  The host selects this path only when the ring window
// exceeds the largest dependency distance plus twice the widest level.
constexpr int kDsCluster = 16;
constexpr int kRingPerCta = 4096;  // 32-byte slots per CTA: 128 KB
constexpr int kDsThreads = 256;

template <int MAXD, int NRHS>
struct RowRegs {
    int p;
    int pc[MAXD];
    double pv[MAXD];
    double pz[NRHS];
    double pd;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ double2 ld_dsmem2(uint32_t addr) {
    double2 v;
#if SFV_DS_MODE == 0
    asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
#else
    asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr) : "memory");
#endif
    return v;
}
__device__ __forceinline__ double ld_dsmem(uint32_t addr) {
    double v;
#if SFV_DS_MODE == 0
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr));
#else
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
#endif
    return v;
}

// Level hand-over of the DSMEM sweep.  The values a level publishes live in exactly one
// physical shared memory (the owning CTA's); a CTA-scope fence (MEMBAR.ALL.CTA) makes the
// writing thread's STS complete, and the relaxed cluster barrier orders every later DSMEM
// read after it.  A cluster-scope release would compile to MEMBAR.ALL.GPU, which also
// waits for the level's outstanding HBM stores (~1 us per level); SFV_DS_STRICT=1 builds
// the strict form for comparison.
#ifndef SFV_DS_STRICT
#define SFV_DS_STRICT 0
#endif
__device__ __forceinline__ void ds_arrive() {
#if SFV_DS_STRICT
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
#else
    asm volatile("fence.acq_rel.cta;" ::: "memory");
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
#endif
}
__device__ __forceinline__ void ds_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }

template <bool UPPER, int NRHS, int MAXD>
__global__ void __launch_bounds__(kDsThreads, 1) tri_dsmem_kernel(TriSet set, const double* __restrict__ src,
                                                                  double* dst) {
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) double ring[];  // [kRingPerCta][4]
    const int rank = static_cast<int>(cluster.block_rank());
    const int comp = NRHS == 3 ? 0 : static_cast<int>(blockIdx.x / kDsCluster);
    const DevTri& t = set.t[comp];
    const int np = t.n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int nwarps = kDsThreads / 32;
    const uint32_t ring_base = smem_u32(ring);
    __shared__ int lp[kLvlChunk + 3];
    int lbase = 0;
    auto stage_levels = [&](int base) {
        __syncthreads();
        lbase = base;
        for (int x = threadIdx.x; x < kLvlChunk + 3; x += blockDim.x)
            lp[x] = base + x <= t.n_levels ? t.level_ptr[base + x] : t.level_ptr[t.n_levels];
        __syncthreads();
    };
    // the k-th position of this thread in level l (-1 if none); levels start on chunk boundaries
    auto my_pos = [&](int l, int k) {
        const int ll = l - lbase;
        const int c0 = lp[ll] >> 5;
        const int c = c0 + (rank - c0 % kDsCluster + kDsCluster) % kDsCluster + kDsCluster * (warp + nwarps * k);
        const int p = c * 32 + lane;
        return p < lp[ll + 1] ? p : -1;
    };
    auto slot_addr = [&](int p, int& owner) {
        const int c = p >> 5;
        owner = c % kDsCluster;
        return ring_base + static_cast<uint32_t>(((c / kDsCluster) % (kRingPerCta / 32)) * 32 + (p & 31)) * 32u;
    };
    auto fetch = [&](RowRegs<MAXD, NRHS>& r, int p) {
        r.p = p;
        if (p < 0 || !SFV_PROBE(8)) return;
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
            r.pc[k] = k < t.maxd ? t.ell_pcol[static_cast<size_t>(k) * np + p] : -1;
            r.pv[k] = k < t.maxd ? t.ell_val[static_cast<size_t>(k) * np + p] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < NRHS; ++k) r.pz[k] = src[3 * static_cast<size_t>(p) + comp + k];
        r.pd = UPPER ? t.diag[p] : 1.0;
    };
    auto solve = [&](const RowRegs<MAXD, NRHS>& r, double* z) {
#pragma unroll
        for (int k = 0; k < NRHS; ++k) z[k] = r.pz[k];
        double dv[MAXD][NRHS];
#pragma unroll
        for (int q = 0; q < MAXD; ++q)  // all dependency loads in flight together
            if (r.pc[q] >= 0) {
                int owner;
                const uint32_t a = mapa(slot_addr(r.pc[q], owner), owner);
                if (NRHS == 3) {
                    const double2 v01 = ld_dsmem2(a);
                    dv[q][0] = v01.x;
                    if (NRHS > 1) dv[q][NRHS > 1 ? 1 : 0] = v01.y;
                    if (NRHS > 2) dv[q][NRHS > 2 ? 2 : 0] = ld_dsmem(a + 16);
                } else {
                    dv[q][0] = ld_dsmem(a);
                }
            }
#pragma unroll
        for (int q = 0; q < MAXD; ++q)  // then the reference's order of subtraction
            if (r.pc[q] >= 0)
#pragma unroll
                for (int k = 0; k < NRHS; ++k) z[k] -= r.pv[q] * dv[q][k];
        if (UPPER)
#pragma unroll
            for (int k = 0; k < NRHS; ++k) z[k] /= r.pd;
        int owner;
        double* slot = ring + (slot_addr(r.p, owner) - ring_base) / 8;  // owner == rank by construction
#pragma unroll
        for (int k = 0; k < NRHS; ++k) slot[k] = z[k];
    };
    auto store = [&](int p, const double* z) {
#pragma unroll
        for (int k = 0; k < NRHS; ++k) dst[3 * static_cast<size_t>(p) + comp + k] = z[k];
    };
    RowRegs<MAXD, NRHS> R0, R1;  // level l in R0 (l even) / R1 (l odd); the other holds l+1
    stage_levels(0);
    fetch(R0, t.n_levels > 0 ? my_pos(0, 0) : -1);
    fetch(R1, t.n_levels > 1 ? my_pos(1, 0) : -1);
    // one level: solve `cur`, extra positions of wide levels, barrier, refill `cur` with level l+3
    auto level = [&](RowRegs<MAXD, NRHS>& cur, int l) {
        double z[NRHS];
        int done_p = -1;
        if (cur.p >= 0) {
            solve(cur, z);
            done_p = cur.p;
        }
        for (int k = 1;; ++k) {  // levels wider than the cluster's first round
            const int p = my_pos(l, k);
            if (p < 0) break;
            if (done_p >= 0) store(done_p, z);
            RowRegs<MAXD, NRHS> w;
            fetch(w, p);
            solve(w, z);
            done_p = p;
        }
        ds_arrive();
        if (done_p >= 0) store(done_p, z);  // HBM copy, outside the release
        const bool restage = l + 3 - lbase > kLvlChunk;
        if (!restage) fetch(cur, l + 2 < t.n_levels ? my_pos(l + 2, 0) : -1);
        ds_wait();
        if (restage) {
            stage_levels(l + 1);
            fetch(cur, l + 2 < t.n_levels ? my_pos(l + 2, 0) : -1);
        }
    };
    for (int l = 0; l < t.n_levels; l += 2) {
        level(R0, l);
        if (l + 1 < t.n_levels) level(R1, l + 1);
    }
}

// position-space gathers / scatters around the sweeps (padding positions get zeros)
__global__ void gather_pos_kernel(const int* __restrict__ order, int np, int comp, int ncomp,
                                  const double* __restrict__ in, double* __restrict__ out) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x) {
        const int i = order[p];
        for (int k = comp; k < comp + ncomp; ++k) out[3 * static_cast<size_t>(p) + k] = i >= 0 ? in[3 * static_cast<size_t>(i) + k] : 0.0;
    }
}
__global__ void scatter_pos_kernel(const int* __restrict__ order, int np, int comp, int ncomp,
                                   const double* __restrict__ in, double* __restrict__ out) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x) {
        const int i = order[p];
        if (i >= 0)
            for (int k = comp; k < comp + ncomp; ++k) out[3 * static_cast<size_t>(i) + k] = in[3 * static_cast<size_t>(p) + k];
    }
}
// y_U[p'] = y_L[map[p']] (map: U position -> L position, -1 on padding)
__global__ void permute_pos_kernel(const int* __restrict__ map, int np, int comp, int ncomp,
                                   const double* __restrict__ in, double* __restrict__ out) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x) {
        const int q = map[p];
        for (int k = comp; k < comp + ncomp; ++k) out[3 * static_cast<size_t>(p) + k] = q >= 0 ? in[3 * static_cast<size_t>(q) + k] : 0.0;
    }
}

__global__ void __launch_bounds__(256) dense_apply_kernel(const double* __restrict__ inv, int n,
                                                          const double* __restrict__ r, double* __restrict__ z) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= n) return;
    const double* row = inv + static_cast<size_t>(warp) * n;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    for (int j = lane; j < n; j += 32) {
        const double a = row[j];
        a0 += a * r[3 * j];
        a1 += a * r[3 * j + 1];
        a2 += a * r[3 * j + 2];
    }
    for (int o = 16; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    if (lane == 0) {
        z[3 * warp] = a0;
        z[3 * warp + 1] = a1;
        z[3 * warp + 2] = a2;
    }
}

// Column t of W = A^{-1} for A = L L^T banded (bandwidth bw): thread t solves
// L y = e_t then L^T x = y in place in W[:, t] (row-major W, so warps access
// consecutive addresses).  Setup only (small-system exact preconditioner).
__global__ void __launch_bounds__(128) band_inverse_kernel(const double* __restrict__ l, int n, int bw,
                                                           double* __restrict__ W) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int w = bw + 1;
    auto L = [&](int i, int j) { return l[static_cast<size_t>(i) * w + (j - i + bw)]; };
    auto X = [&](int i) -> double& { return W[static_cast<size_t>(i) * n + t]; };
    for (int i = 0; i < t; ++i) X(i) = 0.0;
    for (int i = t; i < n; ++i) {
        double s = i == t ? 1.0 : 0.0;
        const int k0 = max(t, i - bw);
        for (int k = k0; k < i; ++k) s -= L(i, k) * X(k);
        X(i) = s / L(i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = X(i);
        const int k1 = min(n - 1, i + bw);
        for (int k = i + 1; k <= k1; ++k) s -= L(k, i) * X(k);
        X(i) = s / L(i, i);
    }
}

// z[perm[i]] = -sum_j W[i][j] r[perm[j]] (K = -A): NRHS = 3 applies one W to the three
// interleaved components; NRHS = 1 applies it to component `comp` only; RS = 1: W spans all
// 3n unknowns (coupled components).
template <int NRHS, int RS = 3>
__global__ void __launch_bounds__(256) dense_apply_perm_kernel(const double* __restrict__ W, int n,
                                                               const int* __restrict__ perm,
                                                               const double* __restrict__ r,
                                                               double* __restrict__ z, int comp) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= n) return;
    const double* row = W + static_cast<size_t>(warp) * n;
    double acc[NRHS];
#pragma unroll
    for (int k = 0; k < NRHS; ++k) acc[k] = 0.0;
    for (int j = lane; j < n; j += 32) {
        const double a = row[j];
        const int pj = perm[j];
#pragma unroll
        for (int k = 0; k < NRHS; ++k) acc[k] += a * r[RS * pj + comp + k];
    }
#pragma unroll
    for (int k = 0; k < NRHS; ++k)
        for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
    if (lane == 0) {
        const int pi = perm[warp];
#pragma unroll
        for (int k = 0; k < NRHS; ++k) z[RS * pi + comp + k] = -acc[k];
    }
}

}  // namespace

// Dense Cholesky of the (permuted) band of -A by cuSOLVER: the band is scattered into a dense
// column-major matrix, factored in place (lower), and the band of L read back out — Cholesky
// does not fill outside the band.  Replaces the host band factorisation for the small-system
// exact preconditioner (parity there is "any exact solve").
__global__ void band_to_dense_kernel(const double* __restrict__ l, int n, int bw, double* __restrict__ D) {
    const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int w = bw + 1;
    if (idx >= static_cast<size_t>(n) * w) return;
    const int i = static_cast<int>(idx / w), k = static_cast<int>(idx % w);
    const int j = i - bw + k;
    if (j < 0) return;
    D[static_cast<size_t>(j) * n + i] = l[idx];  // column-major, lower triangle (row i >= column j)
}
__global__ void dense_to_band_kernel(const double* __restrict__ D, int n, int bw, double* __restrict__ l) {
    const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int w = bw + 1;
    if (idx >= static_cast<size_t>(n) * w) return;
    const int i = static_cast<int>(idx / w), k = static_cast<int>(idx % w);
    const int j = i - bw + k;
    l[idx] = j < 0 ? 0.0 : D[static_cast<size_t>(j) * n + i];
}

__global__ void identity_kernel(int n, double* __restrict__ W) {
    const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx < static_cast<size_t>(n) * n) W[idx] = (idx / n == idx % n) ? 1.0 : 0.0;
}
std::string device_band_cholesky(double* band, int n, int bw, cudaStream_t s, double* W) {
    cusolverDnHandle_t h = nullptr;
    if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) return "lu: cusolver unavailable";
    cusolverDnSetStream(h, s);
    double* D = nullptr;
    double* work = nullptr;
    int* info = nullptr;
    std::string err;
    int lwork = 0, hinfo = 0;
    const size_t nn = static_cast<size_t>(n) * n, nb = static_cast<size_t>(n) * (bw + 1);
    if (cudaMalloc(&D, sizeof(double) * nn) != cudaSuccess || cudaMalloc(&info, sizeof(int)) != cudaSuccess) {
        err = "lu: out of device memory";
    } else {
        cudaMemsetAsync(D, 0, sizeof(double) * nn, s);
        band_to_dense_kernel<<<static_cast<unsigned>((nb + 255) / 256), 256, 0, s>>>(band, n, bw, D);
        if (cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, n, D, n, &lwork) != CUSOLVER_STATUS_SUCCESS ||
            cudaMalloc(&work, sizeof(double) * (lwork > 0 ? lwork : 1)) != cudaSuccess) {
            err = "lu: cusolver workspace";
        } else if (cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, n, D, n, work, lwork, info) != CUSOLVER_STATUS_SUCCESS ||
                   cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                   cudaStreamSynchronize(s) != cudaSuccess) {
            err = "lu: factorisation failed";
        } else if (hinfo != 0) {
            err = "lu: factorisation failed";
        } else if (!W) {
            dense_to_band_kernel<<<static_cast<unsigned>((nb + 255) / 256), 256, 0, s>>>(D, n, bw, band);
            if (cudaStreamSynchronize(s) != cudaSuccess) err = "lu: factorisation failed";
        } else {  // the explicit inverse: L L^T X = I by potrs (two TRSMs over n right-hand sides)
            // X is symmetric, so its column-major image is the row-major W the apply reads
            identity_kernel<<<static_cast<unsigned>((nn + 255) / 256), 256, 0, s>>>(n, W);
            if (cusolverDnDpotrs(h, CUBLAS_FILL_MODE_LOWER, n, n, D, n, W, n, info) != CUSOLVER_STATUS_SUCCESS ||
                cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                cudaStreamSynchronize(s) != cudaSuccess || hinfo != 0)
                err = "lu: factorisation failed";
        }
    }
    cudaFree(D);
    cudaFree(work);
    cudaFree(info);
    cusolverDnDestroy(h);
    return err;
}

void launch_band_inverse(const double* l, int n, int bw, double* W, cudaStream_t s) {
    band_inverse_kernel<<<(n + 127) / 128, 128, 0, s>>>(l, n, bw, W);
}

void launch_dense_apply_perm(const double* W, int n, const int* perm, const double* r, double* z, int comp,
                             cudaStream_t s) {
    if (comp == kDenseCoupled)  // W over all 3n unknowns (coupled components)
        dense_apply_perm_kernel<1, 1><<<(n + 7) / 8, 256, 0, s>>>(W, n, perm, r, z, 0);
    else if (comp < 0)
        dense_apply_perm_kernel<3><<<(n + 7) / 8, 256, 0, s>>>(W, n, perm, r, z, 0);
    else
        dense_apply_perm_kernel<1><<<(n + 7) / 8, 256, 0, s>>>(W, n, perm, r, z, comp);
}

template <bool UPPER, int NRHS, int MAXD>
static cudaError_t launch_cluster_w(const TriSet& set, int ncomp, int csize, const double* src, double* dst,
                                    cudaStream_t s) {
    if (csize == 1) {  // single-CTA sweep: bar.sync per level, 1024 threads
        tri_cluster_kernel<UPPER, NRHS, MAXD, true><<<NRHS == 3 ? 1 : ncomp, 1024, 0, s>>>(set, src, dst);
        return cudaGetLastError();
    }
    auto kern = tri_cluster_kernel<UPPER, NRHS, MAXD, false>;
    if (csize > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csize * (NRHS == 3 ? 1 : ncomp));
    cfg.blockDim = dim3(512);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, set, src, dst);
}

template <bool UPPER, int NRHS, int MAXD>
static cudaError_t launch_dsmem_w(const TriSet& set, int ncomp, const double* src, double* dst, cudaStream_t s) {
    auto kern = tri_dsmem_kernel<UPPER, NRHS, MAXD>;
    const int smem = kRingPerCta * 4 * static_cast<int>(sizeof(double));
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kDsCluster * (NRHS == 3 ? 1 : ncomp));
    cfg.blockDim = dim3(kDsThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kDsCluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, set, src, dst);
}

template <bool UPPER, int NRHS>
static cudaError_t launch_cluster(const TriSet& set, int ncomp, int csize, const double* src, double* dst,
                                  cudaStream_t s) {
    int maxd = 0;
    for (int a = 0; a < (NRHS == 3 ? 1 : ncomp); ++a) maxd = std::max(maxd, set.t[a].maxd);
    if (csize == kDsRingMode) {  // values in distributed shared memory
        if (maxd <= 8) return launch_dsmem_w<UPPER, NRHS, 8>(set, ncomp, src, dst, s);
        if (maxd <= 16) return launch_dsmem_w<UPPER, NRHS, 16>(set, ncomp, src, dst, s);
        return launch_dsmem_w<UPPER, NRHS, 32>(set, ncomp, src, dst, s);
    }
    if (maxd <= 8) return launch_cluster_w<UPPER, NRHS, 8>(set, ncomp, csize, src, dst, s);
    if (maxd <= 16) return launch_cluster_w<UPPER, NRHS, 16>(set, ncomp, csize, src, dst, s);
    return launch_cluster_w<UPPER, NRHS, 32>(set, ncomp, csize, src, dst, s);
}

void launch_ilu_apply(const TriSet& L, const TriSet& U, int ncomp, const double* r, double* y, double* z, int grid,
                      int sleep_ns, int cluster, double* pa, double* pb, const StreamSet* SL, const StreamSet* SU,
                      cudaStream_t s, const PipeSet* PL, const PipeSet* PU) {
    if (cluster == kPipeMode) {  // block-pipelined sweeps, one cluster per component
        for (int c = 0; c < 3; ++c)  // r -> lower-sweep positions
            gather_pos_kernel<<<592, 256, 0, s>>>(PL->t[c].order, PL->t[c].n_pos, c, 1, r, pa);
        launch_tri_pipe(*PL, false, pa, pb, s);
        for (int c = 0; c < 3; ++c)  // y: lower-sweep -> upper-sweep positions
            permute_pos_kernel<<<592, 256, 0, s>>>(PU->t[c].to_lower, PU->t[c].n_pos, c, 1, pb, pa);
        launch_tri_pipe(*PU, true, pa, pb, s);
        for (int c = 0; c < 3; ++c)  // upper-sweep positions -> rows
            scatter_pos_kernel<<<592, 256, 0, s>>>(PU->t[c].order, PU->t[c].n_pos, c, 1, pb, z);
        return;
    }
    if (cluster > 0) {  // level-synchronous position-space sweeps (default)
        const int per = ncomp == 1 ? 3 : 1;
        for (int c = 0; c < ncomp; ++c)  // r -> L positions
            gather_pos_kernel<<<592, 256, 0, s>>>(L.t[c].order, L.t[c].n, c, per, r, pa);
        if (cluster == kStreamMode) {  // the forward sweep stores in U positions, the backward one in rows
            launch_tri_stream(*SL, false, ncomp, pa, pb, s);
            launch_tri_stream(*SU, true, ncomp, pb, z, s);
            return;
        }
        if (ncomp == 1) launch_cluster<false, 3>(L, 1, cluster, pa, pb, s);
        else launch_cluster<false, 1>(L, 3, cluster, pa, pb, s);
        for (int c = 0; c < ncomp; ++c)  // y: L positions -> U positions
            permute_pos_kernel<<<592, 256, 0, s>>>(U.t[c].u2l, U.t[c].n, c, per, pb, pa);
        if (ncomp == 1) launch_cluster<true, 3>(U, 1, cluster, pa, pb, s);
        else launch_cluster<true, 1>(U, 3, cluster, pa, pb, s);
        for (int c = 0; c < ncomp; ++c)  // U positions -> rows
            scatter_pos_kernel<<<592, 256, 0, s>>>(U.t[c].order, U.t[c].n, c, per, pb, z);
        return;
    }
    const int n3 = ncomp < 0 ? L.t[0].n_rows : 3 * L.t[0].n_rows;  // sync-free sentinel polling (SFV_TRI_CLUSTER=0)
    fill_sentinel_kernel<<<592, 256, 0, s>>>(y, n3);
    fill_sentinel_kernel<<<592, 256, 0, s>>>(z, n3);
    if (ncomp < 0) {  // coupled components: one factor over the 3n unknowns
        tri_kernel<false, 1, 1><<<grid, 256, 0, s>>>(L, r, y, sleep_ns);
        tri_kernel<true, 1, 1><<<grid, 256, 0, s>>>(U, y, z, sleep_ns);
    } else if (ncomp == 1) {
        tri_kernel<false, 3><<<grid, 256, 0, s>>>(L, r, y, sleep_ns);  // forward, unit lower: y
        tri_kernel<true, 3><<<grid, 256, 0, s>>>(U, y, z, sleep_ns);   // backward with U: z
    } else {
        const dim3 g(std::max(1, grid / 3), 3);
        tri_kernel<false, 1><<<g, 256, 0, s>>>(L, r, y, sleep_ns);
        tri_kernel<true, 1><<<g, 256, 0, s>>>(U, y, z, sleep_ns);
    }
}

void launch_dense_apply(const double* inv, int n, const double* r, double* z, cudaStream_t s) {
    const int warps_per_block = 8;
    dense_apply_kernel<<<(n + warps_per_block - 1) / warps_per_block, 256, 0, s>>>(inv, n, r, z);
}

}  // namespace sfv

namespace sfv {
int ilu_ring_window() { return kRingPerCta * kDsCluster; }
}  // namespace sfv

// ---------------------------------------------------------------- ILU(<=1) numeric phase
// IlukPrecond's IKJ elimination (linalg.cpp:283-299) on the device, one warp per row, rows in
// dependency-level order over a persistent grid (every awaited row is held by a resident
// warp at an earlier position, so the waits terminate).  Row i waits for row k (flag
// published with release semantics after the row is final), l_ik = a_ik / u_kk by lane 0,
// then the lanes take row k's upper entries and update the matching entries of row i
// (binary search in the sorted row) — each entry of row i sees the same subtractions in the
// same k order as the host loop, so the factor is bit-identical (-fmad=false).
#include "host_threads.h"
#include "precond_dev.h"
#include "precond_host.h"

namespace sfv {
namespace {

__global__ void __launch_bounds__(256) ilu_numeric_kernel(int n, const int* __restrict__ rows,
                                                          const int* __restrict__ rp, const int* __restrict__ col,
                                                          const int* __restrict__ diag, double* val, int* done,
                                                          int* broke) {
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int x = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < n; x += nw) {
        const int i = rows[x];
        const int r1 = rp[i + 1];
        for (int p = rp[i]; p < r1; ++p) {
            const int k = col[p];
            if (k >= i) break;
            if (lane == 0) {
                int f;
                do {
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(done + k) : "memory");
                } while (f == 0);
            }
            __syncwarp();
            const double pivot = __ldcg(val + diag[k]);
            if (pivot == 0.0 || !isfinite(pivot)) {
                if (lane == 0) atomicExch(broke, 1);
                break;
            }
            double lik = 0.0;
            if (lane == 0) {
                lik = val[p] / pivot;
                val[p] = lik;
            }
            lik = __shfl_sync(0xffffffffu, lik, 0);
            const int k1 = rp[k + 1];
            for (int q = diag[k] + 1 + lane; q < k1; q += 32) {
                const int j = col[q];
                int lo = p + 1, hi = r1;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (col[mid] < j) lo = mid + 1;
                    else hi = mid;
                }
                if (lo < r1 && col[lo] == j) val[lo] -= lik * __ldcg(val + q);
            }
            __syncwarp();
        }
        __syncwarp();
        if (lane == 0) {
            const double d = val[diag[i]];
            if (d == 0.0 || !isfinite(d)) atomicExch(broke, 1);
            __threadfence();
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(done + i), "r"(1) : "memory");
        }
    }
}

template <typename T>
T* dev_copy(const T* h, size_t n) {
    T* d = nullptr;
    if (cudaMalloc(&d, sizeof(T) * (n ? n : 1)) != cudaSuccess) return nullptr;
    if (n) cudaMemcpy(d, h, sizeof(T) * n, cudaMemcpyHostToDevice);
    return d;
}

}  // namespace

bool launch_ilu_numeric(int n, const int* rows, const int* rp, const int* col, const int* diag, double* val,
                        cudaStream_t stream) {
    int* d_flags = nullptr;  // done[n] + broke
    if (cudaMalloc(&d_flags, sizeof(int) * (n + 1)) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    cudaMemsetAsync(d_flags, 0, sizeof(int) * (n + 1), stream);
    int* d_broke = d_flags + n;
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ilu_numeric_kernel, 256, 0);
    const int grid = std::max(1, std::min(sms * std::max(per, 1), (n + 7) / 8));
    void* args[] = {&n, const_cast<int**>(&rows), const_cast<int**>(&rp), const_cast<int**>(&col),
                    const_cast<int**>(&diag), &val, &d_flags, &d_broke};
    const bool launched = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(ilu_numeric_kernel), dim3(grid),
                                                      dim3(256), args, 0, stream) == cudaSuccess;
    int broke = 1;
    if (launched) cudaMemcpyAsync(&broke, d_broke, sizeof(int), cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    cudaFree(d_flags);
    cudaGetLastError();
    return launched && broke == 0;
}

bool device_ilu_numeric(ScalarCsr& out, const std::vector<int>& diag, const std::vector<int>& rows,
                        cudaStream_t stream) {
    StageClock sc;
    const int n = out.n;
    const size_t nnz = static_cast<size_t>(out.rp[n]);
    int* d_rows = dev_copy(rows.data(), rows.size());
    int* d_rp = dev_copy(out.rp.data(), out.rp.size());
    int* d_col = dev_copy(out.col.data(), nnz);
    int* d_diag = dev_copy(diag.data(), diag.size());
    double* d_val = dev_copy(out.val.data(), nnz);
    int* d_flags = nullptr;  // done[n] + broke
    const bool alloc = d_rows && d_rp && d_col && d_diag && d_val &&
                       cudaMalloc(&d_flags, sizeof(int) * (n + 1)) == cudaSuccess;
    bool ok = false;
    if (alloc) {
        cudaMemset(d_flags, 0, sizeof(int) * (n + 1));
        int* d_broke = d_flags + n;
        cudaDeviceSynchronize();
        sc.mark("ilu device upload");
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ilu_numeric_kernel, 256, 0);
        const int grid = std::max(1, std::min(sms * std::max(per, 1), (n + 7) / 8));
        // warps spin on rows owned by other blocks: the grid must be co-resident, which only a
        // cooperative launch guarantees (a refused launch falls back to the host factor)
        void* args[] = {const_cast<int*>(&n), &d_rows, &d_rp, &d_col, &d_diag, &d_val, &d_flags, &d_broke};
        const bool launched = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(ilu_numeric_kernel), dim3(grid),
                                                          dim3(256), args, 0, stream) == cudaSuccess;
        cudaStreamSynchronize(stream);
        sc.mark("ilu device kernel");
        int broke = 1;
        if (launched && cudaMemcpy(&broke, d_flags + n, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess &&
            cudaMemcpy(out.val.data(), d_val, sizeof(double) * nnz, cudaMemcpyDeviceToHost) == cudaSuccess)
            ok = broke == 0;
        sc.mark("ilu device download");
    }
    cudaFree(d_rows);
    cudaFree(d_rp);
    cudaFree(d_col);
    cudaFree(d_diag);
    cudaFree(d_val);
    cudaFree(d_flags);
    cudaGetLastError();  // a failed allocation falls back to the host factor, no sticky state
    return ok;
}

}  // namespace sfv
