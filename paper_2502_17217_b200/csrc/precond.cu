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

#include "device.h"

namespace cg = cooperative_groups;

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
template <bool UPPER, int NRHS>
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
        for (int k = 0; k < NRHS; ++k) z[k] = src[3 * i + comp + k];
        for (int q = b; q < e; ++q) {
            const int j = t.col[q];
            const double a = t.val[q];
            unsigned long long wv[NRHS];
            for (;;) {
                bool ready = true;
#pragma unroll
                for (int k = 0; k < NRHS; ++k) {
                    wv[k] = ld_relaxed_u64(&dst[3 * j + comp + k]);
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
        for (int k = 0; k < NRHS; ++k) __stcg(&dst[3 * i + comp + k], publish(z[k]));
    }
}

// Level-synchronous sweep run by ONE thread-block cluster (up to 16 CTAs on 16 SMs):
// the rows of a level are spread over the cluster's threads, then one
// barrier.cluster (release/acquire at cluster scope, ~0.2 us) publishes them to the
// next level.  Nothing spins, so no L2 bandwidth is burnt on polling.  Rows are stored
// per level in ELL form and the NEXT level's matrix entries and right-hand side are
// loaded into registers before the barrier, so the only loads left on the critical
// path are the dependency values themselves (one L2 round trip per level).
constexpr int kLvlChunk = 1024;

template <bool UPPER, int NRHS, int MAXD>
__global__ void __launch_bounds__(512) tri_cluster_kernel(TriSet set, const double* __restrict__ src, double* dst) {
    cg::cluster_group cluster = cg::this_cluster();
    const int comp = NRHS == 3 ? 0 : static_cast<int>(blockIdx.x / cluster.dim_blocks().x);
    const DevTri& t = set.t[comp];
    const int nthr = static_cast<int>(cluster.num_threads());
    const int tid = static_cast<int>(cluster.block_rank()) * blockDim.x + threadIdx.x;
    const int np = t.n;
    // prefetched row (first row of this thread in the upcoming level)
    int pi = -1;
    int pc[MAXD];
    double pv[MAXD], pz[NRHS], pd = 1.0;
    auto fetch = [&](int p) {
        pi = t.order[p];
        if (pi < 0) return;
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
            pc[k] = k < t.maxd ? t.ell_col[static_cast<size_t>(k) * np + p] : -1;
            pv[k] = pc[k] >= 0 ? t.ell_val[static_cast<size_t>(k) * np + p] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < NRHS; ++k) pz[k] = src[3 * pi + comp + k];
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
                for (int k = 0; k < NRHS; ++k) dv[q][k] = __ldcg(&dst[3 * pc[q] + comp + k]);
#pragma unroll
        for (int q = 0; q < MAXD; ++q)  // then the reference's order of subtraction
            if (pc[q] >= 0)
#pragma unroll
                for (int k = 0; k < NRHS; ++k) z[k] -= pv[q] * dv[q][k];
        if (UPPER)
#pragma unroll
            for (int k = 0; k < NRHS; ++k) z[k] /= pd;
#pragma unroll
        for (int k = 0; k < NRHS; ++k) __stcg(&dst[3 * pi + comp + k], z[k]);
    };
    // level boundaries staged once in shared memory (chunks of kLvlChunk levels)
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
        if (p0 < pend && pi >= 0) solve();
        for (int p = p0 + nthr; p < pend; p += nthr) {  // levels wider than the cluster
            fetch(p);
            if (pi >= 0) solve();
        }
        pi = -1;
        // split-phase barrier: publish this level (release), prefetch the next level's
        // rows while the other CTAs arrive, then acquire.
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        const int q0 = lp[ll + 1] + tid;
        if (l + 1 < t.n_levels && q0 < lp[ll + 2]) fetch(q0);
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (ll == kLvlChunk - 1) stage_levels(l + 1);
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
// interleaved components; NRHS = 1 applies it to component `comp` only.
template <int NRHS>
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
        for (int k = 0; k < NRHS; ++k) acc[k] += a * r[3 * pj + comp + k];
    }
#pragma unroll
    for (int k = 0; k < NRHS; ++k)
        for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
    if (lane == 0) {
        const int pi = perm[warp];
#pragma unroll
        for (int k = 0; k < NRHS; ++k) z[3 * pi + comp + k] = -acc[k];
    }
}

}  // namespace

void launch_band_inverse(const double* l, int n, int bw, double* W, cudaStream_t s) {
    band_inverse_kernel<<<(n + 127) / 128, 128, 0, s>>>(l, n, bw, W);
}

void launch_dense_apply_perm(const double* W, int n, const int* perm, const double* r, double* z, int comp,
                             cudaStream_t s) {
    if (comp < 0)
        dense_apply_perm_kernel<3><<<(n + 7) / 8, 256, 0, s>>>(W, n, perm, r, z, 0);
    else
        dense_apply_perm_kernel<1><<<(n + 7) / 8, 256, 0, s>>>(W, n, perm, r, z, comp);
}

template <bool UPPER, int NRHS, int MAXD>
static cudaError_t launch_cluster_w(const TriSet& set, int ncomp, int csize, const double* src, double* dst,
                                    cudaStream_t s) {
    auto kern = tri_cluster_kernel<UPPER, NRHS, MAXD>;
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

template <bool UPPER, int NRHS>
static cudaError_t launch_cluster(const TriSet& set, int ncomp, int csize, const double* src, double* dst,
                                  cudaStream_t s) {
    int maxd = 0;
    for (int a = 0; a < (NRHS == 3 ? 1 : ncomp); ++a) maxd = std::max(maxd, set.t[a].maxd);
    if (maxd <= 8) return launch_cluster_w<UPPER, NRHS, 8>(set, ncomp, csize, src, dst, s);
    if (maxd <= 16) return launch_cluster_w<UPPER, NRHS, 16>(set, ncomp, csize, src, dst, s);
    return launch_cluster_w<UPPER, NRHS, 32>(set, ncomp, csize, src, dst, s);
}

void launch_ilu_apply(const TriSet& L, const TriSet& U, int ncomp, const double* r, double* y, double* z, int grid,
                      int sleep_ns, int cluster, cudaStream_t s) {
    if (cluster > 0) {  // level-synchronous cluster sweep (default)
        if (ncomp == 1) {
            launch_cluster<false, 3>(L, 1, cluster, r, y, s);
            launch_cluster<true, 3>(U, 1, cluster, y, z, s);
        } else {
            launch_cluster<false, 1>(L, 3, cluster, r, y, s);
            launch_cluster<true, 1>(U, 3, cluster, y, z, s);
        }
        return;
    }
    const int n3 = 3 * L.t[0].n_rows;  // sync-free sentinel polling (SFV_TRI_CLUSTER=0)
    fill_sentinel_kernel<<<592, 256, 0, s>>>(y, n3);
    fill_sentinel_kernel<<<592, 256, 0, s>>>(z, n3);
    if (ncomp == 1) {
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
