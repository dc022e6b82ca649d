// precond_stream.cu — the streamed ILU(k) triangular sweep (default on the device path).
//
// Same arithmetic as IlukPrecond::solve (/root/reference/proj/src/linalg.cpp:302-316) on the
// cell graph with three interleaved right-hand sides (SURVEY.md finding 4), in position
// space (rows renumbered in dependency-level order, see precond.cu).  One thread-block
// cluster of 16 CTAs walks the levels; per level:
//
//   * CTA r owns a contiguous chunk-aligned slice of the level's positions and computes
//     them; their values go into CTA r's shared-memory ring, from where later levels read
//     them over DSMEM (one ld.shared::cluster pair per dependency, ~200 cycles);
//   * each position's factor row is a 96-byte record (16-bit DSMEM address of every
//     dependency, its value, the pivot), streamed kStages-1 levels ahead with cp.async into
//     shared-memory stages — the dependent chain per level is only DSMEM loads + FMA-free
//     FP64 arithmetic, never an HBM round trip;
//   * one CTA-scope fence + relaxed cluster barrier hands the level over (a cluster-scope
//     release compiles to MEMBAR.ALL.GPU and would wait for the HBM stores of the results).
//
// The host builds the records and checks that no ring slot is rewritten before its last
// reader and that no level slice exceeds kMaxRows (build_stream_records); otherwise the
// other sweeps in precond.cu are used.  Compiled with -fmad=false: bit-identical results.
#include <cooperative_groups.h>

#include "device.h"

namespace cg = cooperative_groups;

namespace sfv {
namespace {

constexpr int kThreads = 256;
constexpr int kLvl = 1024;

struct Rec {
    unsigned short dep[8];
    unsigned short own;
    unsigned short pad[3];
    double val[8];
    double diag;
};
static_assert(sizeof(Rec) == 96, "record layout");

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t addr, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

template <bool UPPER, int NRHS, int kStages>
__global__ void __launch_bounds__(kThreads, 1) tri_stream_kernel(StreamSet set, const double* __restrict__ src,
                                                                 double* __restrict__ dst) {
    const int kMaxRows = set.max_rows;  // rows per CTA per level (stage stride)
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = static_cast<int>(cluster.block_rank());
    const int comp = NRHS == 3 ? 0 : static_cast<int>(blockIdx.x / kStreamCluster);
    const DevStream& t = set.t[comp];
    extern __shared__ __align__(16) unsigned char smem[];
    double* ring = reinterpret_cast<double*>(smem);                               // [ring][4]
    Rec* stage_rec = reinterpret_cast<Rec*>(smem + static_cast<size_t>(set.ring) * 32);  // [kStages][kMaxRows]
    double* stage_src = reinterpret_cast<double*>(stage_rec + kStages * kMaxRows);  // [kStages][kMaxRows*3]
    int* lp = reinterpret_cast<int*>(stage_src + kStages * kMaxRows * 3);          // [kLvl + 2]
    const uint32_t ring_base = smem_u32(ring);
    int lbase = 0;
    auto stage_levels = [&](int base) {
        __syncthreads();
        lbase = base;
        for (int x = threadIdx.x; x < kLvl + 2; x += kThreads)
            lp[x] = base + x <= t.n_levels ? t.level_ptr[base + x] : t.level_ptr[t.n_levels];
        __syncthreads();
    };
    auto slice = [&](int l, int& a, int& b) {  // this CTA's positions of level l
        const int la = lp[l - lbase], lb = lp[l - lbase + 1];
        const int nch = (lb - la) >> 5, per = (nch + kStreamCluster - 1) / kStreamCluster;
        a = min(lb, la + rank * per * 32);
        b = min(lb, a + per * 32);
    };
    auto issue = [&](int l) {  // async copy of level l's records and right-hand side
        if (l < t.n_levels) {
            int a, b;
            slice(l, a, b);
            const int s = l % kStages;
            const uint32_t rdst = smem_u32(stage_rec + s * kMaxRows);
            const unsigned char* rsrc = reinterpret_cast<const unsigned char*>(t.rec) + static_cast<size_t>(a) * 96;
            for (int u = threadIdx.x; u < (b - a) * 6; u += kThreads) cp16(rdst + u * 16, rsrc + u * 16);
            const uint32_t sdst = smem_u32(stage_src + s * kMaxRows * 3);
            const double* ssrc = src + 3 * static_cast<size_t>(a);
            for (int u = threadIdx.x; u < ((b - a) * 3) / 2; u += kThreads) cp16(sdst + u * 16, ssrc + 2 * u);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    stage_levels(0);
    for (int l = 0; l < kStages - 1; ++l) issue(l);
    for (int l = 0; l < t.n_levels; ++l) {
        if (l + kStages - 1 + 1 - lbase > kLvl) stage_levels(l);  // keep lp[] covering the issue window
        issue(l + kStages - 1);
        asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 1) : "memory");
        __syncthreads();
        int a, b;
        slice(l, a, b);
        const int s = l % kStages;
        for (int j = threadIdx.x; j < b - a; j += kThreads) {
            const Rec& r = stage_rec[s * kMaxRows + j];
            double z[NRHS];
#pragma unroll
            for (int k = 0; k < NRHS; ++k) z[k] = stage_src[(s * kMaxRows + j) * 3 + comp + k];
            double dv[8][NRHS];
#pragma unroll
            for (int q = 0; q < 8; ++q) {  // all dependency loads in flight together
                const unsigned d = r.dep[q];
                if (d != 0xffffu) {
                    const uint32_t ad = mapa(ring_base + (d & 0xfffu) * 32u, static_cast<int>(d >> 12));
                    if (NRHS == 3) {
                        asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];"
                                     : "=d"(dv[q][0]), "=d"(dv[q][NRHS > 1 ? 1 : 0])
                                     : "r"(ad));
                        asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(dv[q][NRHS > 2 ? 2 : 0]) : "r"(ad + 16));
                    } else {
                        asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(dv[q][0]) : "r"(ad));
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 8; ++q)  // the reference's order of subtraction
                if (r.dep[q] != 0xffffu)
#pragma unroll
                    for (int k = 0; k < NRHS; ++k) z[k] -= r.val[q] * dv[q][k];
            if (UPPER)
#pragma unroll
                for (int k = 0; k < NRHS; ++k) z[k] /= r.diag;
            double* slot = ring + static_cast<size_t>(r.own) * 4;
#pragma unroll
            for (int k = 0; k < NRHS; ++k) {
                slot[k] = z[k];
                dst[3 * static_cast<size_t>(a + j) + comp + k] = z[k];
            }
        }
        // hand the level over: CTA-scope fence (the values live in this CTA's shared memory)
        asm volatile("fence.acq_rel.cta;" ::: "memory");
        asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

template <bool UPPER, int NRHS, int ST>
cudaError_t launch_st(const StreamSet& set, int ncomp, const double* src, double* dst, cudaStream_t s) {
    auto kern = tri_stream_kernel<UPPER, NRHS, ST>;
    const int smem = stream_smem_bytes(set.ring, set.max_rows, ST);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kStreamCluster * (NRHS == 3 ? 1 : ncomp));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kStreamCluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, set, src, dst);
}

template <bool UPPER, int NRHS>
cudaError_t launch_one(const StreamSet& set, int ncomp, const double* src, double* dst, cudaStream_t s) {
    switch (set.stages) {
        case 3: return launch_st<UPPER, NRHS, 3>(set, ncomp, src, dst, s);
        case 4: return launch_st<UPPER, NRHS, 4>(set, ncomp, src, dst, s);
        case 5: return launch_st<UPPER, NRHS, 5>(set, ncomp, src, dst, s);
        case 6: return launch_st<UPPER, NRHS, 6>(set, ncomp, src, dst, s);
        case 7: return launch_st<UPPER, NRHS, 7>(set, ncomp, src, dst, s);
        default: return launch_st<UPPER, NRHS, 8>(set, ncomp, src, dst, s);
    }
}

}  // namespace

int stream_smem_bytes(int ring, int max_rows, int stages) {
    return ring * 32 + stages * max_rows * (96 + 24) + (kLvl + 2) * 4;
}

cudaError_t launch_tri_stream(const StreamSet& set, bool upper, int ncomp, const double* src, double* dst,
                              cudaStream_t s) {
    if (upper) return ncomp == 1 ? launch_one<true, 3>(set, 1, src, dst, s) : launch_one<true, 1>(set, 3, src, dst, s);
    return ncomp == 1 ? launch_one<false, 3>(set, 1, src, dst, s) : launch_one<false, 1>(set, 3, src, dst, s);
}

}  // namespace sfv
