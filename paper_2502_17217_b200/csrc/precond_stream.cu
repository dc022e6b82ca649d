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
//   * each position's factor row is a 112-byte record (32-bit DSMEM window offset of every
//     dependency, its value, the pivot), stored field-major per chunk of 32 positions
//     (device.h kStream*: bank-conflict-free shared-memory reads) and streamed kStages-1
//     levels ahead with cp.async into shared-memory stages — the dependent chain per level
//     is only DSMEM loads + FMA-free FP64 arithmetic, never an HBM round trip;
//   * the value ring is one array per right-hand side ([NRHS][ring] doubles), so the 32
//     lanes of a warp store consecutive doubles;
//   * one CTA-scope fence + relaxed cluster barrier hands the level over (a cluster-scope
//     release compiles to MEMBAR.ALL.GPU and would wait for the HBM stores of the results).
//
// The host builds the records and checks that no ring slot is rewritten before its last
// reader and that no level slice exceeds kMaxRows (build_stream_records); otherwise the
// other sweeps in precond.cu are used.  Compiled with -fmad=false: bit-identical results.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

#include "device.h"

namespace cg = cooperative_groups;

// timing probes (scripts/build_variant.py): -DSFV_TS_PROBE=m drops 1: the CTA fence,
// 2: the result stores to HBM, 4: the record prefetch, 8: the dependency loads,
// 16: the whole row loop, 64: every dependency read from the reading CTA (results are then
// wrong); 32: per-phase clock64 totals of
// CTA 0 / CTA 15 printed at exit (results stay right).
#ifndef SFV_TS_PROBE
#define SFV_TS_PROBE 0
#endif
#define TSP(b) (!(SFV_TS_PROBE & (b)))
// hand-over experiments (soak only): 1: cluster-scope fence before the arrive, 2: a
// fence.proxy.async after the rows, 4: the slice recomputed instead of read from the stage header
#ifndef SFV_STREAM_FIX
#define SFV_STREAM_FIX 0
#endif
#ifndef SFV_DIV_CORR
#define SFV_DIV_CORR 1  // 0: plain division in the U sweep
#endif

namespace sfv {
namespace {

#ifndef SFV_STREAM_THREADS
#define SFV_STREAM_THREADS 256
#endif
constexpr int kThreads = SFV_STREAM_THREADS;
constexpr int kLvl = 1024;

// field offsets inside a 3072-byte chunk of 32 records (precond_host.h: pack_stream_chunks)
constexpr int kChunk = kStreamChunk, kRec = kStreamRec, kOffDiag = kStreamOffDiag, kOffDep = kStreamOffDep,
              kOffOwn = kStreamOffOwn, kOffOutIdx = kStreamOffOut;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint32_t a, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
// one TMA bulk copy global -> own shared memory, completing `bytes` on the mbarrier
__device__ __forceinline__ void bulk_copy(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(a),
        "r"(parity)
        : "memory");
}

// kThreads compute threads + one producer warp whose lane 0 streams the records kStages - 1
// levels ahead: a CTA's slice of a level is contiguous in position space, so it is two TMA
// bulk copies (records, right-hand side) completing on the stage's mbarrier (expect_tx).
// The per-level critical path is: wait stage -> rows -> cluster barrier.
template <bool UPPER, int NRHS, int kStages>
__global__ void __launch_bounds__(kThreads + 32, 1) tri_stream_kernel(StreamSet set, const double* __restrict__ src,
                                                                      double* __restrict__ dst
#if defined(SFV_STREAM_DELAY) && SFV_STREAM_DELAY >= 4
                                                                      ,
                                                                      double* tlb_probe  // cold pages, 2 MB apart
#endif
) {
    const int kMaxRows = set.max_rows;  // rows per CTA per level (stage stride)
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = static_cast<int>(cluster.block_rank());
    const int comp = NRHS == 3 ? 0 : static_cast<int>(blockIdx.x / kStreamCluster);
    // constant indices: the parameter is read from the constant bank, not copied to local memory
    const DevStream t = comp == 0 ? set.t[0] : comp == 1 ? set.t[1] : set.t[2];
    const bool producer = threadIdx.x >= kThreads;
    const int ptid = threadIdx.x - kThreads;
    extern __shared__ __align__(16) unsigned char smem[];
    const int ring_n = set.ring;
    // [NRHS][ring_n + 1]: slot ring_n of each array holds +0.0 — the records point an absent
    // dependency there (its factor value is 0), so the dependency loads need no predicate
    const int ring_s = ring_n + 1;
    double* ring = reinterpret_cast<double*>(smem);
    unsigned char* stage_rec = smem + stream_ring_bytes(ring_n);  // [kStages][kMaxRows / 32 chunks]
    double* stage_src = reinterpret_cast<double*>(stage_rec + static_cast<size_t>(kStages) * kMaxRows * kRec);  // [kStages][kMaxRows*3]
    int* lp = reinterpret_cast<int*>(stage_src + kStages * kMaxRows * 3);  // [kLvl + 2]
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(lp + kLvl + 2);  // [kStages], 8-aligned
    double* zero_slot = reinterpret_cast<double*>(mbar + kStages);  // 0.0: read by absent dependencies
    // per stage: (first position, count) of this CTA's slice, written by the producer before
    // the stage's mbarrier arrive, so a compute thread does not redo the slice arithmetic
    int2* stage_hdr = reinterpret_cast<int2*>(zero_slot + 2);  // [kStages]
    const uint32_t zero_addr = smem_u32(zero_slot);
    const uint32_t ring_base = smem_u32(ring);
    const uint32_t ring_lo = ring_base & 0xffffffu;
    const uint32_t mbar_base = smem_u32(mbar);
    int lbase = 0;
    auto stage_levels = [&](int base) {
        __syncthreads();
        lbase = base;
        for (int x = threadIdx.x; x < kLvl + 2; x += blockDim.x)
            lp[x] = base + x <= t.n_levels ? t.level_ptr[base + x] : t.level_ptr[t.n_levels];
        __syncthreads();
    };
    auto slice = [&](int l, int& a, int& b) {  // this CTA's positions of level l
        const int la = lp[l - lbase], lb = lp[l - lbase + 1];
        const int nch = (lb - la) >> 5, per = (nch + kStreamCluster - 1) / kStreamCluster;
        a = min(lb, la + rank * per * 32);
        b = min(lb, a + per * 32);
    };
    auto issue = [&](int l) {  // producer lane 0: level l's records and right-hand side
        if (l >= t.n_levels || ptid != 0) return;
        const int s = l % kStages;
        int a, b;
        slice(l, a, b);
        if (!TSP(4)) b = a;
        const uint32_t bar = mbar_base + 8u * s;
        // positions are chunk (32) aligned: both copies are 16-byte multiples at 16-byte addresses
        stage_hdr[s] = make_int2(a, b - a);
        mbar_expect(bar, static_cast<uint32_t>(b - a) * (kRec + 24u));
        if (b > a) {
            bulk_copy(smem_u32(stage_rec + static_cast<size_t>(s) * kMaxRows * kRec),
                      reinterpret_cast<const unsigned char*>(t.rec) + static_cast<size_t>(a) * kRec,
                      static_cast<uint32_t>(b - a) * kRec, bar);
            bulk_copy(smem_u32(stage_src + s * kMaxRows * 3), src + 3 * static_cast<size_t>(a),
                      static_cast<uint32_t>(b - a) * 24u, bar);
        }
    };
    if (threadIdx.x < kStages) mbar_init(mbar_base + 8u * threadIdx.x, 1);
    if (threadIdx.x == 0) *zero_slot = 0.0;
    if (threadIdx.x < NRHS) ring[threadIdx.x * ring_s + ring_n] = 0.0;
    stage_levels(0);  // its __syncthreads also publishes the mbarrier init
    if (producer)
        for (int l = 0; l < kStages - 1; ++l) issue(l);
    long long ph[5] = {0, 0, 0, 0, 0}, t0 = 0, t1 = 0;
    (void)ph;
    (void)t0;
    (void)t1;
    for (int l = 0; l < t.n_levels; ++l) {
        if (!TSP(32)) t0 = clock64();
        if (l + kStages - 1 + 1 - lbase > kLvl) stage_levels(l);  // keep lp[] covering the issue window
        if (producer) {
            // stage (l - 1) % kStages was consumed before the barrier that ended level l - 1
#if defined(SFV_STREAM_DELAY) && SFV_STREAM_DELAY == 3
            // robustness probe: CTA 5 issues every 32nd level just in time instead of kStages - 1
            // levels ahead, so its compute threads really wait for the TMA copies there
            if (!(rank == 5 && ((l + kStages - 1) & 31) == 7)) issue(l + kStages - 1);
            if (rank == 5 && (l & 31) == 7 && l >= kStages - 1) issue(l);
#elif defined(SFV_STREAM_DELAY) && SFV_STREAM_DELAY == 6
            // ... every CTA, every 8th level
            if (((l + kStages - 1) & 7) != 7) issue(l + kStages - 1);
            if ((l & 7) == 7 && l >= kStages - 1) issue(l);
#else
            issue(l + kStages - 1);
#endif
#ifdef SFV_STREAM_DELAY  // robustness probe: one CTA's producer arrives late at the level's barrier
            if (SFV_STREAM_DELAY == 1 && rank == 5 && (l & 31) == 7) __nanosleep(4000);
#endif
        } else {
#ifdef SFV_STREAM_DELAY  // ... or one CTA's compute threads start their rows late
            if (SFV_STREAM_DELAY == 2 && rank == 5 && (l & 31) == 7) __nanosleep(4000);
#endif
            mbar_wait(mbar_base + 8u * (l % kStages), static_cast<uint32_t>((l / kStages) & 1));
            if (!TSP(32)) {
                t1 = clock64();
                ph[1] += t1 - t0;
                t0 = t1;
            }
            const int s = l % kStages;
            int2 hd = stage_hdr[s];
            if (SFV_STREAM_FIX & 4) {
                int sa, sb;
                slice(l, sa, sb);
                hd = make_int2(sa, sb - sa);
            }
            const int a = hd.x, b = hd.x + hd.y;
            for (int j = threadIdx.x; TSP(16) && j < b - a; j += kThreads) {
                const unsigned char* ch = stage_rec + static_cast<size_t>(s) * kMaxRows * kRec + (j / 32) * kChunk;
                const int ln = j % 32;
                const double* rval = reinterpret_cast<const double*>(ch) + ln;  // [q * 32]
                const uint32_t* rdep = reinterpret_cast<const uint32_t*>(ch + kOffDep) + ln;  // [q * 32]
                uint32_t dep[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) dep[q] = rdep[q * 32];
                double z[NRHS];
#pragma unroll
                for (int k = 0; k < NRHS; ++k) z[k] = stage_src[(s * kMaxRows + j) * 3 + comp + k];
                // Branch-free: an absent dependency reads the +0.0 slot with factor value 0, and
                // z - 0*0 is z bit for bit (also for -0, inf, NaN), as the reference's skipping it.  The eight loads of a right-hand side are one asm statement, so they
                // leave back to back (compiled separately, the scheduler put the eighth after the
                // pivot reciprocal, ~40 instructions later, on the level's critical path).
                // a dep word is the window offset from the ring base (owner << 24 | slot * 8): the
                // load address is one add (ring_lo: the ring base without this CTA's rank byte)
                uint32_t ad[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint32_t d = TSP(64) ? dep[q] : (dep[q] & 0xffffffu) | (static_cast<uint32_t>(rank) << 24);
                    ad[q] = TSP(8) ? d + ring_lo : zero_addr;
                }
                double dv[8][NRHS];
#pragma unroll
                for (int k = 0; k < NRHS; ++k) {
                    uint32_t a8[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) a8[q] = ad[q] + static_cast<uint32_t>(k * ring_s * 8);
                    asm volatile(
                        "ld.shared::cluster.f64 %0, [%8];\n\t"
                        "ld.shared::cluster.f64 %1, [%9];\n\t"
                        "ld.shared::cluster.f64 %2, [%10];\n\t"
                        "ld.shared::cluster.f64 %3, [%11];\n\t"
                        "ld.shared::cluster.f64 %4, [%12];\n\t"
                        "ld.shared::cluster.f64 %5, [%13];\n\t"
                        "ld.shared::cluster.f64 %6, [%14];\n\t"
                        "ld.shared::cluster.f64 %7, [%15];"
                        : "=d"(dv[0][k]), "=d"(dv[1][k]), "=d"(dv[2][k]), "=d"(dv[3][k]), "=d"(dv[4][k]),
                          "=d"(dv[5][k]), "=d"(dv[6][k]), "=d"(dv[7][k])
                        : "r"(a8[0]), "r"(a8[1]), "r"(a8[2]), "r"(a8[3]), "r"(a8[4]), "r"(a8[5]), "r"(a8[6]),
                          "r"(a8[7])
                        : "memory");
                }
                // U: the pivot (read after the loads are out) and its reciprocal overlap their
                // latency; z / dg is finished after them by one correction step (SFV_DIV_CORR)
                double dg = 1.0, rdg = 1.0;
                if (UPPER) {
                    asm volatile("ld.shared.f64 %0, [%1];"
                                 : "=d"(dg)
                                 : "r"(smem_u32(reinterpret_cast<const double*>(ch + kOffDiag) + ln))
                                 : "memory");
                    if (SFV_DIV_CORR) rdg = 1.0 / dg;
                }
                double vq[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) vq[q] = rval[q * 32];
#pragma unroll
                for (int q = 0; q < 8; ++q)  // the reference's order of subtraction
#pragma unroll
                    for (int k = 0; k < NRHS; ++k) z[k] -= vq[q] * dv[q][k];
                if (UPPER) {
#pragma unroll
                    for (int k = 0; k < NRHS; ++k) {
                        if (SFV_DIV_CORR) {
                            // Markstein's correction: with rdg = RN(1 / dg) and q0 = RN(z rdg),
                            // the residual e = z - q0 dg is exact (fma) and RN(q0 + e rdg) is
                            // RN(z / dg) — the same bits as the division, off its latency
                            const double q0 = z[k] * rdg;
                            const double e = __fma_rn(-q0, dg, z[k]);
                            z[k] = __fma_rn(e, rdg, q0);
                        } else {
                            z[k] /= dg;
                        }
                    }
                }
                const int own = reinterpret_cast<const unsigned short*>(ch + kOffOwn)[ln];
                // the backward sweep's position (forward) or the row (backward): no permute /
                // scatter pass after the sweep
                const int oi = reinterpret_cast<const int*>(ch + kOffOutIdx)[ln];
#if defined(SFV_STREAM_DELAY) && SFV_STREAM_DELAY >= 4
                // robustness probe: one thread of CTA 5 stores to a page nobody has touched (a TLB
                // miss in flight) just before the level's ring stores (4) or just after them (5)
                // (7: warp 0 of every CTA, every 4th level, one page per lane)
                const bool cold_store = SFV_STREAM_DELAY == 7 ? j < 32 && (l & 3) == 3 : rank == 5 && j == 0 && (l & 7) == 3;
                double* cold = SFV_STREAM_DELAY == 7
                                   ? tlb_probe + ((static_cast<size_t>(l >> 2) * 48 + comp * 16 + rank) * 32 + j) % (size_t(40) * 288) * (1u << 18)
                                   : tlb_probe + (static_cast<size_t>(comp) * 96 + (l >> 3)) * (1u << 18);
                if ((SFV_STREAM_DELAY == 4 || SFV_STREAM_DELAY == 7) && cold_store) *cold = z[0];
#endif
#pragma unroll
                for (int k = 0; k < NRHS; ++k) {
                    ring[k * ring_s + own] = z[k];
                    if (TSP(2) && oi >= 0) dst[3 * static_cast<size_t>(oi) + comp + k] = z[k];
                }
#if defined(SFV_STREAM_DELAY) && SFV_STREAM_DELAY >= 4
                if (SFV_STREAM_DELAY == 5 && cold_store) *cold = z[0];
#endif
            }
            if (!TSP(32)) {
                t1 = clock64();
                ph[2] += t1 - t0;
                t0 = t1;
            }
            // hand the level over: CTA-scope fence (the values live in this CTA's shared memory)
            if (SFV_STREAM_FIX & 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (SFV_STREAM_FIX & 1) asm volatile("fence.acq_rel.cluster;" ::: "memory");
            else if (TSP(1)) asm volatile("fence.acq_rel.cta;" ::: "memory");
        }
        asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
        if (!TSP(32)) {
            t1 = clock64();
            ph[3] += t1 - t0;
            t0 = t1;
        }
        asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
        if (!TSP(32)) {
            t1 = clock64();
            ph[4] += t1 - t0;
        }
    }
    if (!TSP(32) && (threadIdx.x == 0 || threadIdx.x == kThreads) && (rank == 0 || rank == 15))
        printf("tri_stream U=%d rank %d thr %d levels %d: stage-wait %lld rows %lld fence+arrive %lld "
               "barrier-wait %lld cycles/level\n",
               UPPER ? 1 : 0, rank, threadIdx.x, t.n_levels, ph[1] / t.n_levels, ph[2] / t.n_levels,
               ph[3] / t.n_levels, ph[4] / t.n_levels);
}

template <bool UPPER, int NRHS, int ST>
cudaError_t launch_st(const StreamSet& set, int ncomp, const double* src, double* dst, cudaStream_t s) {
    auto kern = tri_stream_kernel<UPPER, NRHS, ST>;
    const int smem = stream_smem_bytes(set.ring, set.max_rows, ST);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kStreamCluster * (NRHS == 3 ? 1 : ncomp));
    cfg.blockDim = dim3(kThreads + 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kStreamCluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
#if defined(SFV_STREAM_DELAY) && SFV_STREAM_DELAY >= 4
    // 24 GB never written before: every launch gets its own 3 x 96 pages of 2 MB
    static double* probe = [] {
        double* p = nullptr;
        cudaMalloc(&p, size_t(24) << 30);
        return p;
    }();
    static size_t launch = 0;
    double* mine = SFV_STREAM_DELAY == 7 ? probe : probe + (launch++ % 40) * 3 * 96 * (size_t(1) << 18);
    return cudaLaunchKernelEx(&cfg, kern, set, src, dst, mine);
#else
    return cudaLaunchKernelEx(&cfg, kern, set, src, dst);
#endif
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
    return stream_ring_bytes(ring) + stages * max_rows * (kRec + 24) + (kLvl + 2) * 4 + 8 * 8 + 16 + 8 * 8;
}

cudaError_t launch_tri_stream(const StreamSet& set, bool upper, int ncomp, const double* src, double* dst,
                              cudaStream_t s) {
    // one 16-CTA cluster per component also for the shared factor: three concurrent sweeps
    // with a third of the DSMEM loads each beat one sweep carrying three right-hand sides
    // (0.86 vs 1.28 ms per apply at 1M cells).  SFV_STREAM_SPLIT=0 restores the latter.
    static const bool split = [] {
        const char* e = std::getenv("SFV_STREAM_SPLIT");
        return !e || std::atoi(e) != 0;
    }();
    if (ncomp == 1 && split) {
        StreamSet s3 = set;
        s3.t[1] = s3.t[2] = set.t[0];
        return upper ? launch_one<true, 1>(s3, 3, src, dst, s) : launch_one<false, 1>(s3, 3, src, dst, s);
    }
    if (upper) return ncomp == 1 ? launch_one<true, 3>(set, 1, src, dst, s) : launch_one<true, 1>(set, 3, src, dst, s);
    return ncomp == 1 ? launch_one<false, 3>(set, 1, src, dst, s) : launch_one<false, 1>(set, 3, src, dst, s);
}

}  // namespace sfv
