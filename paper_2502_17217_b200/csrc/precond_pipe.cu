// precond_pipe.cu — block-pipelined ILU(k) triangular sweep (sm_100a).
//
// Same arithmetic as IlukPrecond::solve (/root/reference/proj/src/linalg.cpp:302-316), one
// component per 16-CTA cluster.  Instead of one cluster-wide barrier per dependency level
// (precond_stream.cu: 595 levels per sweep at 1M cells, ~0.6 us each), the rows in sweep
// order are cut into 16 contiguous blocks, CTA b owning block b (build_pipe in
// precond_host.cpp).  CTA b walks only the levels present in its block ("steps"):
//
//   consumers (kPipeThreads): per step, wait until the producer has cleared it, compute the
//     step's rows (dependencies in this CTA's value ring, or — bit 31 — in block b-1's ring
//     over DSMEM), store value to the ring and to dst, named barrier among consumers, bump
//     `done`.  Each thread's record for the next step is loaded into registers while the
//     current step computes;
//   producer warp: clears step s once block b-1 has published need[s] steps (the data) and
//     block b+1 has published guard[s] steps (the ring slots step s rewrites have been read
//     remotely), and prefetches the records of later steps into L2;
//   publisher warp: on every `done` bump, a cluster-scope release fence then the progress
//     store read by the neighbours — the expensive fence is off the consumers' path.
//
// Local dependencies are ordered by the consumers' named barrier; remote ones by the
// release (publisher) / acquire (neighbour's producer) pair on the progress word, passed to
// the consumers through per-step mbarriers (hardware-suspended waits).
// Compiled with -fmad=false: bit-identical results.
//
// Status: opt-in (SFV_PIPE=1).  Measured at 1M cells it is slower than the streamed
// level-synchronous sweep (2.3 vs 0.86 ms per apply).  With ILU(1) fill a row's level is
// ~2(i+j+k) on the box, so block b (planes 6.25b..6.25b+6) trails block b-1 by ~12 steps
// and the pipelined critical path is 15 x 12 + ~412 ~ 590 steps: no shorter than the 595
// levels it replaces.  It can only win on the cost of a step, and a step (wait for the
// producer's clearance, rows, named barrier) measured ~2 us here against ~0.7 us per level
// there; relaxing the publisher's cluster fence and the neighbours' acquire polls
// (-DSFV_PIPE_PROBE=2|4) moved it by < 10%.
#include <cooperative_groups.h>
#include <cstdio>

#include "device.h"

namespace cg = cooperative_groups;

// -DSFV_PIPE_PROBE=1: per-role clock64 totals of every CTA printed at exit (timing only)
#ifndef SFV_PIPE_PROBE
#define SFV_PIPE_PROBE 0
#endif

namespace sfv {
namespace {

constexpr int kPT = kPipeThreads;  // consumer threads
constexpr int kPrefetchSteps = 8;  // L2 prefetch distance of the producer

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t addr, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cluster(uint32_t cluster_addr) {
    int v;
#if SFV_PIPE_PROBE & 4  // timing probe: relaxed poll
    asm volatile("ld.relaxed.cluster.shared::cluster.b32 %0, [%1];" : "=r"(v) : "r"(cluster_addr) : "memory");
#else
    asm volatile("ld.acquire.cluster.shared::cluster.b32 %0, [%1];" : "=r"(v) : "r"(cluster_addr) : "memory");
#endif
    return v;
}
__device__ __forceinline__ void mbar_init(uint32_t a, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(a),
        "r"(parity)
        : "memory");
}
constexpr int kClear = 4;  // steps the producer may clear ahead of the consumers (mbarrier ring)
__device__ __forceinline__ void bar_consumers() { asm volatile("bar.sync 1, %0;" ::"n"(kPT) : "memory"); }

struct Row {  // one position's record (registers)
    uint32_t dep[8];
    double val[8];
    double diag;
    double rhs;
};

__device__ __forceinline__ void load_row(const unsigned char* __restrict__ rec, const double* __restrict__ src, int p,
                                         int comp, Row& r) {
    const unsigned char* ch = rec + static_cast<size_t>(p / 32) * kPipeChunk;
    const int ln = p % 32;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        r.dep[q] = __ldcs(reinterpret_cast<const unsigned*>(ch + 2304) + q * 32 + ln);
        r.val[q] = __ldcs(reinterpret_cast<const double*>(ch) + q * 32 + ln);
    }
    r.diag = __ldcs(reinterpret_cast<const double*>(ch + 2048) + ln);
    r.rhs = src[3 * static_cast<size_t>(p) + comp];
}

template <bool UPPER>
__global__ void __launch_bounds__(kPT + 64, 1) tri_pipe_kernel(PipeSet set, const double* __restrict__ src,
                                                               double* __restrict__ dst) {
    cg::cluster_group cluster = cg::this_cluster();
    const int b = static_cast<int>(cluster.block_rank());
    const int comp = static_cast<int>(blockIdx.x / kPipeCluster);
    const DevPipe& t = set.t[comp];
    const int ring_n = set.ring;
    extern __shared__ __align__(16) unsigned char smem[];
    double* ring = reinterpret_cast<double*>(smem);                 // [ring_n]
    int* flags = reinterpret_cast<int*>(ring + ring_n);             // prog, done
    int* prog = flags;
    int* done = flags + 1;
    unsigned long long* clear = reinterpret_cast<unsigned long long*>(flags + 2);  // [kClear] mbarriers
    const uint32_t clear_base = smem_u32(clear);
    const int tid = threadIdx.x;
    if (tid == 0) {
        *prog = 0;
        *done = 0;
    }
    if (tid < kClear) mbar_init(clear_base + 8u * tid, 1);
    cluster.sync();  // counters initialised before any neighbour polls them
    const int base = t.step_off[b];
    const int nsteps = t.step_off[b + 1] - base;
    const int* ptr = t.step_ptr + base + b;  // [nsteps + 1] positions
    if (tid < kPT) {
        // ------------------------------------------------------------ consumers
        Row cur, nxt;
        const int pbase = ptr[0];
        int a0 = pbase, e0 = nsteps > 0 ? ptr[1] : a0;
        if (nsteps > 0 && tid < e0 - a0) load_row(t.rec, src, a0 + tid, comp, cur);
        long long tw = 0, tc = 0, tb = 0, t0 = 0;
        (void)tw;
        (void)tc;
        (void)tb;
        (void)t0;
        for (int s = 0; s < nsteps; ++s) {
            const int a = a0, e = e0;
            int an = e, en = e;
            if (s + 1 < nsteps) {
                an = ptr[s + 1];
                en = ptr[s + 2];
                if (tid < en - an) load_row(t.rec, src, an + tid, comp, nxt);  // in flight during step s
            }
            if (SFV_PIPE_PROBE & 1) t0 = clock64();
            mbar_wait(clear_base + 8u * (s % kClear), static_cast<uint32_t>((s / kClear) & 1));
            if (SFV_PIPE_PROBE & 1) {
                const long long t1 = clock64();
                tw += t1 - t0;
                t0 = t1;
            }
            for (int j = tid; j < e - a; j += kPT) {
                Row r;
                if (j == tid)
                    r = cur;
                else
                    load_row(t.rec, src, a + j, comp, r);
                double dv[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {  // every dependency load in flight together
                    const uint32_t d = r.dep[q];
                    dv[q] = 0.0;
                    if (d != 0xffffffffu) {
                        const uint32_t slot = d & 0x7fffffffu;
                        if (d & 0x80000000u) {
                            const uint32_t ad = mapa(smem_u32(ring + slot), b - 1);
                            asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(dv[q]) : "r"(ad));
                        } else {
                            dv[q] = ring[slot];
                        }
                    }
                }
                double z = r.rhs;
#pragma unroll
                for (int q = 0; q < 8; ++q)  // the reference's order of subtraction
                    if (r.dep[q] != 0xffffffffu) z -= r.val[q] * dv[q];
                if (UPPER) z /= r.diag;
                const int p = a + j;
                ring[(p - pbase) & (ring_n - 1)] = z;
                dst[3 * static_cast<size_t>(p) + comp] = z;
            }
            if (SFV_PIPE_PROBE & 1) {
                const long long t1 = clock64();
                tc += t1 - t0;
                t0 = t1;
            }
            bar_consumers();
            if (SFV_PIPE_PROBE & 1) tb += clock64() - t0;
            if (tid == 0) st_release_cta(done, s + 1);
            cur = nxt;
            a0 = an;
            e0 = en;
        }
        if ((SFV_PIPE_PROBE & 1) && tid == 0)
            printf("pipe U=%d comp %d block %d steps %d: consumer wait %lld compute %lld bar %lld cycles/step\n",
                   UPPER ? 1 : 0, comp, b, nsteps, tw / max(nsteps, 1), tc / max(nsteps, 1), tb / max(nsteps, 1));
    } else if (tid == kPT) {
        // ------------------------------------------------------------ producer
        const uint32_t prev = b > 0 ? mapa(smem_u32(prog), b - 1) : 0u;
        const uint32_t next = b + 1 < kPipeCluster ? mapa(smem_u32(prog), b + 1) : 0u;
        int pv = 0, nx = 0;
        long long tp = 0, tn = 0, t0 = 0;
        (void)tp;
        (void)tn;
        (void)t0;
        for (int s = 0; s < nsteps; ++s) {
            if (s + kPrefetchSteps < nsteps) {  // records of a later step into L2
                const int pa = ptr[s + kPrefetchSteps], pe = ptr[s + kPrefetchSteps + 1];
                const unsigned char* from = t.rec + static_cast<size_t>(pa / 32) * kPipeChunk;
                const uint32_t bytes = static_cast<uint32_t>((pe - pa) / 32) * kPipeChunk;
                if (bytes)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(from), "r"(bytes) : "memory");
            }
            const int nd = t.need[base + s], gd = t.guard[base + s];
            if (SFV_PIPE_PROBE & 1) t0 = clock64();
            if (b > 0)
                while (pv < nd) pv = ld_acquire_cluster(prev);
            if (SFV_PIPE_PROBE & 1) {
                const long long t1 = clock64();
                tp += t1 - t0;
                t0 = t1;
            }
            if (b + 1 < kPipeCluster)
                while (nx < gd) nx = ld_acquire_cluster(next);
            if (SFV_PIPE_PROBE & 1) tn += clock64() - t0;
            // the mbarrier slot of step s was last used by step s - kClear
            while (ld_acquire_cta(done) < s - kClear + 1) __nanosleep(32);
            mbar_arrive(clear_base + 8u * (s % kClear));
        }
        if (SFV_PIPE_PROBE & 1)
            printf("pipe U=%d comp %d block %d: producer wait prev %lld next %lld cycles total, start %lld\n",
                   UPPER ? 1 : 0, comp, b, tp, tn, 0LL);
    } else if (tid == kPT + 32) {
        // ------------------------------------------------------------ publisher
        int pub = 0, npub = 0;
        long long tf = 0;
        (void)tf;
        while (pub < nsteps) {
            const int d = ld_acquire_cta(done);
            if (d == pub) {
                __nanosleep(32);
                continue;
            }
            const long long t0 = (SFV_PIPE_PROBE & 1) ? clock64() : 0;
#if SFV_PIPE_PROBE & 2  // timing probe: CTA-scope fence instead of the cluster-scope release
            asm volatile("fence.acq_rel.cta;" ::: "memory");
#else
            asm volatile("fence.acq_rel.cluster;" ::: "memory");
#endif
            if (SFV_PIPE_PROBE & 1) {
                tf += clock64() - t0;
                ++npub;
            }
            asm volatile("st.relaxed.cluster.shared.b32 [%0], %1;" ::"r"(smem_u32(prog)), "r"(d) : "memory");
            pub = d;
        }
        if (SFV_PIPE_PROBE & 1)
            printf("pipe U=%d comp %d block %d: publisher %d publishes, fence %lld cycles each\n", UPPER ? 1 : 0,
                   comp, b, npub, tf / max(npub, 1));
    }
    cluster.sync();  // no CTA leaves while a neighbour may still read its ring
}

}  // namespace

int pipe_smem_bytes(int ring) { return ring * 8 + 8 + 8 * kClear; }

cudaError_t launch_tri_pipe(const PipeSet& set, bool upper, const double* src, double* dst, cudaStream_t s) {
    auto kern = upper ? tri_pipe_kernel<true> : tri_pipe_kernel<false>;
    const int smem = pipe_smem_bytes(set.ring);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kPipeCluster * 3);
    cfg.blockDim = dim3(kPT + 64);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kPipeCluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, set, src, dst);
}

}  // namespace sfv
