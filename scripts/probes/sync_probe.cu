// sync_probe.cu — cost of one level of a level-synchronous sweep on B200, by primitive:
// (a) barrier.cluster arrive.release/wait.acquire, 16 CTAs x 512 threads, no memory traffic
// (b) the same with one L2 store + dependent L2 load per thread per level
// (c) __syncthreads in one CTA of 1024 threads with the same store/load (L1/L2)
// (d) grid-stride "flag chain": CTA b waits on CTA b-1's per-level counter (ld.acquire)
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <bool MEM>
__global__ void cluster_levels(int levels, double* buf, int n) {
    cg::cluster_group cl = cg::this_cluster();
    const int tid = cl.block_rank() * blockDim.x + threadIdx.x;
    const int nthr = cl.num_threads();
    double acc = 0.0;
    for (int l = 0; l < levels; ++l) {
        if (MEM) {
            const int src = (tid * 7 + l * 131) % nthr;
            acc += __ldcg(&buf[(size_t)(l & 1) * nthr + src]);
            __stcg(&buf[(size_t)((l + 1) & 1) * nthr + tid], acc);
        }
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (acc == 123.456) buf[0] = acc;
}

__global__ void cta_levels(int levels, double* buf) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    double acc = 0.0;
    for (int l = 0; l < levels; ++l) {
        const int src = (tid * 7 + l * 131) % nthr;
        acc += buf[(size_t)(l & 1) * nthr + src];
        buf[(size_t)((l + 1) & 1) * nthr + tid] = acc;
        __syncthreads();
    }
    if (acc == 123.456) buf[0] = acc;
}

__device__ __forceinline__ int ld_acq(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// each CTA b, level l: wait counter[b-1] >= l+1 (previous CTA finished level l), work, publish
__global__ void chain_levels(int levels, double* buf, int* counter) {
    const int b = blockIdx.x;
    double acc = 0.0;
    for (int l = 0; l < levels; ++l) {
        if (b > 0 && threadIdx.x == 0)
            while (ld_acq(&counter[b - 1]) < l + 1) {}
        __syncthreads();
        acc += __ldcg(&buf[(size_t)b * blockDim.x + threadIdx.x]);
        __stcg(&buf[(size_t)b * blockDim.x + threadIdx.x], acc);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            st_rel(&counter[b], l + 1);
        }
    }
}

int main() {
    const int levels = 1190;
    double* buf;
    int* cnt;
    cudaMalloc(&buf, 1 << 24);
    cudaMalloc(&cnt, 4096);
    cudaMemset(buf, 0, 1 << 24);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run_cluster = [&](auto kern, int csize, const char* name) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(csize);
        cfg.blockDim = dim3(512);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim = {(unsigned)csize, 1, 1};
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        for (int w = 0; w < 2; ++w) cudaLaunchKernelEx(&cfg, kern, levels, buf, 0);
        cudaEventRecord(a);
        cudaLaunchKernelEx(&cfg, kern, levels, buf, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-34s csize=%2d  %.3f us/level  (%s)\n", name, csize, 1e3 * ms / levels, cudaGetErrorString(cudaGetLastError()));
    };
    for (int cs : {2, 4, 8, 16}) run_cluster(cluster_levels<false>, cs, "cluster barrier only");
    for (int cs : {2, 4, 8, 16}) run_cluster(cluster_levels<true>, cs, "cluster barrier + L2 st/ld");
    {
        for (int w = 0; w < 2; ++w) cta_levels<<<1, 1024>>>(levels, buf);
        cudaEventRecord(a);
        cta_levels<<<1, 1024>>>(levels, buf);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-34s           %.3f us/level\n", "single CTA bar.sync + st/ld", 1e3 * ms / levels);
    }
    for (int nb : {2, 8, 32}) {
        cudaMemset(cnt, 0, 4096);
        cudaEventRecord(a);
        chain_levels<<<nb, 256>>>(levels, buf, cnt);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-34s nb=%2d     %.3f us/level (pipelined chain, total %.3f ms)\n", "flag chain CTA b waits b-1", nb,
               1e3 * ms / levels, ms);
    }
    return 0;
}
