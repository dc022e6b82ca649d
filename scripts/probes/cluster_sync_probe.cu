// Probe: cost of one level hand-over in a 16-CTA cluster (the ILU sweep's skeleton).
//   mode 0: barrier.cluster.arrive.relaxed + barrier.cluster.wait (the sweep's current hand-over)
//   mode 1: all-to-all flags: after level l every CTA writes l+1 into slot[rank] of every
//           other CTA's shared memory (one remote st per thread t < 16), then waits until its
//           16 local slots reach l+1 (one thread per slot polls, then a CTA barrier)
//   mode 2: mode 1 with st.async? (not used) -> plain remote st.relaxed.cluster
// Prints cycles per level measured with clock64 in CTA 0.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

template <int MODE>
__global__ void probe(int levels, long long* out) {
    __shared__ volatile int slot[16];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = cl.block_rank();
    if (threadIdx.x < 16) slot[threadIdx.x] = 0;
    cl.sync();
    long long t0 = clock64();
    for (int l = 0; l < levels; ++l) {
        if (MODE == 0) {
            asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
            asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
        } else {
            __syncthreads();  // this CTA's rows are done
            if (threadIdx.x < 16) {
                asm volatile("fence.acq_rel.cta;" ::: "memory");
                unsigned a = smem_u32((const void*)&slot[rank]);
                unsigned r;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"((int)threadIdx.x));
                asm volatile("st.relaxed.cluster.shared::cluster.u32 [%0], %1;" ::"r"(r), "r"(l + 1) : "memory");
                while (slot[threadIdx.x] < l + 1) {
                }
            }
            __syncthreads();
        }
    }
    long long t1 = clock64();
    if (rank == 0 && threadIdx.x == 0) out[MODE] = (t1 - t0) / levels;
}

int main() {
    long long* d;
    cudaMalloc(&d, 8 * sizeof(long long));
    auto launch = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(48);
        cfg.blockDim = dim3(288);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 16;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, 2000, d);
    };
    for (int rep = 0; rep < 2; ++rep) {
        launch(probe<0>);
        launch(probe<1>);
        cudaDeviceSynchronize();
    }
    long long h[8];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("cycles per level: barrier.cluster %lld, all-to-all flags %lld  (err %s)\n", h[0], h[1],
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
