// Probe: the shared::cluster address mapa returns, against (rank << 24) | local offset.
#include <cooperative_groups.h>
#include <cstdio>
__global__ void k(unsigned* out) {
    __shared__ double buf[64];
    buf[threadIdx.x] = 0.0;
    unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(&buf[3]));
    if (threadIdx.x < 16) {
        unsigned r;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"((int)threadIdx.x));
        out[2 * threadIdx.x] = r;
        out[2 * threadIdx.x + 1] = a;
    }
}
int main() {
    unsigned* d;
    cudaMalloc(&d, 64 * sizeof(unsigned));
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(64);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, d);
    unsigned h[32];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    for (int r = 0; r < 16; ++r) printf("rank %d: mapa %08x local %08x ((r<<24)|a = %08x)\n", r, h[2 * r], h[2 * r + 1], (r << 24) | h[2 * r + 1]);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
