// krylov.cu — GMRES Arnoldi vector work and Newton vector ops (FP64, sm_100a).
//
// Restates the vector kernels of gmres_solve (/root/reference/proj/src/linalg.cpp:423-538):
// modified Gram-Schmidt (:469-473) as a chain of fused "w -= h_i v_i ; h_{i+1} = w.v_{i+1}"
// passes, the basis normalisation (:500-501), the correction x += V y (:512-515), and the
// Newton/stepping vector updates of nonlinear.cpp.  Every reduction is a fixed-order
// two-level tree (block partials, then one last block in block order), so results are
// run-to-run deterministic; the scalar h_i never leaves the device between passes.
#include <cfloat>

#include <cooperative_groups.h>

#include "device.h"

namespace cg = cooperative_groups;

namespace sfv {
namespace {

constexpr int kT = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int s = kT / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    return sh[0];
}

// last-block finalisation: returns true in the block that must sum the partials
__device__ __forceinline__ bool publish_partial(double part, double* partial, unsigned* counter) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
        partial[blockIdx.x] = part;
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    return last;
}

__device__ __forceinline__ void finish_sum(const double* partial, unsigned* counter, double* out, double* sh) {
    __threadfence();
    double t = 0.0;
    for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x) t += __ldcg(&partial[b]);
    const double tot = block_sum(t, sh);
    if (threadIdx.x == 0) {
        *out = tot;
        *counter = 0u;
    }
}

__global__ void __launch_bounds__(kT) dot_kernel(const double* __restrict__ a, const double* __restrict__ b, int n,
                                                 double* __restrict__ out, double* partial, unsigned* counter) {
    __shared__ double sh[kT];
    double acc = 0.0;
    const int st = gridDim.x * kT;
    int i = blockIdx.x * kT + threadIdx.x;
    // the plain grid-stride order, 8 iterations' loads issued together (same sums)
    for (; i + 7 * st < n; i += 8 * st) {
        double x[8], y[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            x[k] = a[i + k * st];
            y[k] = b[i + k * st];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += x[k] * y[k];
    }
    for (; i < n; i += st) acc += a[i] * b[i];
    const double part = block_sum(acc, sh);
    if (publish_partial(part, partial, counter)) finish_sum(partial, counter, out, sh);
}

__global__ void __launch_bounds__(kT) axpy_dot_kernel(double* __restrict__ w, const double* __restrict__ vi,
                                                      const double* __restrict__ h, const double* __restrict__ vnext,
                                                      int n, double* __restrict__ out, double* partial,
                                                      unsigned* counter) {
    __shared__ double sh[kT];
    const double hi = *h;
    double acc = 0.0;
    const int st = gridDim.x * kT;
    int i = blockIdx.x * kT + threadIdx.x;
    for (; i + 3 * st < n; i += 4 * st) {  // 4 iterations' loads together, same order
        double x[4], y[4], z[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            x[k] = w[i + k * st];
            y[k] = vi[i + k * st];
            z[k] = vnext ? vnext[i + k * st] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double wn = x[k] + (-hi) * y[k];  // axpy(-h_i, v_i, w): w += (-h_i) v_i
            w[i + k * st] = wn;
            acc += vnext ? wn * z[k] : wn * wn;
        }
    }
    for (; i < n; i += st) {
        const double wn = w[i] + (-hi) * vi[i];
        w[i] = wn;
        acc += vnext ? wn * vnext[i] : wn * wn;
    }
    const double part = block_sum(acc, sh);
    if (publish_partial(part, partial, counter)) finish_sum(partial, counter, out, sh);
}

// ---------------------------------------------------------------- reference-order sums
// The reference sums every inner product left to right from 0.0 (std::inner_product,
// linalg.cpp:18-22; vec_norm / field_norm, nonlinear.cpp:13-24): s = RN(s + RN(a_i b_i)).
// That chain cannot be re-associated without changing the bits, so these kernels run it as
// the chain it is: one CTA, warps 1.. form the products of the next chunk in shared memory
// while thread 0 adds the current chunk in index order (one dependent DADD per term, ~13 ms
// per 3M-term sum on B200).  Two sums may share the launch (two independent chains
// interleaved in thread 0: the J.v's |v| and |u|).  Opt-in (sfv_set_option
// "sequential_reductions"): it makes every Krylov and Newton decision bit-identical to the
// CPU reference's, at full size, where a parallel tree differs in the last bits.
constexpr int kSeqT = 512;
constexpr int kSeqChunk = 1024;  // 2 stages x 2 sums x 8 KB of static shared memory

__global__ void __launch_bounds__(kSeqT, 1) seq_dot2_kernel(const double* __restrict__ a1, const double* __restrict__ b1,
                                                          const double* __restrict__ a2, const double* __restrict__ b2,
                                                          int n, double* __restrict__ out1, double* __restrict__ out2) {
    __shared__ double buf[2][2][kSeqChunk];  // [stage][sum][term]
    const bool two = a2 != nullptr;
    const int nch = (n + kSeqChunk - 1) / kSeqChunk;
    auto produce = [&](int k, int t0, int nt) {
        const int base = k * kSeqChunk;
        const int m = min(kSeqChunk, n - base);
        double* p1 = buf[k & 1][0];
        double* p2 = buf[k & 1][1];
        for (int i = t0; i < m; i += nt) {
            p1[i] = __dmul_rn(a1[base + i], b1[base + i]);
            if (two) p2[i] = __dmul_rn(a2[base + i], b2[base + i]);
        }
    };
    if (nch > 0) produce(0, threadIdx.x, kSeqT);
    __syncthreads();
    double s1 = 0.0, s2 = 0.0;
    for (int k = 0; k < nch; ++k) {
        if (threadIdx.x == 0) {
            const int m = min(kSeqChunk, n - k * kSeqChunk);
            const double* p1 = buf[k & 1][0];
            const double* p2 = buf[k & 1][1];
            int i = 0;
            for (; i + 8 <= m; i += 8) {
                double x[8], y[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    x[q] = p1[i + q];
                    y[q] = two ? p2[i + q] : 0.0;
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    s1 = __dadd_rn(s1, x[q]);
                    if (two) s2 = __dadd_rn(s2, y[q]);
                }
            }
            for (; i < m; ++i) {
                s1 = __dadd_rn(s1, p1[i]);
                if (two) s2 = __dadd_rn(s2, p2[i]);
            }
        } else if (threadIdx.x >= 32 && k + 1 < nch) {
            produce(k + 1, threadIdx.x - 32, kSeqT - 32);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *out1 = s1;
        if (two) *out2 = s2;
    }
}

// ε of jacobian_vector_product (nonlinear.cpp:109-115) from reference-order |v| and |u|:
// eps_out[0] = ε (0 when |v| = 0), u_norm = |u| (read instead when cached)
__global__ void seq_eps_finish_kernel(const double* __restrict__ sums, double* __restrict__ eps_out,
                                      double* __restrict__ u_norm, bool cached) {
    const double vn = sqrt(sums[0]);
    const double un = cached ? *u_norm : sqrt(sums[1]);
    *eps_out = vn == 0.0 ? 0.0 : sqrt(DBL_EPSILON) * sqrt(1.0 + un) / vn;
    if (!cached) *u_norm = un;
}

// w += (-h) v  (axpy(-h_i, v_i, w), linalg.cpp:471), h on the device
__global__ void axpy_neg_dev_kernel(double* __restrict__ w, const double* __restrict__ vi, const double* __restrict__ h,
                                    int n) {
    const double hi = *h;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        w[i] = w[i] + (-hi) * vi[i];
}

__global__ void scale_div_kernel(const double* __restrict__ in, const double* __restrict__ d, double dh,
                                 double* __restrict__ out, int n) {
    const double s = d ? *d : dh;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[i] / s;
}

// dx = sum_i y_i v_i accumulated in i order from zero, then x += dx (linalg.cpp:512-515)
// dx = sum_i y_i v_i in the reference's axpy order (linalg.cpp:513), then x += 1.0 * dx
// (:515), or dx alone into dx_out (right preconditioning applies M^-1 to it first, :514)
__global__ void update_kernel(double* __restrict__ x, double* __restrict__ dx_out, const double* __restrict__ V,
                              const double* __restrict__ y, int j, int n) {
    extern __shared__ double ys[];  // [j]
    for (int i = threadIdx.x; i < j; i += blockDim.x) ys[i] = y[i];
    __syncthreads();
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        double dx = 0.0;
        for (int i = 0; i < j; ++i) dx += ys[i] * V[static_cast<size_t>(i) * n + e];
        if (dx_out) dx_out[e] = dx;
        else x[e] += 1.0 * dx;
    }
}

__global__ void sub_from_kernel(const double* __restrict__ b, double* __restrict__ r, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) r[i] = b[i] - r[i];
}

__global__ void negate_kernel(const double* __restrict__ a, double* __restrict__ o, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) o[i] = -a[i];
}

__global__ void axpy_kernel(double* __restrict__ y, double alpha, const double* __restrict__ x, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] += alpha * x[i];
}

__global__ void lincomb_kernel(double* __restrict__ o, const double* __restrict__ u, double s,
                               const double* __restrict__ du, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) o[i] = u[i] + du[i] * s;
}

// run_steps history rotation (nonlinear.cpp:427-437): v_new, a_new by BDF2 then shift
__global__ void bdf2_rotate_kernel(double* uo, double* uoo, double* vo, double* voo, double* ao,
                                   const double* __restrict__ u, double dt, int n) {
    const double idt = 1.0 / (2.0 * dt);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double un = u[i], ut = uo[i], utm1 = uoo[i], vt = vo[i], vtm1 = voo[i];
        const double vn = ((un * 3.0 - ut * 4.0) + utm1) * idt;
        const double an = ((vn * 3.0 - vt * 4.0) + vtm1) * idt;
        uoo[i] = ut;
        uo[i] = un;
        voo[i] = vt;
        vo[i] = vn;
        ao[i] = an;
    }
}

// predict_step_start, transient branch (nonlinear.cpp:165-171)
__global__ void predict_kernel(double* __restrict__ u, const double* __restrict__ uo, const double* __restrict__ vo,
                               const double* __restrict__ ao, double dt, int n) {
    const double h = 0.5 * dt * dt;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        u[i] = (uo[i] + vo[i] * dt) + ao[i] * h;
}

// ---------------------------------------------------------------- fused Arnoldi step
// One cooperative launch per Arnoldi step: the SM-resident grid holds w in shared memory
// (one contiguous chunk per CTA), so the modified Gram-Schmidt chain of linalg.cpp:469-473
// — h_i = w.v_i ; w -= h_i v_i, i = 0..j — streams each basis vector once and never
// writes w back; then h_{j+1} = w.w and v_{j+1} = w / sqrt(h_{j+1}) (linalg.cpp:500-501).
// Each dot is a fixed-order reduction (thread, warp, block in order, then every block
// sums the block partials in block order), so all CTAs agree on h_i bit for bit.
constexpr int kAT = 1024;

__device__ __forceinline__ double warp_sum_d(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    return x;
}
__device__ __forceinline__ double block_sum_fixed(double v, double* sh) {  // result valid in thread 0
    v = warp_sum_d(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = l < kAT / 32 ? sh[l] : 0.0;
        r = warp_sum_d(r);
    }
    __syncthreads();
    return r;
}

constexpr int kAK = 24;  // elements of a basis vector per thread held in registers (n <= 148 * 1024 * 24)

__global__ void __launch_bounds__(kAT, 1) arnoldi_kernel(const double* __restrict__ w_in, const double* __restrict__ V,
                                                        int n, int j, int chunk, double* __restrict__ h,
                                                        double* __restrict__ partial, double* __restrict__ vnext,
                                                        const int* __restrict__ jdev, int vcap) {
    // device-resident cycle (gmres graph): the step index is the cycle state's, and
    // v_{j+1} goes to V[j + 1] when the basis has room for it
    if (jdev) {
        j = *jdev;
        vnext = j + 1 < vcap ? const_cast<double*>(V) + static_cast<size_t>(j + 1) * n : nullptr;
    }
    extern __shared__ double wsh[];  // [chunk]
    __shared__ double sh[kAT / 32];
    __shared__ double bcast;
    cg::grid_group grid = cg::this_grid();
    const int lo = blockIdx.x * chunk;
    const int cnt = max(0, min(chunk, n - lo));
    {  // w into shared memory: all of this thread's loads in flight together
        double x[kAK];
#pragma unroll
        for (int k = 0; k < kAK; ++k) {
            const int e = threadIdx.x + k * kAT;
            x[k] = e < cnt ? w_in[lo + e] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < kAK; ++k) {
            const int e = threadIdx.x + k * kAT;
            if (e < cnt) wsh[e] = x[k];
        }
    }
    __syncthreads();
    const int G = gridDim.x;
    for (int i = 0; i <= j + 1; ++i) {
        const bool norm = i == j + 1;
        const double* vi = V + static_cast<size_t>(i) * n + lo;
        // this thread's slice of v_i (elements threadIdx.x + k kAT) stays in registers for
        // the update after the dot: each basis vector is read once
        double vr[kAK];
#pragma unroll
        for (int k = 0; k < kAK; ++k) {
            const int e = threadIdx.x + k * kAT;
            vr[k] = e < cnt ? (norm ? wsh[e] : vi[e]) : 0.0;
        }
        double acc = 0.0;  // fixed order within the thread (ascending e)
#pragma unroll
        for (int k = 0; k < kAK; ++k) {
            const int e = threadIdx.x + k * kAT;
            if (e < cnt) acc += wsh[e] * vr[k];
        }
        const double bs = block_sum_fixed(acc, sh);
        double* part = partial + (i & 1) * G;  // alternate buffers: no block overwrites one still being read
        if (threadIdx.x == 0) part[blockIdx.x] = bs;
        grid.sync();
        double t = 0.0;
        for (int b = threadIdx.x; b < G; b += kAT) t += __ldcg(&part[b]);
        const double hi = block_sum_fixed(t, sh);
        if (threadIdx.x == 0) {
            bcast = hi;
            if (blockIdx.x == 0) h[i] = hi;
        }
        __syncthreads();
        const double hv = bcast;
        if (norm) {
            if (vnext) {  // v_{j+1} = w / |w|
                const double nr = sqrt(hv);
#pragma unroll
                for (int k = 0; k < kAK; ++k) {
                    const int e = threadIdx.x + k * kAT;
                    if (e < cnt) vnext[lo + e] = vr[k] / nr;
                }
            }
            break;
        }
#pragma unroll
        for (int k = 0; k < kAK; ++k) {  // w += (-h_i) v_i
            const int e = threadIdx.x + k * kAT;
            if (e < cnt) wsh[e] = wsh[e] + (-hv) * vr[k];
        }
        // (each thread rewrites only its own w elements: no barrier needed before the next dot)
    }
}

// ---------------------------------------------------------------- device-resident GMRES step
// The host part of one Arnoldi step of gmres_solve (linalg.cpp:474-498) on the device, one
// thread: the new Hessenberg column from the Arnoldi kernel's h (h[j+1] = w.w), the stored
// Givens rotations, the new rotation, the residual estimate g, the happy-breakdown and target
// tests, the restart / budget limits, and any error word a J.v of this step raised.  It sets
// the WHILE condition of the cycle graph (capi.cpp: gmres_graph), so the whole restart cycle
// runs without a host round trip.  Same expressions as the host loop in capi.cpp: gmres.
__global__ void givens_kernel(GmresDev st, const double* __restrict__ h, const ErrWords* __restrict__ err,
                              cudaGraphConditionalHandle cond) {
    GmresHdr& hd = *st.hdr;
    const int j = hd.j, m = hd.restart;
    double* col = st.H + static_cast<size_t>(j) * (m + 1);
    for (int i = 0; i <= j; ++i) col[i] = h[i];
    col[j + 1] = sqrt(h[j + 1]);
    for (int i = 0; i < j; ++i) {  // apply stored rotations
        const double t = st.cs[i] * col[i] + st.sn[i] * col[i + 1];
        col[i + 1] = -st.sn[i] * col[i] + st.cs[i] * col[i + 1];
        col[i] = t;
    }
    const double denom = sfv_hypot(col[j], col[j + 1]);
    const double cc = denom == 0.0 ? 1.0 : col[j] / denom;
    const double ss = denom == 0.0 ? 0.0 : col[j + 1] / denom;
    st.cs[j] = cc;
    st.sn[j] = ss;
    st.g[j + 1] = -ss * st.g[j];
    st.g[j] = cc * st.g[j];
    col[j] = denom;
    const double subdiag = col[j + 1];
    col[j + 1] = 0.0;
    hd.total += 1;
    hd.j = j + 1;
    constexpr int none = 0x7f7f7f7f;
    const bool bad = err->nan_jv != none || err->nan_cell != none || err->inverted_cell != none ||
                     err->inverted_face != none || err->overflow_cell != none || err->retmap_cell != none;
    hd.happy = subdiag <= 1e-14 * fmax(denom, 1e-300) ? 1 : 0;
    const bool stop = bad || hd.happy || fabs(st.g[j + 1]) <= hd.target || j + 1 >= m || hd.total >= hd.max_iters;
    cudaGraphSetConditional(cond, stop ? 0u : 1u);
}

int grid_for(int n) {
    const int b = (n + 255) / 256;
    return b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16;
}

}  // namespace

int reduce_blocks(int n) {
    const int b = (n + kT * 4 - 1) / (kT * 4);
    return b < 1 ? 1 : (b > 148 * 8 ? 148 * 8 : b);
}

void launch_dot(const double* a, const double* b, int n, double* out, double* scratch, unsigned* counter,
                cudaStream_t s) {
    dot_kernel<<<reduce_blocks(n), kT, 0, s>>>(a, b, n, out, scratch, counter);
}

void launch_axpy_dot(double* w, const double* vi, const double* h, const double* vnext, int n, double* out,
                     double* scratch, unsigned* counter, cudaStream_t s) {
    axpy_dot_kernel<<<reduce_blocks(n), kT, 0, s>>>(w, vi, h, vnext, n, out, scratch, counter);
}

void launch_seq_dot(const double* a, const double* b, int n, double* out, cudaStream_t s) {
    seq_dot2_kernel<<<1, kSeqT, 0, s>>>(a, b, nullptr, nullptr, n, out, nullptr);
}

void launch_seq_axpy_dot(double* w, const double* vi, const double* h, const double* vnext, int n, double* out,
                         cudaStream_t s) {
    axpy_neg_dev_kernel<<<grid_for(n), 256, 0, s>>>(w, vi, h, n);
    seq_dot2_kernel<<<1, kSeqT, 0, s>>>(w, vnext ? vnext : w, nullptr, nullptr, n, out, nullptr);
}

void launch_seq_eps(const double* u, const double* v, int n, double* sums, double* eps_out, double* u_norm,
                    bool cached, cudaStream_t s) {
    seq_dot2_kernel<<<1, kSeqT, 0, s>>>(v, v, cached ? nullptr : u, cached ? nullptr : u, n, sums, sums + 1);
    seq_eps_finish_kernel<<<1, 1, 0, s>>>(sums, eps_out, u_norm, cached);
}

int arnoldi_fused_grid(int n, int* chunk_out) {
    static int sms = 0, max_smem = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cudaFuncSetAttribute(arnoldi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem - 1024);
    }
    const long long chunk = (static_cast<long long>(n) + sms - 1) / sms;
    if (chunk * 8 > max_smem - 1024 || chunk > static_cast<long long>(kAT) * kAK) return 0;  // w must fit on chip
    *chunk_out = static_cast<int>(chunk);
    return sms;
}

bool launch_arnoldi_fused(const double* w, const double* V, int n, int j, double* h, double* partial, double* vnext,
                          cudaStream_t s) {
    int chunk = 0;
    const int grid = arnoldi_fused_grid(n, &chunk);
    if (!grid) return false;
    const int* jdev = nullptr;
    int vcap = 0;
    void* args[] = {&w, &V, &n, &j, &chunk, &h, &partial, &vnext, &jdev, &vcap};
    if (cudaLaunchCooperativeKernel(reinterpret_cast<void*>(arnoldi_kernel), dim3(grid), dim3(kAT), args,
                                    static_cast<size_t>(chunk) * 8, s) == cudaSuccess)
        return true;
    cudaGetLastError();  // a refused cooperative launch is not sticky: clear it so the unfused MGS runs
    return false;
}

bool launch_arnoldi_fused_dev(const double* w, const double* V, int n, const int* jdev, int vcap, double* h,
                              double* partial, cudaStream_t s) {
    int chunk = 0;
    const int grid = arnoldi_fused_grid(n, &chunk);
    if (!grid) return false;
    int j = 0;
    double* vnext = nullptr;
    void* args[] = {&w, &V, &n, &j, &chunk, &h, &partial, &vnext, &jdev, &vcap};
    if (cudaLaunchCooperativeKernel(reinterpret_cast<void*>(arnoldi_kernel), dim3(grid), dim3(kAT), args,
                                    static_cast<size_t>(chunk) * 8, s) == cudaSuccess)
        return true;
    cudaGetLastError();
    return false;
}

void launch_givens(const GmresDev& st, const double* h, const ErrWords* err, cudaGraphConditionalHandle cond,
                   cudaStream_t s) {
    givens_kernel<<<1, 1, 0, s>>>(st, h, err, cond);
}

void launch_scale_div(const double* in, const double* divisor, double* out, int n, cudaStream_t s) {
    scale_div_kernel<<<grid_for(n), 256, 0, s>>>(in, divisor, 0.0, out, n);
}

void launch_scale_div_host(const double* in, double divisor, double* out, int n, cudaStream_t s) {
    scale_div_kernel<<<grid_for(n), 256, 0, s>>>(in, nullptr, divisor, out, n);
}

void launch_update(double* x, const double* V, const double* y, int j, int n, cudaStream_t s) {
    update_kernel<<<grid_for(n), 256, sizeof(double) * (j > 0 ? j : 1), s>>>(x, nullptr, V, y, j, n);
}

void launch_basis_combination(double* dx, const double* V, const double* y, int j, int n, cudaStream_t s) {
    update_kernel<<<grid_for(n), 256, sizeof(double) * (j > 0 ? j : 1), s>>>(nullptr, dx, V, y, j, n);
}

void launch_sub_from(const double* b, double* r, int n, cudaStream_t s) {
    sub_from_kernel<<<grid_for(n), 256, 0, s>>>(b, r, n);
}

void launch_negate(const double* a, double* out, int n, cudaStream_t s) {
    negate_kernel<<<grid_for(n), 256, 0, s>>>(a, out, n);
}

void launch_axpy_host(double* y, double alpha, const double* x, int n, cudaStream_t s) {
    axpy_kernel<<<grid_for(n), 256, 0, s>>>(y, alpha, x, n);
}

void launch_lincomb(double* out, const double* u, double s, const double* du, int n, cudaStream_t st) {
    lincomb_kernel<<<grid_for(n), 256, 0, st>>>(out, u, s, du, n);
}

void launch_bdf2_rotate(double* uo, double* uoo, double* vo, double* voo, double* ao, const double* u, double dt,
                        int n, cudaStream_t s) {
    bdf2_rotate_kernel<<<grid_for(n), 256, 0, s>>>(uo, uoo, vo, voo, ao, u, dt, n);
}

void launch_predict(double* u, const double* uo, const double* vo, const double* ao, double dt, int n,
                    cudaStream_t s) {
    predict_kernel<<<grid_for(n), 256, 0, s>>>(u, uo, vo, ao, dt, n);
}

}  // namespace sfv
