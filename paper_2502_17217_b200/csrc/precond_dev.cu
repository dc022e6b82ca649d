// precond_dev.cu — the ILU(0)/ILU(1) preconditioner set up on the device.
//
// Everything make_preconditioner builds for the default streamed sweep, without a host round
// trip of the matrix:
//   1. J~ = assemble_approximate_jacobian (/root/reference/proj/src/discretisation.cpp:216-262)
//      on the cell graph (c I blocks, SURVEY.md finding 4): one thread per row, the row's
//      entries accumulated over the cell's faces in ascending face order — every entry sees
//      the reference's face-by-face additions in the same order (precond_host.cpp
//      cell_jacobian is the host twin);
//   2. the ILU(k <= 1) pattern (IlukPrecond ctor, linalg.cpp:251-282): for k <= 1 a fill entry
//      (i, j) arises from level-0 entries (i, k), (k, j) alone, so rows are independent;
//   3. the levels of both sweeps (longest dependency chains, linalg.cpp:302-316) by a
//      sync-free pass over rows claimed in sweep order (co-resident grid, release/acquire);
//   4. the IKJ numeric phase (linalg.cpp:283-299): ilu_numeric_kernel of precond.cu, rows in
//      level order — the factor is bit-identical to the host's and the reference's;
//   5. positions (rows grouped by level, ascending row within a level, levels padded to 32),
//      the U -> L position map, and the streamed sweep's 112-byte records with the DSMEM
//      owner / ring slot of every dependency (build_stream_records' layout and its ring check).
// Position order does not change any result: a row's arithmetic is fixed by its entries.
// Returns "" or the reason the caller falls back to the host setup (symmetry patches couple
// components, a row too long for the on-chip lists, more than 8 dependencies, no admissible
// ring, a zero pivot — the host path owns the reference's shifted retry).
#include <algorithm>
#include <cstdio>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "device.h"
#include "precond_dev.h"
#include "sfv_case.h"

namespace sfv {
namespace {

constexpr int kMaxRow = 64;  // entries of one ILU row held in a thread's local list

__device__ __forceinline__ int ld_acq(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---- 1. J~ pattern and values
__global__ void jac_count_kernel(DevTopoView t, int* __restrict__ len, int* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= t.nc) return;
    int k = 1;
    for (int q = t.cf_off[i]; q < t.cf_off[i + 1]; ++q) {
        const int f = t.cf[q];
        if (f < t.nint) ++k;
        else if (t.face_kind[f] == SFV_PATCH_SYMMETRY) atomicOr(flags, 1);
    }
    if (k > kMaxRow) atomicOr(flags, 2);
    len[i] = k;
}

__global__ void jac_fill_kernel(DevTopoView t, double kbar, bool transient, double rho, double dt,
                                const int* __restrict__ rp, int* __restrict__ col, double* __restrict__ val) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= t.nc) return;
    int c[kMaxRow];
    double v[kMaxRow];
    int m = 0;
    c[m++] = i;
    for (int q = t.cf_off[i]; q < t.cf_off[i + 1]; ++q) {
        const int f = t.cf[q];
        if (f < t.nint) c[m++] = t.owner[f] == i ? t.neigh[f] : t.owner[f];
    }
    for (int a = 1; a < m; ++a) {  // ascending columns (discretisation.cpp:223-236)
        const int x = c[a];
        int b = a - 1;
        while (b >= 0 && c[b] > x) {
            c[b + 1] = c[b];
            --b;
        }
        c[b + 1] = x;
    }
    for (int a = 0; a < m; ++a) v[a] = 0.0;
    auto find = [&](int j) {  // first entry of column j (the host's lower_bound)
        int a = 0;
        while (c[a] < j) ++a;
        return a;
    };
    const int di = find(i);
    for (int q = t.cf_off[i]; q < t.cf_off[i + 1]; ++q) {
        const int f = t.cf[q];
        // alpha is unity in the matrix (discretisation.cpp:239-240)
        const double coeff = kbar * t.delmag[f] / t.dmag[f] * t.amag[f];
        if (f < t.nint) {
            const int o = t.owner[f] == i ? t.neigh[f] : t.owner[f];
            v[find(o)] += coeff * 1.0;
            v[di] += -coeff * 1.0;
        } else if (t.face_kind[f] == SFV_PATCH_DISPLACEMENT) {
            v[di] += -coeff * 1.0;
        }
    }
    if (transient) v[di] += (-2.25 * rho * t.vol[i] / (dt * dt)) * 1.0;
    for (int a = 0; a < m; ++a) {
        col[rp[i] + a] = c[a];
        val[rp[i] + a] = v[a];
    }
}

// ---- 2. ILU(k <= 1) pattern: A(i) plus, for level 1, every j > k of an original row k < i of
// row i's original entries (iluk_factor_parallel's symbolic phase)
template <bool FILL>
__device__ __forceinline__ int ilu_row(int i, int level, const int* __restrict__ arp, const int* __restrict__ acol,
                                       int* c) {
    int m = 0;
    for (int p = arp[i]; p < arp[i + 1]; ++p) c[m++] = acol[p];
    const int orig = m;
    if (level >= 1)
        for (int x = 0; x < orig && c[x] < i; ++x) {
            const int k = c[x];
            for (int q = arp[k]; q < arp[k + 1]; ++q) {
                const int j = acol[q];
                if (j <= k) continue;
                bool have = false;
                for (int y = 0; y < m; ++y) have |= c[y] == j;
                if (have) continue;
                if (m == kMaxRow) return -1;
                c[m++] = j;
            }
        }
    if (FILL && m > orig)
        for (int a = 1; a < m; ++a) {
            const int x = c[a];
            int b = a - 1;
            while (b >= 0 && c[b] > x) {
                c[b + 1] = c[b];
                --b;
            }
            c[b + 1] = x;
        }
    return m;
}

__global__ void ilu_count_kernel(int n, int level, const int* __restrict__ arp, const int* __restrict__ acol,
                                 int* __restrict__ len, int* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int c[kMaxRow];
    const int m = ilu_row<false>(i, level, arp, acol, c);
    if (m < 0) atomicOr(flags, 2);
    len[i] = m < 0 ? 0 : m;
}

__global__ void ilu_fill_kernel(int n, int level, const int* __restrict__ arp, const int* __restrict__ acol,
                                const double* __restrict__ aval, const int* __restrict__ rp, int* __restrict__ col,
                                double* __restrict__ val, int* __restrict__ diag,
                                unsigned long long* __restrict__ nnz_lu) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int c[kMaxRow];
    const int m = ilu_row<true>(i, level, arp, acol, c);
    const int b = rp[i];
    int lo = 0, d = -1;
    for (int a = 0; a < m; ++a) {
        col[b + a] = c[a];
        val[b + a] = 0.0;  // fill entries start at 0
        if (c[a] < i) ++lo;
        if (c[a] == i) d = b + a;
    }
    // A at the pattern positions (both rows ascending)
    int a = 0;
    for (int p = arp[i]; p < arp[i + 1]; ++p) {
        while (c[a] < acol[p]) ++a;
        val[b + a] = aval[p];
    }
    diag[i] = d;
    atomicAdd(nnz_lu, static_cast<unsigned long long>(lo));
    atomicAdd(nnz_lu + 1, static_cast<unsigned long long>(m - lo - (d >= 0 ? 1 : 0)));
}

// ---- 3. sweep levels, sync-free: rows claimed in sweep order; a row waits only on rows
// claimed before it (the grid is co-resident: cooperative launch)
template <bool UPPER>
__global__ void level_kernel(int n, const int* __restrict__ rp, const int* __restrict__ col, int* lev, int* ticket,
                             int* maxlev) {
    int top = 0;
    while (true) {
        int x = 0;
        x = atomicAdd(ticket, 1);
        if (x >= n) break;
        const int i = UPPER ? n - 1 - x : x;
        int l = 0;
        if (UPPER) {
            for (int p = rp[i + 1] - 1; p >= rp[i] && col[p] > i; --p) {
                int v;
                while ((v = ld_acq(lev + col[p])) < 0) __nanosleep(64);  // back off: the polls share L2
                l = max(l, v + 1);
            }
        } else {
            for (int p = rp[i]; p < rp[i + 1] && col[p] < i; ++p) {
                int v;
                while ((v = ld_acq(lev + col[p])) < 0) __nanosleep(64);
                l = max(l, v + 1);
            }
        }
        st_rel(lev + i, l);
        top = max(top, l);
    }
    atomicMax(maxlev, top);
}

__global__ void count_levels_kernel(int n, const int* __restrict__ lev, int* __restrict__ cnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) atomicAdd(cnt + lev[i], 1);
}

__global__ void iota_kernel(int n, int* __restrict__ a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = i;
}

// sorted (level, row) pairs -> order[position] = row, pos[row] = position
__global__ void place_kernel(int n, const int* __restrict__ slev, const int* __restrict__ srow,
                             const int* __restrict__ ucum, const int* __restrict__ lptr, int* __restrict__ order,
                             int* __restrict__ pos) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= n) return;
    const int l = slev[x];
    const int p = lptr[l] + (x - ucum[l]);
    order[p] = srow[x];
    pos[srow[x]] = p;
}

__global__ void u2l_kernel(int np, const int* __restrict__ uorder, const int* __restrict__ lpos, int* __restrict__ u2l) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < np) u2l[p] = uorder[p] >= 0 ? lpos[uorder[p]] : -1;
}

// ---- 5. streamed-sweep records.  Level l's positions are cut into cs chunk-aligned slices
// (CTA r owns [la + r per 32, ...)); a CTA's ordinal counts its positions over all levels;
// cum[r * (nl + 1) + l] = positions CTA r owns in levels < l.
struct Slicing {
    int np, nl, cs, ring;
    const int* lptr;
    const int* cum;
};
__device__ __forceinline__ int level_of(const Slicing& s, int p) {
    int lo = 0, hi = s.nl;  // largest l with lptr[l] <= p
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s.lptr[mid] <= p) lo = mid;
        else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ void owner_ordinal(const Slicing& s, int p, int l, int& r, int& ord) {
    const int la = s.lptr[l], lb = s.lptr[l + 1];
    const int nch = (lb - la) >> 5, per = max(1, (nch + s.cs - 1) / s.cs);
    r = ((p - la) >> 5) / per;
    ord = s.cum[r * (s.nl + 1) + l] + (p - (la + r * per * 32));
}

// the dependencies of position p (a row's entries in the reference's subtraction order)
template <bool UPPER>
__device__ __forceinline__ int row_deps(int i, const int* __restrict__ rp, const int* __restrict__ col, int* dq,
                                        int* dk, int& dpos) {
    int m = 0;
    dpos = -1;
    if (UPPER) {
        for (int p = rp[i + 1] - 1; p >= rp[i] && col[p] >= i; --p) {
            if (col[p] == i) {
                dpos = p;
            } else {
                if (m < 8) {
                    dq[m] = col[p];
                    dk[m] = p;
                }
                ++m;
            }
        }
    } else {
        for (int p = rp[i]; p < rp[i + 1] && col[p] < i; ++p) {
            if (m < 8) {
                dq[m] = col[p];
                dk[m] = p;
            }
            ++m;
        }
    }
    return m;
}

// pass 1: the smallest ring with no slot rewritten before its last reader, and the row width
template <bool UPPER>
__global__ void ring_need_kernel(Slicing s, const int* __restrict__ order, const int* __restrict__ pos,
                                 const int* __restrict__ rp, const int* __restrict__ col, int* need, int* wide) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= s.np) return;
    const int i = order[p];
    if (i < 0) return;
    int dq[8], dk[8], dpos;
    const int m = row_deps<UPPER>(i, rp, col, dq, dk, dpos);
    if (m > 8) {
        atomicOr(wide, 1);
        return;
    }
    const int l = level_of(s, p);
    int req = 0;
    for (int k = 0; k < m; ++k) {
        const int q = pos[dq[k]];
        int r, o;
        owner_ordinal(s, q, level_of(s, q), r, o);
        // the slot of q is rewritten by r's (o + ring)-th position: it must lie after level l
        req = max(req, s.cum[r * (s.nl + 1) + l + 1] - o);
    }
    atomicMax(need, req);
}

// pass 2: the records in the device chunk layout (device.h kStream*: val[8][32], diag[32],
// dep[8][32], own[32], out[32], zero tail; 3584 bytes per 32 positions)
// out (kOffOut): the forward sweep stores each value at its row's backward-sweep position
// (out_pos), the backward sweep at its row
template <bool UPPER>
__global__ void records_kernel(Slicing s, const int* __restrict__ order, const int* __restrict__ pos,
                               const int* __restrict__ rp, const int* __restrict__ col, const double* __restrict__ val,
                               const int* __restrict__ out_pos, unsigned char* __restrict__ rec) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const int nchunk = (s.np + 31) / 32;
    if (p >= nchunk * 32) return;
    unsigned char* cb = rec + static_cast<size_t>(p >> 5) * kStreamChunk;
    double* cval = reinterpret_cast<double*>(cb);
    double* cdiag = reinterpret_cast<double*>(cb + kStreamOffDiag);
    uint32_t* cdep = reinterpret_cast<uint32_t*>(cb + kStreamOffDep);
    uint16_t* cown = reinterpret_cast<uint16_t*>(cb + kStreamOffOwn);
    int* cout = reinterpret_cast<int*>(cb + kStreamOffOut);
    const int ln = p & 31;
    if (ln < (kStreamChunk - kStreamOffEnd) / 8) reinterpret_cast<uint64_t*>(cb + kStreamOffEnd)[ln] = 0ull;
    int r = 0, o = 0, l = 0;
    if (p < s.np) {
        l = level_of(s, p);
        owner_ordinal(s, p, l, r, o);
    }
    for (int k = 0; k < 8; ++k) {
        cval[k * 32 + ln] = 0.0;
        cdep[k * 32 + ln] = stream_dep(r, s.ring);  // absent: the reader's +0.0 slot
    }
    if (p >= s.np) {  // tail of the last chunk
        cdiag[ln] = 0.0;
        cown[ln] = 0;
        cout[ln] = -1;
        return;
    }
    cown[ln] = static_cast<uint16_t>(o % s.ring);
    cdiag[ln] = 1.0;
    const int i = order[p];
    cout[ln] = i < 0 ? -1 : out_pos ? out_pos[i] : i;
    if (i < 0) return;  // level padding: no dependencies, unit pivot
    int dq[8], dk[8], dpos;
    const int m = row_deps<UPPER>(i, rp, col, dq, dk, dpos);
    if (UPPER) cdiag[ln] = dpos >= 0 ? val[dpos] : 0.0;
    for (int k = 0; k < m; ++k) {
        const int q = pos[dq[k]];
        int rq, oq;
        owner_ordinal(s, q, level_of(s, q), rq, oq);
        cdep[k * 32 + ln] = stream_dep(rq, oq % s.ring);
        cval[k * 32 + ln] = val[dk[k]];
    }
}

struct Tmp {  // scratch freed at scope exit
    std::vector<void*> v;
    template <class T>
    T* get(size_t n) {
        void* p = nullptr;
        if (cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(T)) != cudaSuccess) return nullptr;
        v.push_back(p);
        return static_cast<T*>(p);
    }
    ~Tmp() {
        for (void* p : v) cudaFree(p);
    }
};

template <class T>
T* keep_alloc(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(T)) != cudaSuccess) return nullptr;
    return static_cast<T*>(p);
}

int exclusive_scan(Tmp& tmp, const int* in, int* out, int n, cudaStream_t s) {  // returns the total
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n + 1, s);
    void* w = tmp.get<unsigned char>(bytes);
    if (!w) return -1;
    cub::DeviceScan::ExclusiveSum(w, bytes, in, out, n + 1, s);
    int tot = 0;
    cudaMemcpyAsync(&tot, out + n, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    return tot;
}

int coop_grid(const void* kern, int block) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, block, 0);
    return std::max(1, sms * std::max(1, per));
}

// one sweep's schedule: levels, positions and order / pos maps
template <bool UPPER>
std::string sweep_schedule(Tmp& tmp, int n, const int* rp, const int* col, int cs, cudaStream_t s, DevSweep& out,
                           std::vector<int>& lptr_h, int** pos_out, int** sorted_rows) {
    int* lev = tmp.get<int>(n);
    int* misc = tmp.get<int>(2);  // ticket, max level
    if (!lev || !misc) return "device ilu: out of memory";
    cudaMemsetAsync(lev, 0xff, sizeof(int) * n, s);
    cudaMemsetAsync(misc, 0, sizeof(int) * 2, s);
    {
        auto kern = level_kernel<UPPER>;
        const int grid = coop_grid(reinterpret_cast<const void*>(kern), 256);
        int nn = n;
        int* ticket = misc;
        int* maxl = misc + 1;
        void* args[] = {&nn, const_cast<int**>(&rp), const_cast<int**>(&col), &lev, &ticket, &maxl};
        if (cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(std::min(grid, (n + 255) / 256)), dim3(256),
                                        args, 0, s) != cudaSuccess) {
            cudaGetLastError();
            return "device ilu: level pass refused";
        }
    }
    int top = 0;
    cudaMemcpyAsync(&top, misc + 1, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const int nl = top + 1;
    int* cnt = tmp.get<int>(nl + 1);
    int* ucum = tmp.get<int>(nl + 1);
    if (!cnt || !ucum) return "device ilu: out of memory";
    cudaMemsetAsync(cnt, 0, sizeof(int) * (nl + 1), s);
    count_levels_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, lev, cnt);
    std::vector<int> cnt_h(nl);
    cudaMemcpyAsync(cnt_h.data(), cnt, sizeof(int) * nl, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    lptr_h.assign(nl + 1, 0);
    std::vector<int> ucum_h(nl + 1, 0);
    for (int l = 0; l < nl; ++l) {
        lptr_h[l + 1] = lptr_h[l] + (cnt_h[l] + 31) / 32 * 32;
        ucum_h[l + 1] = ucum_h[l] + cnt_h[l];
    }
    const int np = lptr_h[nl];
    // rows sorted by (level, row): a stable radix sort of the levels over the row indices
    int* rows = tmp.get<int>(n);
    int* srows = keep_alloc<int>(n);
    int* slev = tmp.get<int>(n);
    int* lptr = keep_alloc<int>(nl + 1);
    int* order = keep_alloc<int>(np);
    int* pos = tmp.get<int>(n);
    if (!rows || !srows || !slev || !lptr || !order || !pos) {
        cudaFree(srows);
        cudaFree(lptr);
        cudaFree(order);
        return "device ilu: out of memory";
    }
    iota_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, rows);
    int bits = 1;
    while ((1 << bits) <= top) ++bits;
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, lev, slev, rows, srows, n, 0, bits, s);
    void* w = tmp.get<unsigned char>(bytes);
    if (!w) {
        cudaFree(srows);
        cudaFree(lptr);
        cudaFree(order);
        return "device ilu: out of memory";
    }
    cub::DeviceRadixSort::SortPairs(w, bytes, lev, slev, rows, srows, n, 0, bits, s);
    cudaMemcpyAsync(lptr, lptr_h.data(), sizeof(int) * (nl + 1), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(ucum, ucum_h.data(), sizeof(int) * (nl + 1), cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(order, 0xff, sizeof(int) * np, s);
    place_kernel<<<(n + 255) / 256, 256, 0, s>>>(n, slev, srows, ucum, lptr, order, pos);
    cudaStreamSynchronize(s);  // lptr_h / ucum_h are host locals
    out.n_pos = np;
    out.n_levels = nl;
    out.order = order;
    out.level_ptr = lptr;
    *pos_out = pos;
    if (sorted_rows) *sorted_rows = srows;
    else cudaFree(srows);
    (void)cs;
    return "";
}

// cum[r][l] of the slicing on the host (nl x cs ints)
std::vector<int> slice_cum(const std::vector<int>& lptr, int cs) {
    const int nl = static_cast<int>(lptr.size()) - 1;
    std::vector<int> cum(static_cast<size_t>(cs) * (nl + 1), 0);
    for (int l = 0; l < nl; ++l) {
        const int la = lptr[l], lb = lptr[l + 1];
        const int nch = (lb - la) / 32, per = std::max(1, (nch + cs - 1) / cs);
        for (int r = 0; r < cs; ++r) {
            const int a = std::min(lb, la + r * per * 32), b = std::min(lb, a + per * 32);
            cum[static_cast<size_t>(r) * (nl + 1) + l + 1] = cum[static_cast<size_t>(r) * (nl + 1) + l] + (b - a);
        }
    }
    return cum;
}

}  // namespace

void DevSweep::release() {
    cudaFree(order);
    cudaFree(level_ptr);
    cudaFree(rec);
    cudaFree(u2l);
    order = level_ptr = u2l = nullptr;
    rec = nullptr;
}

std::string device_ilu_setup(const DevTopoView& t, double kbar, bool transient, double rho, double dt, int level,
                             cudaStream_t s, DevIluSetup& out, double* timing) {
    auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](int k) {
        if (!timing) return;
        cudaStreamSynchronize(s);
        const auto n = std::chrono::steady_clock::now();
        timing[k] = std::chrono::duration<double, std::milli>(n - t0).count();
        t0 = n;
    };
    const int n = t.nc;
    const int cs = kStreamCluster;
    if (level > 1) return "device ilu: level > 1";
    Tmp tmp;
    int* flags = tmp.get<int>(2);
    int* alen = tmp.get<int>(n + 1);
    int* arp = tmp.get<int>(n + 1);
    if (!flags || !alen || !arp) return "device ilu: out of memory";
    cudaMemsetAsync(flags, 0, sizeof(int) * 2, s);
    cudaMemsetAsync(alen + n, 0, sizeof(int), s);
    const int g = (n + 255) / 256;
    // 1. J~
    jac_count_kernel<<<g, 256, 0, s>>>(t, alen, flags);
    const int annz = exclusive_scan(tmp, alen, arp, n, s);
    int fl = 0;
    cudaMemcpy(&fl, flags, sizeof(int), cudaMemcpyDeviceToHost);
    if (fl & 1) return "device ilu: symmetry patches (diagonal blocks per component)";
    if (fl & 2 || annz < 0) return "device ilu: row too long";
    int* acol = tmp.get<int>(annz);
    double* aval = tmp.get<double>(annz);
    if (!acol || !aval) return "device ilu: out of memory";
    jac_fill_kernel<<<g, 256, 0, s>>>(t, kbar, transient, rho, dt, arp, acol, aval);
    mark(0);
    // 2. ILU(k) pattern with A at its positions
    int* len = tmp.get<int>(n + 1);
    int* rp = tmp.get<int>(n + 1);
    if (!len || !rp) return "device ilu: out of memory";
    cudaMemsetAsync(len + n, 0, sizeof(int), s);
    ilu_count_kernel<<<g, 256, 0, s>>>(n, level, arp, acol, len, flags);
    const int nnz = exclusive_scan(tmp, len, rp, n, s);
    cudaMemcpy(&fl, flags, sizeof(int), cudaMemcpyDeviceToHost);
    if (fl & 2 || nnz < 0) return "device ilu: row too long";
    int* col = tmp.get<int>(nnz);
    double* val = tmp.get<double>(nnz);
    int* diag = tmp.get<int>(n);
    unsigned long long* nnz_lu = tmp.get<unsigned long long>(2);
    if (!col || !val || !diag || !nnz_lu) return "device ilu: out of memory";
    cudaMemsetAsync(nnz_lu, 0, 2 * sizeof(unsigned long long), s);
    ilu_fill_kernel<<<g, 256, 0, s>>>(n, level, arp, acol, aval, rp, col, val, diag, nnz_lu);
    unsigned long long nlu[2] = {0, 0};
    cudaMemcpyAsync(nlu, nnz_lu, sizeof nlu, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    out.nnz_L = static_cast<long long>(nlu[0]);
    out.nnz_U = static_cast<long long>(nlu[1]);
    mark(1);
    // 3. both sweeps' levels and positions
    std::vector<int> lptr_l, lptr_u;
    int *lpos = nullptr, *upos = nullptr, *lrows = nullptr;
    out.release();
    if (std::string e = sweep_schedule<false>(tmp, n, rp, col, cs, s, out.L, lptr_l, &lpos, &lrows); !e.empty())
        return e;
    tmp.v.push_back(lrows);  // freed with the scratch
    if (std::string e = sweep_schedule<true>(tmp, n, rp, col, cs, s, out.U, lptr_u, &upos, nullptr); !e.empty()) {
        out.release();
        return e;
    }
    mark(2);
    // 4. numeric phase, rows in lower-sweep level order (bit-identical IKJ)
    if (!launch_ilu_numeric(n, lrows, rp, col, diag, val, s)) {
        out.release();
        return "device ilu: zero pivot";
    }
    mark(3);
    // 5. U -> L map and the records of both sweeps
    out.U.u2l = keep_alloc<int>(out.U.n_pos);
    if (!out.U.u2l) {
        out.release();
        return "device ilu: out of memory";
    }
    u2l_kernel<<<(out.U.n_pos + 255) / 256, 256, 0, s>>>(out.U.n_pos, out.U.order, lpos, out.U.u2l);
    int rows_l = 32, rows_u = 32;
    for (auto* lp : {&lptr_l, &lptr_u})
        for (size_t l = 0; l + 1 < lp->size(); ++l) {
            const int nch = ((*lp)[l + 1] - (*lp)[l]) / 32;
            (lp == &lptr_l ? rows_l : rows_u) =
                std::max(lp == &lptr_l ? rows_l : rows_u, (nch + cs - 1) / cs * 32);
        }
    out.max_rows = std::max(rows_l, rows_u);
    if (out.max_rows > kStreamMaxRows) {
        out.release();
        return "device ilu: level slice wider than the streamed sweep's stage";
    }
    const std::vector<int> cum_l = slice_cum(lptr_l, cs), cum_u = slice_cum(lptr_u, cs);
    int* dcum = tmp.get<int>(cum_l.size() + cum_u.size());
    int* need = tmp.get<int>(2);
    if (!dcum || !need) {
        out.release();
        return "device ilu: out of memory";
    }
    cudaMemcpyAsync(dcum, cum_l.data(), sizeof(int) * cum_l.size(), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(dcum + cum_l.size(), cum_u.data(), sizeof(int) * cum_u.size(), cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(need, 0, sizeof(int) * 2, s);
    Slicing sl{out.L.n_pos, out.L.n_levels, cs, 0, out.L.level_ptr, dcum};
    Slicing su{out.U.n_pos, out.U.n_levels, cs, 0, out.U.level_ptr, dcum + cum_l.size()};
    ring_need_kernel<false><<<(sl.np + 255) / 256, 256, 0, s>>>(sl, out.L.order, lpos, rp, col, need, need + 1);
    ring_need_kernel<true><<<(su.np + 255) / 256, 256, 0, s>>>(su, out.U.order, upos, rp, col, need, need + 1);
    int nh[2] = {0, 0};
    cudaMemcpyAsync(nh, need, sizeof nh, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (nh[1]) {
        out.release();
        return "device ilu: a row has more than 8 dependencies";
    }
    out.ring = 0;
    for (int cand : {1024, 2048, 3072, 4095})  // (the +0.0 slot is slot index `ring`, 12 bits)
        if (cand >= nh[0]) {
            out.ring = cand;
            break;
        }
    if (!out.ring) {
        out.release();
        return "device ilu: no admissible value ring";
    }
    sl.ring = su.ring = out.ring;
    for (int w = 0; w < 2; ++w) {
        DevSweep& sw = w ? out.U : out.L;
        const size_t nchunk = (static_cast<size_t>(sw.n_pos) + 31) / 32;
        sw.rec = keep_alloc<unsigned char>(nchunk * kStreamChunk);
        if (!sw.rec) {
            out.release();
            return "device ilu: out of memory";
        }
        const int gp = static_cast<int>((nchunk * 32 + 255) / 256);
        if (w) records_kernel<true><<<gp, 256, 0, s>>>(su, out.U.order, upos, rp, col, val, nullptr, sw.rec);
        else records_kernel<false><<<gp, 256, 0, s>>>(sl, out.L.order, lpos, rp, col, val, upos, sw.rec);
    }
    if (cudaStreamSynchronize(s) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        out.release();
        return "device ilu: cuda error";
    }
    mark(4);
    return "";
}

}  // namespace sfv
