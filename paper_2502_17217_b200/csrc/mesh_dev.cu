// mesh_dev.cu — the config-5 tet mesh built on the device.
//
// The same mesh as host_mesh.cpp kuhn_tets, array for array: points, the six-tet parity-mirrored
// Kuhn split, faces found by sorting the 4 nt triangle keys (stable radix sorts reproduce the
// host's (k1, c, tag) order), internal / boundary pairing, the cell renumbering (the seeded
// Fisher-Yates permutation, a sequential chain of swaps, stays on the host), reverse
// Cuthill-McKee on the device, face orientation, and the two final face sorts.
//
// RCM (host rcm()): a breadth-first order is reproduced level by level — a node enters the
// next level from its first-ordered neighbour in the current level (its parent), and the
// level is ordered by (parent position, node id) for the pseudo-peripheral passes, or by
// (parent position, degree, id) for Cuthill-McKee (the host's stable sort by degree of each
// parent's unseen neighbours, whose adjacency lists are ascending).  Only a connected cell
// graph is handled here; otherwise the caller builds the mesh on the host.
#include <algorithm>
#include <climits>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "host_mesh.h"

namespace sfv {
namespace {

template <class T>
struct DBuf {  // device buffer freed at scope exit
    T* p = nullptr;
    size_t n = 0;
    bool alloc(size_t k) {
        n = k;
        return cudaMalloc(&p, std::max<size_t>(1, k) * sizeof(T)) == cudaSuccess;
    }
    ~DBuf() {
        if (p) cudaFree(p);
    }
};

__global__ void points_kernel(int n, double e0, double e1, double e2, double* __restrict__ pts) {
    const int np1 = n + 1;
    const long long np = static_cast<long long>(np1) * np1 * np1;
    const long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (p >= np) return;
    const int i = static_cast<int>(p % np1), j = static_cast<int>((p / np1) % np1), k = static_cast<int>(p / np1 / np1);
    pts[3 * p] = e0 * i / n;
    pts[3 * p + 1] = e1 * j / n;
    pts[3 * p + 2] = e2 * k / n;
}

// tet vertices and the four triangle keys of every tet (host kuhn_tets, same vertex order)
__global__ void tets_kernel(int n, int* __restrict__ tv, unsigned long long* __restrict__ k1, unsigned* __restrict__ kc) {
    const int nt = 6 * n * n * n;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const int h = t / 6, pr = t % 6;
    const int i = h % n, j = (h / n) % n, k = h / n / n;
    const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    const int np1 = n + 1;
    int loc[3] = {0, 0, 0};
    const int base[3] = {i, j, k};
    int v[4];
    for (int s = 0; s < 4; ++s) {
        if (s > 0) loc[perms[pr][s - 1]] = 1;
        int g[3];
        for (int a = 0; a < 3; ++a) g[a] = base[a] + ((base[a] & 1) ? 1 - loc[a] : loc[a]);
        v[s] = g[0] + np1 * (g[1] + np1 * g[2]);
        tv[4 * t + s] = v[s];
    }
    for (int lf = 0; lf < 4; ++lf) {
        int p[3], q = 0;
        for (int s = 0; s < 4; ++s)
            if (s != lf) p[q++] = v[s];
        if (p[0] > p[1]) { const int x = p[0]; p[0] = p[1]; p[1] = x; }
        if (p[1] > p[2]) { const int x = p[1]; p[1] = p[2]; p[2] = x; }
        if (p[0] > p[1]) { const int x = p[0]; p[0] = p[1]; p[1] = x; }
        const size_t x = 4 * static_cast<size_t>(t) + lf;
        k1[x] = (static_cast<unsigned long long>(p[0]) << 32) | static_cast<unsigned>(p[1]);
        kc[x] = static_cast<unsigned>(p[2]);
    }
}

__global__ void iota_u32(size_t n, unsigned* __restrict__ a) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) a[i] = static_cast<unsigned>(i);
}
__global__ void gather_k1(size_t n, const unsigned* __restrict__ idx, const unsigned long long* __restrict__ k1,
                          unsigned long long* __restrict__ out) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = k1[idx[i]];
}

// sorted keys: x starts an internal pair (flag 1) or is a boundary triangle (flag 2)
__global__ void pair_flags(size_t n, const unsigned* __restrict__ tag, const unsigned long long* __restrict__ k1s,
                           const unsigned* __restrict__ kc, int* __restrict__ fi, int* __restrict__ fb) {
    const size_t x = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (x >= n) return;
    // k1s: the sorted first key words; kc by original triangle index
    auto same = [&](size_t a, size_t b) { return k1s[a] == k1s[b] && kc[tag[a]] == kc[tag[b]]; };
    const bool prev = x > 0 && same(x - 1, x), next = x + 1 < n && same(x, x + 1);
    // the host walk pairs x with x + 1 when equal; a conforming mesh has at most two equal keys
    fi[x] = next && !prev ? 1 : 0;
    fb[x] = !next && !prev ? 1 : 0;
}

__global__ void compact(size_t n, const int* __restrict__ flag, const int* __restrict__ at, unsigned* __restrict__ out) {
    const size_t x = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (x < n && flag[x]) out[at[x]] = static_cast<unsigned>(x);
}

// ---- cell graph (new ids) for RCM
__global__ void degree_kernel(int ni, const unsigned* __restrict__ ifx, const unsigned* __restrict__ tag,
                              const int* __restrict__ newid, int* __restrict__ deg) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= ni) return;
    const size_t x = ifx[f];
    atomicAdd(deg + newid[tag[x] / 4], 1);
    atomicAdd(deg + newid[tag[x + 1] / 4], 1);
}
__global__ void adj_fill(int ni, const unsigned* __restrict__ ifx, const unsigned* __restrict__ tag,
                         const int* __restrict__ newid, const int* __restrict__ off, int* __restrict__ fill,
                         int* __restrict__ adj) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= ni) return;
    const size_t x = ifx[f];
    const int a = newid[tag[x] / 4], b = newid[tag[x + 1] / 4];
    adj[off[a] + atomicAdd(fill + a, 1)] = b;
    adj[off[b] + atomicAdd(fill + b, 1)] = a;
}
__global__ void adj_sort(int n, const int* __restrict__ off, int* __restrict__ adj) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    for (int a = off[c] + 1; a < off[c + 1]; ++a) {
        const int x = adj[a];
        int b = a - 1;
        while (b >= off[c] && adj[b] > x) {
            adj[b + 1] = adj[b];
            --b;
        }
        adj[b + 1] = x;
    }
}

// BFS level step: parent[v] = first frontier position reaching v
__global__ void bfs_parent(int p0, int p1, const int* __restrict__ order, const int* __restrict__ off,
                           const int* __restrict__ adj, const int* __restrict__ vis, int* __restrict__ parent) {
    const int p = p0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= p1) return;
    const int u = order[p];
    for (int e = off[u]; e < off[u + 1]; ++e)
        if (!vis[adj[e]]) atomicMin(parent + adj[e], p);
}
template <bool CM>
__global__ void bfs_claim(int p0, int p1, const int* __restrict__ order, const int* __restrict__ off,
                          const int* __restrict__ adj, const int* __restrict__ vis, const int* __restrict__ parent,
                          int* __restrict__ cnt, unsigned long long* __restrict__ key, int* __restrict__ cand) {
    const int p = p0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= p1) return;
    const int u = order[p];
    for (int e = off[u]; e < off[u + 1]; ++e) {
        const int v = adj[e];
        if (vis[v] || parent[v] != p) continue;
        const int at = atomicAdd(cnt, 1);
        const unsigned long long d = CM ? static_cast<unsigned long long>(off[v + 1] - off[v]) : 0ull;
        key[at] = (static_cast<unsigned long long>(p) << 36) | (d << 30) | static_cast<unsigned long long>(v);
        cand[at] = v;
    }
}
__global__ void bfs_place(int p1, int m, const int* __restrict__ cand, int* __restrict__ order, int* __restrict__ vis) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= m) return;
    order[p1 + x] = cand[x];
    vis[cand[x]] = 1;
}
__global__ void set_one(int v, int* __restrict__ order, int* __restrict__ vis) {
    order[0] = v;
    vis[v] = 1;
}

// ---- output faces
struct OutF {
    int own, nei, a, b, c, patch;
};
__device__ __forceinline__ void lat(int p, int np1, int o[3]) {
    o[0] = p % np1;
    o[1] = (p / np1) % np1;
    o[2] = p / (np1 * np1);
}
__device__ __forceinline__ void orient(int np1, int& a, int& b, int& c, int d) {
    int pa[3], pb[3], pc[3], pd[3];
    lat(a, np1, pa), lat(b, np1, pb), lat(c, np1, pc), lat(d, np1, pd);
    long long e1[3], e2[3], e3[3];
    for (int s = 0; s < 3; ++s) {
        e1[s] = pb[s] - pa[s];
        e2[s] = pc[s] - pa[s];
        e3[s] = pd[s] - pa[s];
    }
    const long long nx = e1[1] * e2[2] - e1[2] * e2[1], ny = e1[2] * e2[0] - e1[0] * e2[2],
                    nz = e1[0] * e2[1] - e1[1] * e2[0];
    if (nx * e3[0] + ny * e3[1] + nz * e3[2] > 0) {
        const int t = b;
        b = c;
        c = t;
    }
    if (b < a && b < c) {
        const int t0 = a;
        a = b;
        b = c;
        c = t0;
    } else if (c < a && c < b) {
        const int t0 = c;
        c = b;
        b = a;
        a = t0;
    }
}
__global__ void internal_faces(int ni, int np1, const unsigned* __restrict__ ifx, const unsigned* __restrict__ tag,
                               const unsigned long long* __restrict__ k1s, const unsigned* __restrict__ kc,
                               const int* __restrict__ tv, const int* __restrict__ newid, OutF* __restrict__ out,
                               unsigned long long* __restrict__ key) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= ni) return;
    const size_t x = ifx[f];
    const unsigned long long k = k1s[x];
    int a = static_cast<int>(k >> 32), b = static_cast<int>(k & 0xffffffffu), c = static_cast<int>(kc[tag[x]]);
    int own = newid[tag[x] / 4], nei = newid[tag[x + 1] / 4];
    unsigned own_tag = tag[x];
    if (own > nei) {
        const int t = own;
        own = nei;
        nei = t;
        own_tag = tag[x + 1];
    }
    orient(np1, a, b, c, tv[4 * (own_tag / 4) + (own_tag % 4)]);
    out[f] = {own, nei, a, b, c, -1};
    key[f] = (static_cast<unsigned long long>(own) << 32) | static_cast<unsigned>(nei);
}
__global__ void boundary_faces(int nb, int n, const unsigned* __restrict__ bfx, const unsigned* __restrict__ tag,
                               const unsigned long long* __restrict__ k1s, const unsigned* __restrict__ kc,
                               const int* __restrict__ tv, const int* __restrict__ newid, OutF* __restrict__ out,
                               unsigned long long* __restrict__ key) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nb) return;
    const size_t x = bfx[f];
    const unsigned long long k = k1s[x];
    const int np1 = n + 1;
    int a = static_cast<int>(k >> 32), b = static_cast<int>(k & 0xffffffffu), c = static_cast<int>(kc[tag[x]]);
    int la[3], lb[3], lc[3];
    lat(a, np1, la), lat(b, np1, lb), lat(c, np1, lc);
    int side = -1;
    for (int ax = 0; ax < 3 && side < 0; ++ax) {
        if (la[ax] == 0 && lb[ax] == 0 && lc[ax] == 0) side = 2 * ax;
        else if (la[ax] == n && lb[ax] == n && lc[ax] == n) side = 2 * ax + 1;
    }
    const unsigned t = tag[x];
    orient(np1, a, b, c, tv[4 * (t / 4) + (t % 4)]);
    const int own = newid[t / 4];
    out[f] = {own, -1, a, b, c, side};
    // (patch, owner, a): 3 + 28 + 32 bits; unique (two faces of one tet are never coplanar)
    key[f] = (static_cast<unsigned long long>(side + 1) << 60) | (static_cast<unsigned long long>(own) << 32) |
             static_cast<unsigned>(a);
}
__global__ void apply_perm(int m, const int* __restrict__ idx, const OutF* __restrict__ in, OutF* __restrict__ out) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f < m) out[f] = in[idx[f]];
}
__global__ void iota_i32(int n, int* __restrict__ a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = i;
}

template <class K, class V>
bool sort_pairs(const K* kin, K* kout, const V* vin, V* vout, size_t n, int end_bit, cudaStream_t s = 0) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, n, 0, end_bit, s);
    DBuf<unsigned char> w;
    if (!w.alloc(bytes)) return false;
    return cub::DeviceRadixSort::SortPairs(w.p, bytes, kin, kout, vin, vout, n, 0, end_bit, s) == cudaSuccess;
}
bool exclusive_sum(const int* in, int* out, size_t n) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n);
    DBuf<unsigned char> w;
    if (!w.alloc(bytes)) return false;
    return cub::DeviceScan::ExclusiveSum(w.p, bytes, in, out, n) == cudaSuccess;
}
inline unsigned gblocks(size_t n) { return static_cast<unsigned>((n + 255) / 256); }

// one breadth-first order from `start` into order[0..], CM or plain; returns the count, and
// (plain) the host's pseudo-peripheral candidate: the first-ordered node of minimum degree in
// the deepest level
template <bool CM>
int bfs(int n, const int* off, const int* adj, int start, int* order, int* vis, int* parent, int* cnt,
        unsigned long long* key, unsigned long long* key2, int* cand, int* cand2, int* far_out,
        const std::vector<int>* offh = nullptr) {
    cudaMemset(vis, 0, sizeof(int) * n);
    cudaMemset(parent, 0x7f, sizeof(int) * n);
    set_one<<<1, 1>>>(start, order, vis);
    int p0 = 0, p1 = 1;
    while (true) {
        cudaMemset(cnt, 0, sizeof(int));
        bfs_parent<<<gblocks(p1 - p0), 256>>>(p0, p1, order, off, adj, vis, parent);
        bfs_claim<CM><<<gblocks(p1 - p0), 256>>>(p0, p1, order, off, adj, vis, parent, cnt, key, cand);
        int m = 0;
        cudaMemcpy(&m, cnt, sizeof(int), cudaMemcpyDeviceToHost);
        if (m == 0) break;
        if (!sort_pairs(key, key2, cand, cand2, m, 64)) return -1;
        bfs_place<<<gblocks(m), 256>>>(p1, m, cand2, order, vis);
        p0 = p1;
        p1 += m;
    }
    if (far_out) {  // deepest level [p0, p1): first node of minimum degree
        std::vector<int> lv(p1 - p0);
        cudaMemcpy(lv.data(), order + p0, sizeof(int) * (p1 - p0), cudaMemcpyDeviceToHost);
        int best = lv[0], bd = INT_MAX;
        for (int v : lv) {
            const int d = (*offh)[v + 1] - (*offh)[v];
            if (d < bd) {
                bd = d;
                best = v;
            }
        }
        *far_out = p1 - p0 == 1 && p0 == 0 ? start : best;
    }
    return p1;
}

}  // namespace

std::string device_kuhn_tets(const double ext[3], int n, const int kinds[6], const std::vector<int>* perm_newid,
                             bool do_rcm, HostMesh& m) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return "no device";
    }
    const int np1 = n + 1;
    const size_t npts = static_cast<size_t>(np1) * np1 * np1;
    const long long ntl = 6LL * n * n * n;
    if (ntl >= (1LL << 28) || npts >= (1ull << 31)) return "mesh too large for the device generator";
    const int nt = static_cast<int>(ntl);
    const size_t nk = 4 * static_cast<size_t>(nt);
    DBuf<double> pts;
    DBuf<int> tv;
    DBuf<unsigned long long> k1, k1s;
    DBuf<unsigned> kc, kcs, idx, tag;
    if (!pts.alloc(3 * npts) || !tv.alloc(4 * static_cast<size_t>(nt)) || !k1.alloc(nk) || !k1s.alloc(nk) ||
        !kc.alloc(nk) || !kcs.alloc(nk) || !idx.alloc(nk) || !tag.alloc(nk))
        return "device mesh: out of memory";
    points_kernel<<<gblocks(npts), 256>>>(n, ext[0], ext[1], ext[2], pts.p);
    tets_kernel<<<gblocks(nt), 256>>>(n, tv.p, k1.p, kc.p);
    // lexicographic (k1, c, tag): stable by c, then stable by k1 (tags start ascending)
    iota_u32<<<gblocks(nk), 256>>>(nk, idx.p);
    if (!sort_pairs(kc.p, kcs.p, idx.p, tag.p, nk, 32)) return "device mesh: sort failed";
    gather_k1<<<gblocks(nk), 256>>>(nk, tag.p, k1.p, k1s.p);
    if (!sort_pairs(k1s.p, k1.p, tag.p, idx.p, nk, 64)) return "device mesh: sort failed";
    // now k1 holds the sorted k1, idx the sorted tags
    std::swap(k1.p, k1s.p);  // k1s: sorted keys
    std::swap(idx.p, tag.p);  // tag: sorted tags
    DBuf<int> fi, fb, ai, ab;
    if (!fi.alloc(nk + 1) || !fb.alloc(nk + 1) || !ai.alloc(nk + 1) || !ab.alloc(nk + 1))
        return "device mesh: out of memory";
    pair_flags<<<gblocks(nk), 256>>>(nk, tag.p, k1s.p, kc.p, fi.p, fb.p);
    cudaMemset(fi.p + nk, 0, sizeof(int));
    cudaMemset(fb.p + nk, 0, sizeof(int));
    if (!exclusive_sum(fi.p, ai.p, nk + 1) || !exclusive_sum(fb.p, ab.p, nk + 1)) return "device mesh: scan failed";
    int ni = 0, nb = 0;
    cudaMemcpy(&ni, ai.p + nk, sizeof(int), cudaMemcpyDeviceToHost);
    cudaMemcpy(&nb, ab.p + nk, sizeof(int), cudaMemcpyDeviceToHost);
    DBuf<unsigned> ifx, bfx;
    if (!ifx.alloc(ni) || !bfx.alloc(nb)) return "device mesh: out of memory";
    compact<<<gblocks(nk), 256>>>(nk, fi.p, ai.p, ifx.p);
    compact<<<gblocks(nk), 256>>>(nk, fb.p, ab.p, bfx.p);
    // cell renumbering: the host's permutation, then RCM on the device
    DBuf<int> newid;
    if (!newid.alloc(nt)) return "device mesh: out of memory";
    if (perm_newid) cudaMemcpy(newid.p, perm_newid->data(), sizeof(int) * nt, cudaMemcpyHostToDevice);
    else iota_i32<<<gblocks(nt), 256>>>(nt, newid.p);
    if (do_rcm) {
        DBuf<int> deg, off, fill, adj, order, vis, parent, cnt, cand, cand2, pos;
        DBuf<unsigned long long> key, key2;
        if (!deg.alloc(nt + 1) || !off.alloc(nt + 1) || !fill.alloc(nt) || !adj.alloc(2 * static_cast<size_t>(ni)) ||
            !order.alloc(nt) || !vis.alloc(nt) || !parent.alloc(nt) || !cnt.alloc(1) || !cand.alloc(nt) ||
            !cand2.alloc(nt) || !key.alloc(nt) || !key2.alloc(nt) || !pos.alloc(nt))
            return "device mesh: out of memory";
        cudaMemset(deg.p, 0, sizeof(int) * (nt + 1));
        cudaMemset(fill.p, 0, sizeof(int) * nt);
        degree_kernel<<<gblocks(ni), 256>>>(ni, ifx.p, tag.p, newid.p, deg.p);
        if (!exclusive_sum(deg.p, off.p, nt + 1)) return "device mesh: scan failed";
        adj_fill<<<gblocks(ni), 256>>>(ni, ifx.p, tag.p, newid.p, off.p, fill.p, adj.p);
        adj_sort<<<gblocks(nt), 256>>>(nt, off.p, adj.p);
        // s0: the first node of minimum degree (the host's stable sort by degree)
        std::vector<int> offh(nt + 1);
        cudaMemcpy(offh.data(), off.p, sizeof(int) * (nt + 1), cudaMemcpyDeviceToHost);
        int s0 = 0;
        for (int c = 1; c < nt; ++c)
            if (offh[c + 1] - offh[c] < offh[s0 + 1] - offh[s0]) s0 = c;
        int start = s0;
        for (int pass = 0; pass < 4; ++pass) {
            int far = start;
            const int got = bfs<false>(nt, off.p, adj.p, start, order.p, vis.p, parent.p, cnt.p, key.p, key2.p,
                                       cand.p, cand2.p, &far, &offh);
            if (got < 0) return "device mesh: bfs failed";
            if (got != nt) return "device mesh: the cell graph is not connected";
            if (far == start) break;
            start = far;
        }
        const int got = bfs<true>(nt, off.p, adj.p, start, order.p, vis.p, parent.p, cnt.p, key.p, key2.p, cand.p,
                                  cand2.p, nullptr);
        if (got != nt) return "device mesh: bfs failed";
        // reverse: pos[order[i]] = nt - 1 - i; newid <- pos[newid]
        std::vector<int> ord(nt), nid(nt), ps(nt);
        cudaMemcpy(ord.data(), order.p, sizeof(int) * nt, cudaMemcpyDeviceToHost);
        for (int i = 0; i < nt; ++i) ps[ord[i]] = nt - 1 - i;
        cudaMemcpy(pos.p, ps.data(), sizeof(int) * nt, cudaMemcpyHostToDevice);
        cudaMemcpy(nid.data(), newid.p, sizeof(int) * nt, cudaMemcpyDeviceToHost);
        for (int c = 0; c < nt; ++c) nid[c] = ps[nid[c]];
        cudaMemcpy(newid.p, nid.data(), sizeof(int) * nt, cudaMemcpyHostToDevice);
    }
    // faces: orientation, then internal by (owner, neighbour), boundary by (patch, owner, a)
    DBuf<OutF> of, of2;
    DBuf<unsigned long long> fk, fk2;
    DBuf<int> fidx, fidx2;
    const size_t nfc = static_cast<size_t>(ni) + nb;
    if (!of.alloc(nfc) || !of2.alloc(nfc) || !fk.alloc(nfc) || !fk2.alloc(nfc) || !fidx.alloc(nfc) ||
        !fidx2.alloc(nfc))
        return "device mesh: out of memory";
    internal_faces<<<gblocks(ni), 256>>>(ni, np1, ifx.p, tag.p, k1s.p, kc.p, tv.p, newid.p, of.p, fk.p);
    boundary_faces<<<gblocks(nb), 256>>>(nb, n, bfx.p, tag.p, k1s.p, kc.p, tv.p, newid.p, of.p + ni, fk.p + ni);
    iota_i32<<<gblocks(nfc), 256>>>(static_cast<int>(nfc), fidx.p);
    if (!sort_pairs(fk.p, fk2.p, fidx.p, fidx2.p, ni, 64)) return "device mesh: sort failed";
    if (!sort_pairs(fk.p + ni, fk2.p + ni, fidx.p, fidx2.p + ni, nb, 63)) return "device mesh: sort failed";
    apply_perm<<<gblocks(ni), 256>>>(ni, fidx2.p, of.p, of2.p);
    apply_perm<<<gblocks(nb), 256>>>(nb, fidx2.p + ni, of.p + ni, of2.p + ni);
    std::vector<OutF> out(nfc);
    m.points.resize(npts);
    if (cudaMemcpy(out.data(), of2.p, sizeof(OutF) * nfc, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(&m.points[0].x, pts.p, sizeof(double) * 3 * npts, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaGetLastError() != cudaSuccess)
        return "device mesh: cuda error";
    m.n_cells = nt;
    m.n_internal = ni;
    m.face_off.resize(nfc + 1);
    m.face_pts.resize(3 * nfc);
    m.owner.resize(nfc);
    m.neighbour.resize(nfc);
    m.face_off[0] = 0;
    for (size_t f = 0; f < nfc; ++f) {
        m.face_pts[3 * f] = out[f].a;
        m.face_pts[3 * f + 1] = out[f].b;
        m.face_pts[3 * f + 2] = out[f].c;
        m.face_off[f + 1] = static_cast<int>(3 * (f + 1));
        m.owner[f] = out[f].own;
        m.neighbour[f] = out[f].nei;
    }
    m.patches.clear();
    for (int side = 0; side < 6; ++side) {
        Patch pa{kinds[side], 0, 0};
        int first = -1, cntp = 0;
        for (size_t x = ni; x < nfc; ++x)
            if (out[x].patch == side) {
                if (first < 0) first = static_cast<int>(x);
                ++cntp;
            }
        pa.start = first < 0 ? static_cast<int>(nfc) : first;
        pa.count = cntp;
        m.patches.push_back(pa);
    }
    return m.finalise();
}

}  // namespace sfv
