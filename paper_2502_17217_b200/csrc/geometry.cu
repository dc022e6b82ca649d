// geometry.cu — compute_geometry (/root/reference/proj/src/mesh.cpp:347-510) on the device.
//
// The four passes of the host restatement (host_mesh.cpp) as four kernels: per face
// (centroid and area vector by a fan about the vertex average), per cell (volume and
// centroid by pyramids about the cell's vertex average, faces in cell_faces order), per face
// (d, w, Delta) and per cell (least-squares tensor, its inverse, the per-(cell, face)
// vectors).  Every entry runs the sequential arithmetic of the reference for that entry
// (same operations, same order; compiled with -fmad=false), so the result is bit-identical
// to the host pass and to the reference.  Errors: the first failing face / cell of a pass,
// with the reference's message, exactly what the sequential loop reports.
#include <cmath>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "host_mesh.h"
#include "precond_dev.h"
#include "sfv_case.h"

namespace sfv {
namespace {

struct G3 {
    double x, y, z;
};
__device__ __forceinline__ G3 gadd(G3 a, G3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ G3 gsub(G3 a, G3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ G3 gscale(G3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ G3 gvdiv(G3 a, double s) { return gscale(a, 1.0 / s); }  // types.hpp:30
__device__ __forceinline__ double gdot(G3 a, G3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ G3 gcross(G3 a, G3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double gnorm(G3 a) { return sqrt(gdot(a, a)); }
__device__ __forceinline__ double gcomp(G3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }
__device__ __forceinline__ G3 ld(const double* p, long long i) { return {p[3 * i], p[3 * i + 1], p[3 * i + 2]}; }
__device__ __forceinline__ void st(double* p, long long i, G3 v) {
    p[3 * i] = v.x;
    p[3 * i + 1] = v.y;
    p[3 * i + 2] = v.z;
}

struct Topo {
    int nf, nc, nint;
    const double* pts;
    const int* face_off;
    const int* face_pts;
    const int* owner;
    const int* neigh;
    const int* cf_off;
    const int* cf;
    const int* face_kind;  // patch kind of a boundary face (SFV_PATCH_*), -1 internal
};

struct Geo {
    double *fc, *area, *amag, *normal, *d, *dmag, *w, *delta, *delmag;
    double *vol, *cen, *ginv, *ls;
    signed char* sing;
    int* err;  // [3]: first failing face of pass 1, cell of pass 2, 2 * face + kind of pass 3
};

// pass 1: face centroid + area by fan decomposition about the vertex average
__global__ void face_area_kernel(Topo t, Geo g) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= t.nf) return;
    const int b = t.face_off[f], n = t.face_off[f + 1] - b;
    G3 centre{0.0, 0.0, 0.0};
    for (int i = 0; i < n; ++i) centre = gadd(centre, ld(t.pts, t.face_pts[b + i]));
    centre = gvdiv(centre, static_cast<double>(n));
    G3 area{0.0, 0.0, 0.0}, cacc{0.0, 0.0, 0.0};
    double aacc = 0.0;
    for (int i = 0; i < n; ++i) {
        const G3 p0 = ld(t.pts, t.face_pts[b + i]);
        const G3 p1 = ld(t.pts, t.face_pts[b + (i + 1) % n]);
        const G3 tri = gscale(gcross(gsub(p0, centre), gsub(p1, centre)), 0.5);
        const double tmag = gnorm(tri);
        area = gadd(area, tri);
        cacc = gadd(cacc, gscale(gvdiv(gadd(gadd(centre, p0), p1), 3.0), tmag));
        aacc += tmag;
    }
    st(g.area, f, area);
    st(g.fc, f, aacc > 0.0 ? gvdiv(cacc, aacc) : centre);
    const double am = gnorm(area);
    g.amag[f] = am;
    if (am <= 0.0) {
        atomicMin(&g.err[0], f);
        return;
    }
    st(g.normal, f, gvdiv(area, am));
}

// pass 2: volumes and centroids by pyramids about the vertex average
__global__ void cell_volume_kernel(Topo t, Geo g) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= t.nc) return;
    G3 a{0.0, 0.0, 0.0};
    int cnt = 0;
    for (int q = t.cf_off[c]; q < t.cf_off[c + 1]; ++q) {
        const int f = t.cf[q];
        for (int x = t.face_off[f]; x < t.face_off[f + 1]; ++x) {
            a = gadd(a, ld(t.pts, t.face_pts[x]));
            ++cnt;
        }
    }
    const G3 apex = gvdiv(a, static_cast<double>(cnt));
    double vol = 0.0;
    G3 cen{0.0, 0.0, 0.0};
    for (int q = t.cf_off[c]; q < t.cf_off[c + 1]; ++q) {
        const int f = t.cf[q];
        const int b = t.face_off[f], n = t.face_off[f + 1] - b;
        const double sign = t.owner[f] == c ? 1.0 : -1.0;
        const G3 fc = ld(g.fc, f);
        for (int i = 0; i < n; ++i) {
            const G3 p0 = ld(t.pts, t.face_pts[b + i]);
            const G3 p1 = ld(t.pts, t.face_pts[b + (i + 1) % n]);
            const double v = sign * gdot(gsub(fc, apex), gcross(gsub(p0, apex), gsub(p1, apex))) / 6.0;
            vol += v;
            cen = gadd(cen, gscale(gadd(gadd(gadd(apex, fc), p0), p1), v * 0.25));
        }
    }
    g.vol[c] = vol;
    if (!(vol > 0.0)) {
        atomicMin(&g.err[1], c);
        st(g.cen, c, cen);
        return;
    }
    st(g.cen, c, gvdiv(cen, vol));
}

// pass 3: d, w, delta
__global__ void face_d_kernel(Topo t, Geo g) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= t.nf) return;
    const G3 n = ld(g.normal, f);
    const G3 xp = ld(g.cen, t.owner[f]);
    const G3 fc = ld(g.fc, f);
    G3 d;
    double w = 1.0;
    if (f < t.nint) {
        const G3 xn = ld(g.cen, t.neigh[f]);
        d = gsub(xn, xp);
        const double denom = gdot(n, gsub(xn, xp));
        if (!(denom > 0.0)) {
            st(g.d, f, d);
            atomicMin(&g.err[2], 2 * f);
            return;
        }
        w = gdot(n, gsub(xn, fc)) / denom;
    } else if (t.face_kind[f] == SFV_PATCH_SYMMETRY) {
        d = gscale(n, -2.0 * gdot(gsub(xp, fc), n));
        w = 0.5;
    } else {
        d = gsub(fc, xp);
    }
    st(g.d, f, d);
    g.w[f] = w;
    g.dmag[f] = gnorm(d);
    const double dn = gdot(d, n);
    if (!(dn > 0.0)) {
        atomicMin(&g.err[2], 2 * f + 1);
        return;
    }
    const G3 del = gvdiv(d, dn);
    st(g.delta, f, del);
    g.delmag[f] = gnorm(del);
}

// pass 4: least-squares tensors and per-(cell, face) vectors
__global__ void cell_ls_kernel(Topo t, Geo g) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= t.nc) return;
    auto incl = [&](int f) { return f < t.nint || t.face_kind[f] == SFV_PATCH_SYMMETRY; };
    double G[3][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
    for (int q = t.cf_off[c]; q < t.cf_off[c + 1]; ++q) {
        const int f = t.cf[q];
        if (!incl(f)) continue;
        const G3 d = ld(g.d, f);
        const double sc = g.amag[f] / gdot(d, d);
        const double wt = t.owner[f] == c ? g.w[f] : 1.0 - g.w[f];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) G[i][j] += (gcomp(d, i) * gcomp(d, j)) * sc * wt;
    }
    double sc = 0.0;
    for (int i = 0; i < 3; ++i) sc = fmax(sc, fabs(G[i][i]));
    const double det = G[0][0] * (G[1][1] * G[2][2] - G[1][2] * G[2][1]) -
                       G[0][1] * (G[1][0] * G[2][2] - G[1][2] * G[2][0]) +
                       G[0][2] * (G[1][0] * G[2][1] - G[1][1] * G[2][0]);
    if (sc <= 0.0 || fabs(det) < 1e-10 * sc * sc * sc) {
        g.sing[c] = 1;
        for (int k = 0; k < 9; ++k) g.ginv[9 * static_cast<long long>(c) + k] = 0.0;
        for (int q = t.cf_off[c]; q < t.cf_off[c + 1]; ++q) st(g.ls, q, G3{0.0, 0.0, 0.0});
        return;
    }
    g.sing[c] = 0;
    const double id = 1.0 / det;
    double A[3][3];
    A[0][0] = (G[1][1] * G[2][2] - G[1][2] * G[2][1]) * id;
    A[0][1] = (G[0][2] * G[2][1] - G[0][1] * G[2][2]) * id;
    A[0][2] = (G[0][1] * G[1][2] - G[0][2] * G[1][1]) * id;
    A[1][0] = (G[1][2] * G[2][0] - G[1][0] * G[2][2]) * id;
    A[1][1] = (G[0][0] * G[2][2] - G[0][2] * G[2][0]) * id;
    A[1][2] = (G[0][2] * G[1][0] - G[0][0] * G[1][2]) * id;
    A[2][0] = (G[1][0] * G[2][1] - G[1][1] * G[2][0]) * id;
    A[2][1] = (G[0][1] * G[2][0] - G[0][0] * G[2][1]) * id;
    A[2][2] = (G[0][0] * G[1][1] - G[0][1] * G[1][0]) * id;
    for (int k = 0; k < 9; ++k) g.ginv[9 * static_cast<long long>(c) + k] = A[k / 3][k % 3];
    for (int q = t.cf_off[c]; q < t.cf_off[c + 1]; ++q) {
        const int f = t.cf[q];
        if (!incl(f)) {
            st(g.ls, q, G3{0.0, 0.0, 0.0});
            continue;
        }
        G3 d = ld(g.d, f);
        double w = g.w[f];
        if (f < t.nint && t.neigh[f] == c) {
            d = {-d.x, -d.y, -d.z};
            w = 1.0 - w;
        }
        const G3 mvd = {A[0][0] * d.x + A[0][1] * d.y + A[0][2] * d.z, A[1][0] * d.x + A[1][1] * d.y + A[1][2] * d.z,
                        A[2][0] * d.x + A[2][1] * d.y + A[2][2] * d.z};
        st(g.ls, q, gscale(mvd, w * g.amag[f] / gdot(d, d)));
    }
}

}  // namespace

template <typename T>
struct Buf {
    T* p = nullptr;
    ~Buf() {
        if (p) cudaFree(p);
    }
    bool alloc(size_t n) { return cudaMalloc(&p, sizeof(T) * (n ? n : 1)) == cudaSuccess; }
    bool up(const T* h, size_t n) { return alloc(n) && (!n || cudaMemcpy(p, h, sizeof(T) * n, cudaMemcpyHostToDevice) == cudaSuccess); }
    bool down(T* h, size_t n) const { return !n || cudaMemcpy(h, p, sizeof(T) * n, cudaMemcpyDeviceToHost) == cudaSuccess; }
};

namespace {

// Layout of the default J.v path from the device-resident geometry (capi.cpp build_layout,
// host twin): per cell, its face slots in cell_faces order — face | neighbour bit, other cell
// or -(2 + patch), least-squares vector — into the tiled tables; per boundary face its
// cell * 8 + slot.
__global__ void slot_layout_kernel(Topo t, const int* __restrict__ face_patch, const double* __restrict__ ls,
                                   int spad, int* __restrict__ tsl, double* __restrict__ tls,
                                   int* __restrict__ bnd) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= t.nc) return;
    const size_t tb = static_cast<size_t>(i >> 5) * (2 * spad * 32) + (i & 31);
    const size_t lb = static_cast<size_t>(i >> 5) * (3 * spad * 32) + (i & 31);
    int s = 0;
    for (int q = t.cf_off[i]; q < t.cf_off[i + 1]; ++q, ++s) {
        const int f = t.cf[q];
        const bool nb = f < t.nint && t.neigh[f] == i;
        tsl[tb + 32 * s] = f | (nb ? static_cast<int>(0x80000000u) : 0);
        tsl[tb + 32 * (spad + s)] = f < t.nint ? (nb ? t.owner[f] : t.neigh[f]) : -(2 + face_patch[f]);
        tls[lb + 32 * (3 * s)] = ls[3 * static_cast<size_t>(q)];
        tls[lb + 32 * (3 * s + 1)] = ls[3 * static_cast<size_t>(q) + 1];
        tls[lb + 32 * (3 * s + 2)] = ls[3 * static_cast<size_t>(q) + 2];
        if (f >= t.nint) bnd[f - t.nint] = i * 8 + s;
    }
}
// face records: Gamma, Delta, |Delta| / |d|, |Gamma|, w (the host's rec[] of build_layout:
// sqrt of the left-to-right dot, then one divide — the per-face constants of rhie_chow)
__global__ void face_record_kernel(int nf, const double* __restrict__ area, const double* __restrict__ delta,
                                   const double* __restrict__ dmag, const double* __restrict__ w,
                                   double* __restrict__ f9) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nf) return;
    const double a0 = area[3 * f], a1 = area[3 * f + 1], a2 = area[3 * f + 2];
    const double d0 = delta[3 * f], d1 = delta[3 * f + 1], d2 = delta[3 * f + 2];
    const double rec[9] = {a0, a1, a2, d0, d1, d2, sqrt(d0 * d0 + d1 * d1 + d2 * d2) / dmag[f],
                           sqrt(a0 * a0 + a1 * a1 + a2 * a2), w[f]};
    const size_t b = static_cast<size_t>(f >> 5) * (9 * 32) + (f & 31);
    for (int q = 0; q < 9; ++q) f9[b + 32 * q] = rec[q];
}

}  // namespace

// device buffers kept from device_geometry for device_layout
struct DeviceGeometry {
    Buf<double> pts, fc, area, amag, normal, d, dmag, w, delta, delmag, vol, cen, ginv, ls;
    Buf<int> foff, fpts, own, nei, cfo, cfq, fkd, fpatch, err;
    Buf<signed char> sing;
    Topo t{};
};

void free_device_geometry(DeviceGeometry* g) { delete g; }

DevTopoView device_topo(const DeviceGeometry* g) {
    DevTopoView v;
    v.nc = g->t.nc;
    v.nf = g->t.nf;
    v.nint = g->t.nint;
    v.owner = g->t.owner;
    v.neigh = g->t.neigh;
    v.cf_off = g->t.cf_off;
    v.cf = g->t.cf;
    v.face_kind = g->t.face_kind;
    v.amag = g->amag.p;
    v.dmag = g->dmag.p;
    v.delmag = g->delmag.p;
    v.vol = g->vol.p;
    return v;
}

std::string device_layout(const DeviceGeometry* dg, int spad, int* tsl, double* tls, double* f9, int* bnd) {
    const Topo& t = dg->t;
    const int ntc = (t.nc + 31) / 32;
    cudaMemset(tsl, 0xff, sizeof(int) * static_cast<size_t>(ntc) * 2 * spad * 32);
    cudaMemset(tls, 0, sizeof(double) * static_cast<size_t>(ntc) * 3 * spad * 32);
    cudaMemset(f9, 0, sizeof(double) * static_cast<size_t>((t.nf + 31) / 32) * 9 * 32);
    slot_layout_kernel<<<(t.nc + 255) / 256, 256>>>(t, dg->fpatch.p, dg->ls.p, spad, tsl, tls, bnd);
    face_record_kernel<<<(t.nf + 255) / 256, 256>>>(t.nf, dg->area.p, dg->delta.p, dg->dmag.p, dg->w.p, f9);
    if (cudaDeviceSynchronize() != cudaSuccess || cudaGetLastError() != cudaSuccess) return "cuda: device layout failed";
    return "";
}

// the device-resident geometry fields download_geometry has not copied yet
std::string download_geometry(const DeviceGeometry* dg, HostGeometry& g) {
    if (!g.ls.empty() || !dg) return "";
    const Topo& t = dg->t;
    const int nf = t.nf, nc = t.nc;
    size_t ncf = 0;
    {
        int last = 0;
        if (cudaMemcpy(&last, dg->cfo.p + nc, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
            return "cuda: geometry download failed";
        ncf = static_cast<size_t>(last);
    }
    g.face_centroid.resize(nf);
    g.area.resize(nf);
    g.d.resize(nf);
    g.w.resize(nf);
    g.delta.resize(nf);
    g.centroid.resize(nc);
    g.g_inv.resize(9 * static_cast<size_t>(nc));
    g.ls.resize(ncf);
    const bool dn = dg->fc.down(&g.face_centroid[0].x, 3 * nf) && dg->area.down(&g.area[0].x, 3 * nf) &&
                    dg->d.down(&g.d[0].x, 3 * nf) && dg->w.down(g.w.data(), nf) &&
                    dg->delta.down(&g.delta[0].x, 3 * nf) && dg->cen.down(&g.centroid[0].x, 3 * nc) &&
                    dg->ginv.down(g.g_inv.data(), 9 * static_cast<size_t>(nc)) && dg->ls.down(&g.ls[0].x, 3 * ncf);
    return dn ? "" : "cuda: geometry download failed";
}

// compute_geometry on the device; fills g exactly as compute_geometry (host_mesh.cpp) does.
// Returns "" or the reference's error text (the first failing face / cell of the first
// failing pass), "cuda: ..." on a device failure.
std::string device_geometry(const HostMesh& m, HostGeometry& g, DeviceGeometry** keep) {
    const int nf = m.n_faces(), nc = m.n_cells;
    const size_t np = m.points.size(), ncf = m.cf.size();
    std::vector<int> fk(nf, -1);
    for (int f = m.n_internal; f < nf; ++f) fk[f] = m.patches[m.face_patch[f]].kind;
    DeviceGeometry* dg = new DeviceGeometry;
    struct Own {
        DeviceGeometry*& p;
        DeviceGeometry** keep;
        ~Own() {
            if (keep && p) *keep = p;
            else delete p;
        }
    } own_dg{dg, keep};
    Buf<double>&pts = dg->pts, &fc = dg->fc, &area = dg->area, &amag = dg->amag, &normal = dg->normal, &d = dg->d,
                &dmag = dg->dmag, &w = dg->w, &delta = dg->delta, &delmag = dg->delmag, &vol = dg->vol,
                &cen = dg->cen, &ginv = dg->ginv, &ls = dg->ls;
    Buf<int>&foff = dg->foff, &fpts = dg->fpts, &own = dg->own, &nei = dg->nei, &cfo = dg->cfo, &cfq = dg->cfq,
             &fkd = dg->fkd, &err = dg->err;
    Buf<signed char>& sing = dg->sing;
    if (keep && !dg->fpatch.up(m.face_patch.data(), m.face_patch.size())) return "cuda: out of device memory";
    const bool ok = pts.up(&m.points[0].x, 3 * np) && foff.up(m.face_off.data(), m.face_off.size()) &&
                    fpts.up(m.face_pts.data(), m.face_pts.size()) && own.up(m.owner.data(), nf) &&
                    nei.up(m.neighbour.data(), nf) && cfo.up(m.cf_off.data(), m.cf_off.size()) &&
                    cfq.up(m.cf.data(), ncf) && fkd.up(fk.data(), nf) && fc.alloc(3 * nf) && area.alloc(3 * nf) &&
                    amag.alloc(nf) && normal.alloc(3 * nf) && d.alloc(3 * nf) && dmag.alloc(nf) && w.alloc(nf) &&
                    delta.alloc(3 * nf) && delmag.alloc(nf) && vol.alloc(nc) && cen.alloc(3 * nc) &&
                    ginv.alloc(9 * static_cast<size_t>(nc)) && ls.alloc(3 * ncf) && sing.alloc(nc) && err.alloc(3);
    if (!ok) return "cuda: out of device memory for compute_geometry";
    cudaMemset(err.p, 0x7f, 3 * sizeof(int));
    cudaMemset(normal.p, 0, 3 * sizeof(double) * nf);
    cudaMemset(delta.p, 0, 3 * sizeof(double) * nf);
    cudaMemset(delmag.p, 0, sizeof(double) * nf);
    const Topo t{nf, nc, m.n_internal, pts.p, foff.p, fpts.p, own.p, nei.p, cfo.p, cfq.p, fkd.p};
    dg->t = t;
    const Geo gg{fc.p, area.p, amag.p, normal.p, d.p, dmag.p, w.p, delta.p, delmag.p, vol.p, cen.p, ginv.p, ls.p,
                 sing.p, err.p};
    const int bf = (nf + 255) / 256, bc = (nc + 255) / 256;
    int e[3];
    auto errs = [&]() { return cudaMemcpy(e, err.p, sizeof e, cudaMemcpyDeviceToHost) == cudaSuccess; };
    constexpr int kNone = 0x7f7f7f7f;
    face_area_kernel<<<bf, 256>>>(t, gg);
    if (!errs()) return "cuda: compute_geometry failed";
    if (e[0] != kNone) return "compute_geometry: zero-area face " + std::to_string(e[0]);
    cell_volume_kernel<<<bc, 256>>>(t, gg);
    if (!errs()) return "cuda: compute_geometry failed";
    if (e[1] != kNone) return "compute_geometry: non-positive volume in cell " + std::to_string(e[1]);
    face_d_kernel<<<bf, 256>>>(t, gg);
    if (!errs()) return "cuda: compute_geometry failed";
    if (e[2] != kNone) {
        const int f = e[2] >> 1;
        return (e[2] & 1) ? "compute_geometry: degenerate centroid geometry at face " + std::to_string(f)
                          : "compute_geometry: face " + std::to_string(f) + " area vector does not leave the owner";
    }
    cell_ls_kernel<<<bc, 256>>>(t, gg);
    // what the host reads later (J~ assembly: |Gamma|, |d|, |Delta|, n, volume; the singular
    // flags) now; the rest stays on the device until download_geometry (lazy: only the
    // geometry API and the alternative J.v layouts read it)
    g.area_mag.resize(nf);
    g.normal.resize(nf);
    g.d_mag.resize(nf);
    g.delta_mag.resize(nf);
    g.volume.resize(nc);
    g.g_singular.resize(nc);
    bool dn = amag.down(g.area_mag.data(), nf) && normal.down(&g.normal[0].x, 3 * nf) &&
              dmag.down(g.d_mag.data(), nf) && delmag.down(g.delta_mag.data(), nf) && vol.down(g.volume.data(), nc) &&
              sing.down(g.g_singular.data(), nc);
    if (dn && !keep) dn = download_geometry(dg, g).empty();
    if (!dn || cudaGetLastError() != cudaSuccess) return "cuda: compute_geometry failed";
    return "";
}

}  // namespace sfv
