// host_mesh.cpp — mesh generators and geometry precompute (host, once per run).
//
// Restates /root/reference/proj/src/mesh.cpp arithmetic exactly (see host_mesh.h);
// every V3 helper below mirrors the operator of include/solidfv/types.hpp it stands for.
#include "host_threads.h"
#include "host_mesh.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <limits>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "sfv_case.h"

namespace sfv {
namespace {

inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 scale(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline V3 vdiv(V3 a, double s) { return scale(a, 1.0 / s); }  // types.hpp:30
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline double norm(V3 a) { return std::sqrt(dot(a, a)); }
inline double comp(V3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

struct M3 {
    double m[3][3];
};
inline M3 mzero() { M3 r; std::memset(&r, 0, sizeof r); return r; }
inline M3 outer(V3 a, V3 b) {
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[i][j] = comp(a, i) * comp(b, j);
    return r;
}
inline M3 mscale(M3 a, double s) {
    for (auto& row : a.m)
        for (double& v : row) v *= s;
    return a;
}
inline void madd_to(M3& a, const M3& b) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) a.m[i][j] += b.m[i][j];
}
inline double mdet(const M3& a) {
    return a.m[0][0] * (a.m[1][1] * a.m[2][2] - a.m[1][2] * a.m[2][1]) -
           a.m[0][1] * (a.m[1][0] * a.m[2][2] - a.m[1][2] * a.m[2][0]) +
           a.m[0][2] * (a.m[1][0] * a.m[2][1] - a.m[1][1] * a.m[2][0]);
}
inline M3 minverse(const M3& a) {
    const double id = 1.0 / mdet(a);
    M3 r;
    r.m[0][0] = (a.m[1][1] * a.m[2][2] - a.m[1][2] * a.m[2][1]) * id;
    r.m[0][1] = (a.m[0][2] * a.m[2][1] - a.m[0][1] * a.m[2][2]) * id;
    r.m[0][2] = (a.m[0][1] * a.m[1][2] - a.m[0][2] * a.m[1][1]) * id;
    r.m[1][0] = (a.m[1][2] * a.m[2][0] - a.m[1][0] * a.m[2][2]) * id;
    r.m[1][1] = (a.m[0][0] * a.m[2][2] - a.m[0][2] * a.m[2][0]) * id;
    r.m[1][2] = (a.m[0][2] * a.m[1][0] - a.m[0][0] * a.m[1][2]) * id;
    r.m[2][0] = (a.m[1][0] * a.m[2][1] - a.m[1][1] * a.m[2][0]) * id;
    r.m[2][1] = (a.m[0][1] * a.m[2][0] - a.m[0][0] * a.m[2][1]) * id;
    r.m[2][2] = (a.m[0][0] * a.m[1][1] - a.m[0][1] * a.m[1][0]) * id;
    return r;
}
inline V3 mv(const M3& a, V3 v) {
    return {a.m[0][0] * v.x + a.m[0][1] * v.y + a.m[0][2] * v.z,
            a.m[1][0] * v.x + a.m[1][1] * v.y + a.m[1][2] * v.z,
            a.m[2][0] * v.x + a.m[2][1] * v.y + a.m[2][2] * v.z};
}

// SplitMix64, counter-seeded per point (mesh.cpp:220-229, :328)
struct SplitMix64 {
    uint64_t state;
    uint64_t next() {
        uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

V3 raw_face_area(const HostMesh& m, int f) {  // mesh.cpp:231-246, 3-D branch
    const int b = m.face_off[f], e = m.face_off[f + 1], n = e - b;
    V3 centre{};
    for (int q = b; q < e; ++q) centre = add(centre, m.points[m.face_pts[q]]);
    centre = vdiv(centre, static_cast<double>(n));
    V3 a{};
    for (int i = 0; i < n; ++i) {
        const V3 p0 = m.points[m.face_pts[b + i]];
        const V3 p1 = m.points[m.face_pts[b + (i + 1) % n]];
        a = add(a, scale(cross(sub(p0, centre), sub(p1, centre)), 0.5));
    }
    return a;
}

std::vector<double> cell_volumes(const HostMesh& m) {  // mesh.cpp:249-286, 3-D branch
    std::vector<V3> sum(m.n_cells);
    std::vector<int> cnt(m.n_cells, 0);
    for (int f = 0; f < m.n_faces(); ++f)
        for (int q = m.face_off[f]; q < m.face_off[f + 1]; ++q) {
            const V3 p = m.points[m.face_pts[q]];
            sum[m.owner[f]] = add(sum[m.owner[f]], p);
            ++cnt[m.owner[f]];
            if (m.neighbour[f] >= 0) {
                sum[m.neighbour[f]] = add(sum[m.neighbour[f]], p);
                ++cnt[m.neighbour[f]];
            }
        }
    std::vector<double> vol(m.n_cells, 0.0);
    for (int f = 0; f < m.n_faces(); ++f) {
        const int b = m.face_off[f], n = m.face_off[f + 1] - b;
        for (int side = 0; side < 2; ++side) {
            const int c = side == 0 ? m.owner[f] : m.neighbour[f];
            if (c < 0) continue;
            const double sign = side == 0 ? 1.0 : -1.0;
            const V3 apex = vdiv(sum[c], static_cast<double>(cnt[c]));
            V3 fc{};
            for (int i = 0; i < n; ++i) fc = add(fc, m.points[m.face_pts[b + i]]);
            fc = vdiv(fc, static_cast<double>(n));
            for (int i = 0; i < n; ++i) {
                const V3 q0 = sub(fc, apex);
                const V3 q1 = sub(m.points[m.face_pts[b + i]], apex);
                const V3 q2 = sub(m.points[m.face_pts[b + (i + 1) % n]], apex);
                vol[c] += sign * dot(q0, cross(q1, q2)) / 6.0;
            }
        }
    }
    return vol;
}

}  // namespace

std::string HostMesh::finalise() {  // Mesh::finalise (mesh.cpp:29-62)
    const int nf = n_faces();
    if (static_cast<int>(neighbour.size()) != nf || static_cast<int>(face_off.size()) != nf + 1)
        return "mesh: owner/neighbour size mismatch";
    face_patch.assign(nf, -1);
    for (std::size_t p = 0; p < patches.size(); ++p) {
        const Patch& pa = patches[p];
        if (pa.start < n_internal || pa.start + pa.count > nf)
            return "mesh: patch range outside boundary faces";
        for (int f = pa.start; f < pa.start + pa.count; ++f) {
            if (face_patch[f] != -1) return "mesh: face in two patches";
            face_patch[f] = static_cast<int>(p);
        }
    }
    for (int f = 0; f < nf; ++f) {
        const bool boundary = neighbour[f] < 0;
        if (boundary != (f >= n_internal)) return "mesh: internal faces must precede boundary faces";
        if (boundary && face_patch[f] == -1) return "mesh: boundary face not in any patch";
        if (owner[f] < 0 || owner[f] >= n_cells || neighbour[f] >= n_cells)
            return "mesh: face cell index out of range";
    }
    cf_off.assign(n_cells + 1, 0);
    for (int f = 0; f < nf; ++f) {
        ++cf_off[owner[f] + 1];
        if (neighbour[f] >= 0) ++cf_off[neighbour[f] + 1];
    }
    for (int c = 0; c < n_cells; ++c) {
        if (cf_off[c + 1] == 0) return "mesh: cell without faces";
        cf_off[c + 1] += cf_off[c];
    }
    cf.assign(cf_off[n_cells], 0);
    std::vector<int> fill(cf_off.begin(), cf_off.end() - 1);
    for (int f = 0; f < nf; ++f) {
        cf[fill[owner[f]]++] = f;
        if (neighbour[f] >= 0) cf[fill[neighbour[f]]++] = f;
    }
    return "";
}

HostMesh box_hex(const double ext[3], const int div[3], const int kinds[6]) {
    const int nx = div[0], ny = div[1], nz = div[2];
    auto pid = [&](int i, int j, int k) { return i + (nx + 1) * (j + (ny + 1) * k); };
    auto cid = [&](int i, int j, int k) { return i + nx * (j + ny * k); };
    HostMesh m;
    m.n_cells = nx * ny * nz;
    m.points.reserve(static_cast<std::size_t>(nx + 1) * (ny + 1) * (nz + 1));
    for (int k = 0; k <= nz; ++k)
        for (int j = 0; j <= ny; ++j)
            for (int i = 0; i <= nx; ++i)
                m.points.push_back({ext[0] * i / nx, ext[1] * j / ny, ext[2] * k / nz});
    m.face_off.push_back(0);
    auto add_face = [&](int a, int b, int c, int d, int own, int nei) {
        m.face_pts.insert(m.face_pts.end(), {a, b, c, d});
        m.face_off.push_back(static_cast<int>(m.face_pts.size()));
        m.owner.push_back(own);
        m.neighbour.push_back(nei);
    };
    // internal faces, owner = lower cell (mesh.cpp:100-118)
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i + 1 < nx; ++i)
                add_face(pid(i + 1, j, k), pid(i + 1, j + 1, k), pid(i + 1, j + 1, k + 1), pid(i + 1, j, k + 1),
                         cid(i, j, k), cid(i + 1, j, k));
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j + 1 < ny; ++j)
            for (int i = 0; i < nx; ++i)
                add_face(pid(i, j + 1, k), pid(i, j + 1, k + 1), pid(i + 1, j + 1, k + 1), pid(i + 1, j + 1, k),
                         cid(i, j, k), cid(i, j + 1, k));
    for (int k = 0; k + 1 < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i)
                add_face(pid(i, j, k + 1), pid(i + 1, j, k + 1), pid(i + 1, j + 1, k + 1), pid(i, j + 1, k + 1),
                         cid(i, j, k), cid(i, j, k + 1));
    m.n_internal = m.n_faces();
    auto begin_patch = [&](int side) { m.patches.push_back({kinds[side], m.n_faces(), 0}); };
    auto end_patch = [&] { m.patches.back().count = m.n_faces() - m.patches.back().start; };
    begin_patch(0);  // xmin (mesh.cpp:127-132)
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            add_face(pid(0, j, k), pid(0, j, k + 1), pid(0, j + 1, k + 1), pid(0, j + 1, k), cid(0, j, k), -1);
    end_patch();
    begin_patch(1);  // xmax
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            add_face(pid(nx, j, k), pid(nx, j + 1, k), pid(nx, j + 1, k + 1), pid(nx, j, k + 1), cid(nx - 1, j, k), -1);
    end_patch();
    begin_patch(2);  // ymin
    for (int k = 0; k < nz; ++k)
        for (int i = 0; i < nx; ++i)
            add_face(pid(i, 0, k), pid(i + 1, 0, k), pid(i + 1, 0, k + 1), pid(i, 0, k + 1), cid(i, 0, k), -1);
    end_patch();
    begin_patch(3);  // ymax
    for (int k = 0; k < nz; ++k)
        for (int i = 0; i < nx; ++i)
            add_face(pid(i, ny, k), pid(i, ny, k + 1), pid(i + 1, ny, k + 1), pid(i + 1, ny, k), cid(i, ny - 1, k), -1);
    end_patch();
    begin_patch(4);  // zmin
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i)
            add_face(pid(i, j, 0), pid(i, j + 1, 0), pid(i + 1, j + 1, 0), pid(i + 1, j, 0), cid(i, j, 0), -1);
    end_patch();
    begin_patch(5);  // zmax
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i)
            add_face(pid(i, j, nz), pid(i + 1, j, nz), pid(i + 1, j + 1, nz), pid(i, j + 1, nz), cid(i, j, nz - 1), -1);
    end_patch();
    m.finalise();
    return m;
}

std::string distort(HostMesh& mesh, double factor, uint64_t seed) {  // mesh.cpp:290-345
    if (factor < 0.0 || factor >= 0.5) return "distort_mesh: factor must be in [0, 0.5)";
    if (factor == 0.0) return "";
    const int np = static_cast<int>(mesh.points.size());
    std::vector<double> min_edge(np, std::numeric_limits<double>::max());
    for (int f = 0; f < mesh.n_faces(); ++f) {
        const int b = mesh.face_off[f], n = mesh.face_off[f + 1] - b;
        for (int i = 0; i < n; ++i) {
            const int a = mesh.face_pts[b + i], c = mesh.face_pts[b + (i + 1) % n];
            if (n == 2 && i == 1) break;
            const double len = norm(sub(mesh.points[a], mesh.points[c]));
            min_edge[a] = std::min(min_edge[a], len);
            min_edge[c] = std::min(min_edge[c], len);
        }
    }
    // distinct boundary plane normals per point (at most 3 matter: >=2 freezes the point)
    std::vector<V3> plane0(np);
    std::vector<int> nplanes(np, 0);
    std::vector<V3> plane1(np);
    for (int f = mesh.n_internal; f < mesh.n_faces(); ++f) {
        V3 n = raw_face_area(mesh, f);
        const double mag = norm(n);
        if (mag == 0.0) return "distort_mesh: zero-area boundary face";
        n = vdiv(n, mag);
        for (int q = mesh.face_off[f]; q < mesh.face_off[f + 1]; ++q) {
            const int p = mesh.face_pts[q];
            bool known = false;
            if (nplanes[p] >= 1 && std::abs(dot(plane0[p], n)) > 1.0 - 1e-8) known = true;
            if (nplanes[p] >= 2 && std::abs(dot(plane1[p], n)) > 1.0 - 1e-8) known = true;
            if (!known) {
                if (nplanes[p] == 0) plane0[p] = n;
                else if (nplanes[p] == 1) plane1[p] = n;
                ++nplanes[p];
            }
        }
    }
    const std::vector<V3> orig = mesh.points;
    (void)orig;
    for (int p = 0; p < np; ++p) {
        if (nplanes[p] >= 2) continue;
        SplitMix64 rng{seed * 0x9E3779B97F4A7C15ULL ^ (static_cast<uint64_t>(p) + 1) * 0xD1B54A32D192ED03ULL};
        V3 v;
        v.x = 2.0 * rng.uniform01() - 1.0;
        v.y = 2.0 * rng.uniform01() - 1.0;
        v.z = 2.0 * rng.uniform01() - 1.0;
        const double mag_draw = rng.uniform01();
        if (nplanes[p] == 1) {
            const V3 n = plane0[p];
            v = sub(v, scale(n, dot(v, n)));
        }
        const double vn = norm(v);
        if (vn < 1e-12) continue;
        mesh.points[p] = add(mesh.points[p], scale(v, factor * min_edge[p] * mag_draw / vn));
    }
    for (double vol : cell_volumes(mesh))
        if (!(vol > 0.0)) return "distort_mesh: negative cell volume, retry with smaller factor";
    return "";
}

namespace {

// Runs body(i) for i in [0, n) on up to 16 threads; body returns "" or an error.  Returns
// the error of the smallest failing index, i.e. what the sequential loop would report.
std::string parallel_for(int n, const std::function<std::string(int)>& body) {
    const int nth = host_threads();
    if (n < 4096 || nth == 1) {
        for (int i = 0; i < n; ++i)
            if (std::string e = body(i); !e.empty()) return e;
        return "";
    }
    std::vector<int> first(nth, n);
    std::vector<std::string> msg(nth);
    std::vector<std::thread> th;
    const int ch = (n + nth - 1) / nth;
    for (int k = 0; k < nth; ++k)
        th.emplace_back([&, k] {
            for (int i = k * ch; i < std::min(n, (k + 1) * ch); ++i)
                if (std::string e = body(i); !e.empty()) {
                    first[k] = i;
                    msg[k] = e;
                    return;
                }
        });
    for (auto& t : th) t.join();
    for (int k = 0; k < nth; ++k)  // ranges are ascending: the first thread with an error has the smallest index
        if (first[k] < n) return msg[k];
    return "";
}

}  // namespace

// Every pass is either per face, or per cell accumulating its faces in ascending face
// order (cell_faces order) — the order in which the reference's face loops reach the cell —
// so each pass runs in parallel with the sequential arithmetic of every entry.
std::string compute_geometry(const HostMesh& m, HostGeometry& g) {  // mesh.cpp:347-510
    const int nf = m.n_faces(), nc = m.n_cells;
    g.face_centroid.assign(nf, V3{});
    g.area.assign(nf, V3{});
    g.area_mag.assign(nf, 0.0);
    g.normal.assign(nf, V3{});
    g.d.assign(nf, V3{});
    g.d_mag.assign(nf, 0.0);
    g.w.assign(nf, 1.0);
    g.delta.assign(nf, V3{});
    g.delta_mag.assign(nf, 0.0);
    auto kind = [&](int f) { return m.patches[m.face_patch[f]].kind; };
    // pass 1: face centroid + area by fan decomposition about the vertex average
    std::string e = parallel_for(nf, [&](int f) -> std::string {
        const int b = m.face_off[f], n = m.face_off[f + 1] - b;
        V3 centre{};
        for (int i = 0; i < n; ++i) centre = add(centre, m.points[m.face_pts[b + i]]);
        centre = vdiv(centre, static_cast<double>(n));
        V3 area{}, cacc{};
        double aacc = 0.0;
        for (int i = 0; i < n; ++i) {
            const V3 p0 = m.points[m.face_pts[b + i]];
            const V3 p1 = m.points[m.face_pts[b + (i + 1) % n]];
            const V3 tri = scale(cross(sub(p0, centre), sub(p1, centre)), 0.5);
            const double tmag = norm(tri);
            area = add(area, tri);
            cacc = add(cacc, scale(vdiv(add(add(centre, p0), p1), 3.0), tmag));
            aacc += tmag;
        }
        g.area[f] = area;
        g.face_centroid[f] = aacc > 0.0 ? vdiv(cacc, aacc) : centre;
        g.area_mag[f] = norm(area);
        if (g.area_mag[f] <= 0.0) return "compute_geometry: zero-area face " + std::to_string(f);
        g.normal[f] = vdiv(area, g.area_mag[f]);
        return "";
    });
    if (!e.empty()) return e;
    // pass 2: volumes and centroids by pyramids about the vertex average
    std::vector<V3> apex(nc);
    g.volume.assign(nc, 0.0);
    g.centroid.assign(nc, V3{});
    e = parallel_for(nc, [&](int c) -> std::string {
        V3 a{};
        int cnt = 0;
        for (int q = m.cf_off[c]; q < m.cf_off[c + 1]; ++q) {
            const int f = m.cf[q];
            for (int x = m.face_off[f]; x < m.face_off[f + 1]; ++x) {
                a = add(a, m.points[m.face_pts[x]]);
                ++cnt;
            }
        }
        apex[c] = vdiv(a, static_cast<double>(cnt));
        for (int q = m.cf_off[c]; q < m.cf_off[c + 1]; ++q) {
            const int f = m.cf[q];
            const int b = m.face_off[f], n = m.face_off[f + 1] - b;
            const double sign = m.owner[f] == c ? 1.0 : -1.0;
            for (int i = 0; i < n; ++i) {
                const V3 p0 = m.points[m.face_pts[b + i]];
                const V3 p1 = m.points[m.face_pts[b + (i + 1) % n]];
                const V3 fc = g.face_centroid[f];
                const double v = sign * dot(sub(fc, apex[c]), cross(sub(p0, apex[c]), sub(p1, apex[c]))) / 6.0;
                g.volume[c] += v;
                g.centroid[c] = add(g.centroid[c], scale(add(add(add(apex[c], fc), p0), p1), v * 0.25));
            }
        }
        if (!(g.volume[c] > 0.0)) return "compute_geometry: non-positive volume in cell " + std::to_string(c);
        g.centroid[c] = vdiv(g.centroid[c], g.volume[c]);
        return "";
    });
    if (!e.empty()) return e;
    // pass 3: d, w, delta
    e = parallel_for(nf, [&](int f) -> std::string {
        const V3 n = g.normal[f];
        const V3 xp = g.centroid[m.owner[f]];
        if (f < m.n_internal) {
            const V3 xn = g.centroid[m.neighbour[f]];
            g.d[f] = sub(xn, xp);
            const double denom = dot(n, sub(xn, xp));
            if (!(denom > 0.0))
                return "compute_geometry: face " + std::to_string(f) + " area vector does not leave the owner";
            g.w[f] = dot(n, sub(xn, g.face_centroid[f])) / denom;
        } else if (kind(f) == SFV_PATCH_SYMMETRY) {
            g.d[f] = scale(n, -2.0 * dot(sub(xp, g.face_centroid[f]), n));
            g.w[f] = 0.5;
        } else {
            g.d[f] = sub(g.face_centroid[f], xp);
        }
        g.d_mag[f] = norm(g.d[f]);
        const double dn = dot(g.d[f], n);
        if (!(dn > 0.0)) return "compute_geometry: degenerate centroid geometry at face " + std::to_string(f);
        g.delta[f] = vdiv(g.d[f], dn);
        g.delta_mag[f] = norm(g.delta[f]);
        return "";
    });
    if (!e.empty()) return e;
    // pass 4: least-squares tensors and per-(cell, face) vectors
    g.g_inv.assign(9 * static_cast<std::size_t>(nc), 0.0);
    g.g_singular.assign(nc, 0);
    g.ls.assign(m.cf.size(), V3{});
    auto incl = [&](int f) { return f < m.n_internal || kind(f) == SFV_PATCH_SYMMETRY; };
    parallel_for(nc, [&](int c) -> std::string {
        M3 G = mzero();
        for (int q = m.cf_off[c]; q < m.cf_off[c + 1]; ++q) {
            const int f = m.cf[q];
            if (!incl(f)) continue;
            const M3 dd = mscale(outer(g.d[f], g.d[f]), g.area_mag[f] / dot(g.d[f], g.d[f]));
            madd_to(G, mscale(dd, m.owner[f] == c ? g.w[f] : 1.0 - g.w[f]));
        }
        double sc = 0.0;
        for (int i = 0; i < 3; ++i) sc = std::max(sc, std::abs(G.m[i][i]));
        if (sc <= 0.0 || std::abs(mdet(G)) < 1e-10 * sc * sc * sc) {
            g.g_singular[c] = 1;
            return "";
        }
        const M3 ginv = minverse(G);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) g.g_inv[9 * static_cast<std::size_t>(c) + 3 * i + j] = ginv.m[i][j];
        for (int q = m.cf_off[c]; q < m.cf_off[c + 1]; ++q) {
            const int f = m.cf[q];
            if (!incl(f)) continue;
            V3 d = g.d[f];
            double w = g.w[f];
            if (f < m.n_internal && m.neighbour[f] == c) {
                d = {-d.x, -d.y, -d.z};
                w = 1.0 - w;
            }
            g.ls[q] = scale(mv(ginv, d), w * g.area_mag[f] / dot(d, d));
        }
        return "";
    });
    return "";
}

// ---------------------------------------------------------------- config 5 tets

namespace {

uint64_t splitmix_at(uint64_t seed, uint64_t i) {
    SplitMix64 r{seed * 0x9E3779B97F4A7C15ULL ^ (i + 1) * 0xD1B54A32D192ED03ULL};
    return r.next();
}

// reverse Cuthill-McKee over the cell graph (CSR), starting each component from a
// minimum-degree pseudo-peripheral node.
std::vector<int> rcm(const std::vector<int>& off, const std::vector<int>& adj) {
    const int n = static_cast<int>(off.size()) - 1;
    std::vector<int> order;
    order.reserve(n);
    std::vector<char> seen(n, 0);
    std::vector<int> level(n, -1), q;
    q.reserve(n);
    auto deg = [&](int v) { return off[v + 1] - off[v]; };
    std::vector<int> by_deg(n);
    std::iota(by_deg.begin(), by_deg.end(), 0);
    std::stable_sort(by_deg.begin(), by_deg.end(), [&](int a, int b) { return deg(a) < deg(b); });
    std::vector<int> nb;
    for (int s0 : by_deg) {
        if (seen[s0]) continue;
        int start = s0;
        for (int pass = 0; pass < 4; ++pass) {
            q.clear();
            q.push_back(start);
            level[start] = 0;
            int far = start;
            for (std::size_t h = 0; h < q.size(); ++h) {
                const int u = q[h];
                for (int e = off[u]; e < off[u + 1]; ++e) {
                    const int v = adj[e];
                    if (level[v] >= 0) continue;
                    level[v] = level[u] + 1;
                    q.push_back(v);
                    if (level[v] > level[far] || (level[v] == level[far] && deg(v) < deg(far))) far = v;
                }
            }
            for (int t : q) level[t] = -1;
            if (far == start) break;
            start = far;
        }
        const std::size_t base = order.size();
        order.push_back(start);
        seen[start] = 1;
        for (std::size_t h = base; h < order.size(); ++h) {
            const int u = order[h];
            nb.clear();
            for (int e = off[u]; e < off[u + 1]; ++e)
                if (!seen[adj[e]]) {
                    seen[adj[e]] = 1;
                    nb.push_back(adj[e]);
                }
            std::stable_sort(nb.begin(), nb.end(), [&](int a, int b) { return deg(a) < deg(b); });
            order.insert(order.end(), nb.begin(), nb.end());
        }
    }
    std::reverse(order.begin(), order.end());
    return order;
}

struct FaceKey {
    uint64_t k1;  // (a << 32) | b, a < b < c sorted point ids
    uint32_t c;
    uint32_t tag;  // tet * 4 + local face
    bool operator<(const FaceKey& o) const { return k1 != o.k1 ? k1 < o.k1 : c != o.c ? c < o.c : tag < o.tag; }
};

}  // namespace

HostMesh kuhn_tets(const double ext[3], int n, const int kinds[6], uint64_t perm_seed, bool permute, bool do_rcm,
                   bool* on_device) {
    if (on_device) *on_device = false;
    // on the device when there is one (mesh_dev.cu, the same mesh array for array); the seeded
    // Fisher-Yates permutation is a sequential chain of swaps and is drawn here
    if (!std::getenv("SFV_HOST_MESH") && n >= 8) {
        const long long ntl = 6LL * n * n * n;
        std::vector<int> newid;
        if (permute && ntl < (1LL << 28)) {
            const int nt = static_cast<int>(ntl);
            std::vector<int> perm(nt);
            std::iota(perm.begin(), perm.end(), 0);
            for (int i = nt - 1; i > 0; --i) {
                const int r = static_cast<int>(splitmix_at(perm_seed, static_cast<uint64_t>(i)) % static_cast<uint64_t>(i + 1));
                std::swap(perm[i], perm[r]);
            }
            newid.resize(nt);
            for (int i = 0; i < nt; ++i) newid[perm[i]] = i;
        }
        HostMesh dm;
        if (device_kuhn_tets(ext, n, kinds, permute ? &newid : nullptr, do_rcm, dm).empty()) {
            if (on_device) *on_device = true;
            return dm;
        }
    }
    const int np1 = n + 1;
    auto pid = [&](int i, int j, int k) { return i + np1 * (j + np1 * k); };
    HostMesh m;
    m.points.reserve(static_cast<std::size_t>(np1) * np1 * np1);
    for (int k = 0; k <= n; ++k)
        for (int j = 0; j <= n; ++j)
            for (int i = 0; i <= n; ++i) m.points.push_back({ext[0] * i / n, ext[1] * j / n, ext[2] * k / n});
    // six Kuhn tets per hex along the (mirrored) main diagonal
    static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    const long long ntet = 6LL * n * n * n;
    std::vector<int> tv(4 * ntet);
    long long t = 0;
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i)
                for (const auto& pr : perms) {
                    int loc[3] = {0, 0, 0};
                    const int base[3] = {i, j, k};
                    for (int s = 0; s < 4; ++s) {
                        if (s > 0) loc[pr[s - 1]] = 1;
                        int g[3];
                        for (int a = 0; a < 3; ++a) g[a] = base[a] + ((base[a] & 1) ? 1 - loc[a] : loc[a]);
                        tv[4 * t + s] = pid(g[0], g[1], g[2]);
                    }
                    ++t;
                }
    const int nt = static_cast<int>(ntet);
    // faces: sort keys of the 4 * nt triangles; equal keys pair into internal faces
    std::vector<FaceKey> keys(4 * static_cast<std::size_t>(nt));
    for (int c = 0; c < nt; ++c)
        for (int lf = 0; lf < 4; ++lf) {
            int p[3], q = 0;
            for (int s = 0; s < 4; ++s)
                if (s != lf) p[q++] = tv[4 * c + s];
            std::sort(p, p + 3);
            keys[4 * static_cast<std::size_t>(c) + lf] = {(static_cast<uint64_t>(p[0]) << 32) | static_cast<uint32_t>(p[1]),
                                                         static_cast<uint32_t>(p[2]), static_cast<uint32_t>(4 * c + lf)};
        }
    std::sort(keys.begin(), keys.end());
    // cell renumbering: random permutation (Fisher-Yates on SplitMix64) then RCM
    std::vector<int> newid(nt);
    std::iota(newid.begin(), newid.end(), 0);
    if (permute) {
        std::vector<int> perm(nt);
        std::iota(perm.begin(), perm.end(), 0);
        for (int i = nt - 1; i > 0; --i) {
            const int r = static_cast<int>(splitmix_at(perm_seed, static_cast<uint64_t>(i)) % static_cast<uint64_t>(i + 1));
            std::swap(perm[i], perm[r]);
        }
        for (int i = 0; i < nt; ++i) newid[perm[i]] = i;
    }
    struct IFace {
        int a, b;  // old tet ids
        uint32_t key_idx;
    };
    std::vector<IFace> ifaces;
    std::vector<uint32_t> bfaces;
    ifaces.reserve(2 * static_cast<std::size_t>(nt));
    for (std::size_t x = 0; x < keys.size();) {
        if (x + 1 < keys.size() && keys[x + 1].k1 == keys[x].k1 && keys[x + 1].c == keys[x].c) {
            ifaces.push_back({static_cast<int>(keys[x].tag / 4), static_cast<int>(keys[x + 1].tag / 4), static_cast<uint32_t>(x)});
            x += 2;
        } else {
            bfaces.push_back(static_cast<uint32_t>(x));
            x += 1;
        }
    }
    if (do_rcm) {
        std::vector<int> off(nt + 1, 0);
        for (const IFace& f : ifaces) {
            ++off[newid[f.a] + 1];
            ++off[newid[f.b] + 1];
        }
        for (int c = 0; c < nt; ++c) off[c + 1] += off[c];
        std::vector<int> adj(off[nt]);
        std::vector<int> fill(off.begin(), off.end() - 1);
        for (const IFace& f : ifaces) {
            const int a = newid[f.a], b = newid[f.b];
            adj[fill[a]++] = b;
            adj[fill[b]++] = a;
        }
        for (int c = 0; c < nt; ++c) std::sort(adj.begin() + off[c], adj.begin() + off[c + 1]);
        const std::vector<int> order = rcm(off, adj);
        std::vector<int> pos(nt);
        for (int i = 0; i < nt; ++i) pos[order[i]] = i;
        for (int c = 0; c < nt; ++c) newid[c] = pos[newid[c]];
    }
    // lattice coordinates of a point id, for exact orientation and patch detection
    auto lat = [&](int p, int out[3]) {
        out[0] = p % np1;
        out[1] = (p / np1) % np1;
        out[2] = p / (np1 * np1);
    };
    // orient (a, b, c) so the right-hand normal leaves the cell whose 4th vertex is d
    auto orient = [&](int& a, int& b, int& c, int d) {
        int pa[3], pb[3], pc[3], pd[3];
        lat(a, pa), lat(b, pb), lat(c, pc), lat(d, pd);
        long long e1[3], e2[3], e3[3];
        for (int s = 0; s < 3; ++s) {
            e1[s] = pb[s] - pa[s];
            e2[s] = pc[s] - pa[s];
            e3[s] = pd[s] - pa[s];
        }
        const long long nx = e1[1] * e2[2] - e1[2] * e2[1], ny = e1[2] * e2[0] - e1[0] * e2[2],
                        nz = e1[0] * e2[1] - e1[1] * e2[0];
        if (nx * e3[0] + ny * e3[1] + nz * e3[2] > 0) std::swap(b, c);
        // rotate the smallest id first (deterministic point order)
        if (b < a && b < c) { const int t0 = a; a = b; b = c; c = t0; }
        else if (c < a && c < b) { const int t0 = c; c = b; b = a; a = t0; }
    };
    auto fourth = [&](uint32_t tag) { return tv[4 * (tag / 4) + (tag % 4)]; };
    struct OutFace {
        int own, nei, a, b, c, patch;
    };
    std::vector<OutFace> out;
    out.reserve(ifaces.size() + bfaces.size());
    for (const IFace& f : ifaces) {
        const FaceKey& k = keys[f.key_idx];
        int a = static_cast<int>(k.k1 >> 32), b = static_cast<int>(k.k1 & 0xffffffffu), c = static_cast<int>(k.c);
        int own = newid[f.a], nei = newid[f.b];
        uint32_t own_tag = k.tag;
        if (own > nei) {
            std::swap(own, nei);
            own_tag = keys[f.key_idx + 1].tag;
        }
        orient(a, b, c, fourth(own_tag));
        out.push_back({own, nei, a, b, c, -1});
    }
    for (uint32_t x : bfaces) {
        const FaceKey& k = keys[x];
        int a = static_cast<int>(k.k1 >> 32), b = static_cast<int>(k.k1 & 0xffffffffu), c = static_cast<int>(k.c);
        int la[3], lb[3], lc[3];
        lat(a, la), lat(b, lb), lat(c, lc);
        int side = -1;
        for (int ax = 0; ax < 3 && side < 0; ++ax) {
            if (la[ax] == 0 && lb[ax] == 0 && lc[ax] == 0) side = 2 * ax;
            else if (la[ax] == n && lb[ax] == n && lc[ax] == n) side = 2 * ax + 1;
        }
        orient(a, b, c, fourth(k.tag));
        out.push_back({newid[k.tag / 4], -1, a, b, c, side});
    }
    const std::size_t ni = ifaces.size();
    std::sort(out.begin(), out.begin() + ni, [](const OutFace& x, const OutFace& y) {
        return x.own != y.own ? x.own < y.own : x.nei < y.nei;
    });
    std::sort(out.begin() + ni, out.end(), [](const OutFace& x, const OutFace& y) {
        return x.patch != y.patch ? x.patch < y.patch : x.own != y.own ? x.own < y.own : x.a < y.a;
    });
    m.n_cells = nt;
    m.n_internal = static_cast<int>(ni);
    m.face_off.reserve(out.size() + 1);
    m.face_off.push_back(0);
    for (const OutFace& f : out) {
        m.face_pts.insert(m.face_pts.end(), {f.a, f.b, f.c});
        m.face_off.push_back(static_cast<int>(m.face_pts.size()));
        m.owner.push_back(f.own);
        m.neighbour.push_back(f.nei);
    }
    for (int side = 0; side < 6; ++side) {
        Patch pa{kinds[side], 0, 0};
        int first = -1, cnt = 0;
        for (std::size_t x = ni; x < out.size(); ++x)
            if (out[x].patch == side) {
                if (first < 0) first = static_cast<int>(x);
                ++cnt;
            }
        pa.start = first < 0 ? static_cast<int>(out.size()) : first;
        pa.count = cnt;
        m.patches.push_back(pa);
    }
    m.finalise();
    return m;
}

}  // namespace sfv
