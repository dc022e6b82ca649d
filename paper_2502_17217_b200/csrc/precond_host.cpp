// precond_host.cpp — preconditioner setup on the host (once per run, as in the reference:
// run_steps factors once and reuses the factor for every step, nonlinear.cpp:390-400).
#include "host_threads.h"
#include "device.h"
#include "precond_host.h"

#include <algorithm>
#include <thread>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <functional>
#include <numeric>

#include "sfv_case.h"

namespace sfv {

std::string cell_jacobian(const HostMesh& m, const HostGeometry& g, double kbar, bool transient, double rho,
                          double dt, std::vector<ScalarCsr>& comps) {
    const int nc = m.n_cells;
    // pattern: diagonal plus one entry per internal face side, columns sorted
    // (discretisation.cpp:223-236); built per cell from its face list, rows in parallel
    std::vector<int> rp(nc + 1, 0);
    const int nthp = host_threads();
    auto prows = [&](const std::function<void(int, int)>& body) {
        std::vector<std::thread> th;
        const int ch = (nc + nthp - 1) / nthp;
        for (int k = 0; k < nthp; ++k) th.emplace_back(body, std::min(nc, k * ch), std::min(nc, (k + 1) * ch));
        for (auto& x : th) x.join();
    };
    prows([&](int c0, int c1) {
        for (int c = c0; c < c1; ++c) {
            int k = 1;
            for (int q = m.cf_off[c]; q < m.cf_off[c + 1]; ++q) k += m.cf[q] < m.n_internal;
            rp[c + 1] = k;
        }
    });
    for (int c = 0; c < nc; ++c) rp[c + 1] += rp[c];
    rawvec<int> col(rp[nc]);
    prows([&](int c0, int c1) {
        for (int c = c0; c < c1; ++c) {
            int x = rp[c];
            col[x++] = c;
            for (int q = m.cf_off[c]; q < m.cf_off[c + 1]; ++q) {
                const int f = m.cf[q];
                if (f < m.n_internal) col[x++] = m.owner[f] == c ? m.neighbour[f] : m.owner[f];
            }
            std::sort(col.begin() + rp[c], col.begin() + rp[c + 1]);
        }
    });
    bool sym = false, coupled = false;
    auto find = [&](int i, int j) {
        return static_cast<int>(std::lower_bound(col.begin() + rp[i], col.begin() + rp[i + 1], j) - col.begin());
    };
    for (int f = m.n_internal; f < m.n_faces(); ++f)
        if (m.patches[m.face_patch[f]].kind == SFV_PATCH_SYMMETRY) {
            sym = true;
            const V3 n = g.normal[f];
            if (n.x * n.y != 0.0 || n.x * n.z != 0.0 || n.y * n.z != 0.0) coupled = true;
        }
    if (coupled) {
        // A symmetry plane that is not axis-aligned puts -coeff n (x) n with off-diagonal entries on
        // the diagonal block (discretisation.cpp:250-251), so the components do not separate: the
        // matrix is the reference's expand_scalar() (linalg.cpp:135-158) — rows 3 i + a, every
        // block all nine entries (zeros included, they are part of the ILU pattern) — with each
        // entry accumulated by the reference's own operations in its face order.
        comps.assign(1, ScalarCsr{});
        ScalarCsr& s = comps[0];
        s.n = 3 * nc;
        s.rp.assign(3 * static_cast<size_t>(nc) + 1, 0);
        for (int i = 0; i < nc; ++i)
            for (int a = 0; a < 3; ++a) s.rp[3 * i + a + 1] = 3 * (rp[i + 1] - rp[i]);
        for (int r = 0; r < 3 * nc; ++r) s.rp[r + 1] += s.rp[r];
        s.col.resize(s.rp[3 * nc]);
        s.val.resize(s.rp[3 * nc]);
        prows([&](int c0, int c1) {
            for (int i = c0; i < c1; ++i) {
                const int nb = rp[i + 1] - rp[i];
                double* row[3];
                for (int a = 0; a < 3; ++a) {
                    row[a] = s.val.data() + s.rp[3 * i + a];
                    int* cc = s.col.data() + s.rp[3 * i + a];
                    for (int k = 0; k < nb; ++k)
                        for (int b = 0; b < 3; ++b) {
                            cc[3 * k + b] = 3 * col[rp[i] + k] + b;
                            row[a][3 * k + b] = 0.0;
                        }
                }
                const int kd = find(i, i) - rp[i];
                auto add = [&](int k, double c, const double* nn) {  // block k of the row += c * M
                    for (int a = 0; a < 3; ++a)
                        for (int b = 0; b < 3; ++b)
                            row[a][3 * k + b] += (nn ? nn[a] * nn[b] : (a == b ? 1.0 : 0.0)) * c;
                };
                for (int q = m.cf_off[i]; q < m.cf_off[i + 1]; ++q) {
                    const int f = m.cf[q];
                    const double coeff = kbar * g.delta_mag[f] / g.d_mag[f] * g.area_mag[f];
                    if (f < m.n_internal) {
                        const int o = m.owner[f] == i ? m.neighbour[f] : m.owner[f];
                        add(find(i, o) - rp[i], coeff, nullptr);
                        add(kd, -coeff, nullptr);
                    } else {
                        const int kind = m.patches[m.face_patch[f]].kind;
                        if (kind == SFV_PATCH_DISPLACEMENT) {
                            add(kd, -coeff, nullptr);
                        } else if (kind == SFV_PATCH_SYMMETRY) {
                            const double nn[3] = {g.normal[f].x, g.normal[f].y, g.normal[f].z};
                            add(kd, -coeff, nn);
                        }
                    }
                }
                if (transient) add(kd, -2.25 * rho * g.volume[i] / (dt * dt), nullptr);
            }
        });
        return "";
    }
    const int ncomp = sym ? 3 : 1;
    comps.assign(ncomp, ScalarCsr{});
    for (int a = 0; a < ncomp; ++a) {
        ScalarCsr& s = comps[a];
        s.n = nc;
        s.rp = rp;
        s.col = col;
        s.val.assign(col.size(), 0.0);
        // The reference adds the face contributions face by face in ascending face order
        // (discretisation.cpp:224-262).  Every entry of row i is touched only by faces of
        // cell i, and cell_faces[i] is in ascending face order, so assembling row by row over
        // cell_faces gives every entry the same sequence of additions: rows in parallel.
        auto rows = [&](int i0, int i1) {
            for (int i = i0; i < i1; ++i) {
                for (int q = m.cf_off[i]; q < m.cf_off[i + 1]; ++q) {
                    const int f = m.cf[q];
                    // alpha is unity in the matrix (discretisation.cpp:239-240)
                    const double coeff = kbar * g.delta_mag[f] / g.d_mag[f] * g.area_mag[f];
                    if (f < m.n_internal) {
                        const int o = m.owner[f] == i ? m.neighbour[f] : m.owner[f];
                        s.val[find(i, o)] += coeff * 1.0;
                        s.val[find(i, i)] += -coeff * 1.0;
                    } else {
                        const int kind = m.patches[m.face_patch[f]].kind;
                        if (kind == SFV_PATCH_DISPLACEMENT) {
                            s.val[find(i, i)] += -coeff * 1.0;
                        } else if (kind == SFV_PATCH_SYMMETRY) {
                            const double na = a == 0 ? g.normal[f].x : (a == 1 ? g.normal[f].y : g.normal[f].z);
                            s.val[find(i, i)] += (na * na) * -coeff;
                        }
                    }
                }
                if (transient) s.val[find(i, i)] += (-2.25 * rho * g.volume[i] / (dt * dt)) * 1.0;
            }
        };
        const int nth = host_threads();
        std::vector<std::thread> th;
        const int ch = (nc + nth - 1) / nth;
        for (int k = 0; k < nth; ++k) th.emplace_back(rows, std::min(nc, k * ch), std::min(nc, (k + 1) * ch));
        for (auto& x : th) x.join();
    }
    return "";
}

namespace {

// Spin barrier for the level-synchronous host factorisation (one wait per level).
struct SpinBarrier {
    explicit SpinBarrier(int n) : count(n) {}
    void wait() {
        const int g = gen.load(std::memory_order_acquire);
        if (arrived.fetch_add(1, std::memory_order_acq_rel) == count - 1) {
            arrived.store(0, std::memory_order_relaxed);
            gen.fetch_add(1, std::memory_order_acq_rel);
        } else {
            while (gen.load(std::memory_order_acquire) == g) std::this_thread::yield();
        }
    }
    const int count;
    std::atomic<int> arrived{0}, gen{0};
};

// ILU(0) / ILU(1) with the reference's arithmetic, multi-threaded.  For level <= 1 the
// pattern of row i depends only on the original pattern (a fill entry i,j arises from
// level-0 entries i,k and k,j alone), so rows are built independently; the numeric IKJ
// phase reads only final rows k < i of row i's lower pattern, so rows run level by level
// (levels of the final lower pattern) with each row's operations in the sequential order:
// the factor is bit-identical.  Returns false on a breakdown (the caller reruns the
// sequential code for the reference's exact message).
bool iluk_factor_parallel(const ScalarCsr& a, int level, ScalarCsr& out, int nthreads, const IluNumericFn& numeric) {
    StageClock sc;
    const int n = a.n;
    // symbolic phase: each thread builds a contiguous block of rows into one flat buffer
    std::vector<int> rlen(n, 0);
    std::vector<std::vector<int>> flat(nthreads);
    const int rch = (n + nthreads - 1) / nthreads;
    auto worker_sym = [&](int t) {
        std::vector<int> mark(n, -1);
        std::vector<int> c;
        std::vector<int>& fl = flat[t];
        fl.reserve(static_cast<size_t>(a.rp[std::min(n, (t + 1) * rch)] - a.rp[std::min(n, t * rch)]) * 2);
        for (int i = t * rch; i < std::min(n, (t + 1) * rch); ++i) {
            c.assign(a.col.begin() + a.rp[i], a.col.begin() + a.rp[i + 1]);
            if (!std::binary_search(c.begin(), c.end(), i)) c.insert(std::lower_bound(c.begin(), c.end(), i), i);
            for (int j : c) mark[j] = i;
            const size_t orig = c.size();
            if (level >= 1) {
                for (size_t x = 0; x < orig && c[x] < i; ++x) {
                    const int k = c[x];
                    for (int q = a.rp[k]; q < a.rp[k + 1]; ++q) {
                        const int j = a.col[q];
                        if (j <= k || mark[j] == i) continue;
                        mark[j] = i;
                        c.push_back(j);
                    }
                }
            }
            if (c.size() > orig) std::sort(c.begin(), c.end());  // merge the fill (level 1), columns distinct
            fl.insert(fl.end(), c.begin(), c.end());
            rlen[i] = static_cast<int>(c.size());
        }
    };
    {
        std::vector<std::thread> th;
        for (int t = 0; t < nthreads; ++t) th.emplace_back(worker_sym, t);
        for (auto& t : th) t.join();
    }
    sc.mark("ilu symbolic");
    out.n = n;
    out.rp.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) out.rp[i + 1] = out.rp[i] + rlen[i];
    out.col.resize(out.rp[n]);
    out.val.resize(out.rp[n]);  // zeroed per row block below (fill entries start at 0)
    std::vector<int> diag(n, -1);
    {  // each thread places its block of rows and locates their diagonals
        std::vector<std::thread> th;
        for (int t = 0; t < nthreads; ++t)
            th.emplace_back([&, t] {
                const int i0 = std::min(n, t * rch), i1 = std::min(n, (t + 1) * rch);
                if (i0 < i1) {
                    std::copy(flat[t].begin(), flat[t].end(), out.col.begin() + out.rp[i0]);
                    std::fill(out.val.begin() + out.rp[i0], out.val.begin() + out.rp[i1], 0.0);
                }
                std::vector<int>().swap(flat[t]);
                for (int i = i0; i < i1; ++i)
                    diag[i] = static_cast<int>(std::lower_bound(out.col.begin() + out.rp[i], out.col.begin() + out.rp[i + 1], i) -
                                               out.col.begin());
            });
        for (auto& x : th) x.join();
    }
    sc.mark("ilu csr assembly");
    // levels of the final lower pattern
    std::vector<int> lev(n, 0);
    int nlev = 0;
    for (int i = 0; i < n; ++i) {
        int l = 0;
        for (int p = out.rp[i]; p < out.rp[i + 1] && out.col[p] < i; ++p) l = std::max(l, lev[out.col[p]] + 1);
        lev[i] = l;
        nlev = std::max(nlev, l + 1);
    }
    std::vector<int> lptr(nlev + 1, 0), rows(n);
    for (int i = 0; i < n; ++i) ++lptr[lev[i] + 1];
    for (int l = 0; l < nlev; ++l) lptr[l + 1] += lptr[l];
    {
        std::vector<int> fill(lptr.begin(), lptr.end() - 1);
        for (int i = 0; i < n; ++i) rows[fill[lev[i]]++] = i;
    }
    sc.mark("ilu levels");
    if (numeric) {  // A at the pattern positions (row blocks in parallel), then the device numeric phase
        std::vector<std::thread> th;
        for (int t = 0; t < nthreads; ++t)
            th.emplace_back([&, t] {
                std::vector<int> pos(n, 0);
                for (int i = std::min(n, t * rch); i < std::min(n, (t + 1) * rch); ++i) {
                    for (int q = out.rp[i]; q < out.rp[i + 1]; ++q) pos[out.col[q]] = q + 1;
                    for (int p = a.rp[i]; p < a.rp[i + 1]; ++p) out.val[pos[a.col[p]] - 1] = a.val[p];
                    for (int q = out.rp[i]; q < out.rp[i + 1]; ++q) pos[out.col[q]] = 0;
                }
            });
        for (auto& x : th) x.join();
        sc.mark("ilu scatter A");
        const bool ok = numeric(out, diag, rows);
        sc.mark("ilu numeric (device)");
        return ok;
    }
    std::atomic<bool> broke{false};
    SpinBarrier bar(nthreads);
    auto worker_num = [&](int t) {
        std::vector<int> pos(n, 0);
        for (int L = 0; L < nlev; ++L) {
            for (int x = lptr[L] + t; x < lptr[L + 1]; x += nthreads) {
                const int i = rows[x];
                // values of the original matrix at the pattern positions (fill = 0)
                for (int q = out.rp[i]; q < out.rp[i + 1]; ++q) pos[out.col[q]] = q + 1;
                for (int p = a.rp[i]; p < a.rp[i + 1]; ++p) out.val[pos[a.col[p]] - 1] = a.val[p];
                // IKJ on the fixed pattern (linalg.cpp:283-299)
                for (int p = out.rp[i]; p < out.rp[i + 1] && out.col[p] < i; ++p) {
                    const int k = out.col[p];
                    const double pivot = out.val[diag[k]];
                    if (pivot == 0.0 || !std::isfinite(pivot)) {
                        broke = true;
                        break;
                    }
                    const double lik = (out.val[p] /= pivot);
                    for (int q = out.rp[k]; q < out.rp[k + 1]; ++q) {
                        if (out.col[q] <= k) continue;
                        if (pos[out.col[q]]) out.val[pos[out.col[q]] - 1] -= lik * out.val[q];
                    }
                }
                for (int q = out.rp[i]; q < out.rp[i + 1]; ++q) pos[out.col[q]] = 0;
                const double d = out.val[diag[i]];
                if (d == 0.0 || !std::isfinite(d)) broke = true;
            }
            bar.wait();
        }
    };
    {
        std::vector<std::thread> th;
        for (int t = 0; t < nthreads; ++t) th.emplace_back(worker_num, t);
        for (auto& t : th) t.join();
    }
    sc.mark("ilu numeric");
    return !broke;
}

}  // namespace

std::string iluk_factor(const ScalarCsr& a, int level, ScalarCsr& out, const IluNumericFn& numeric) {
    const int n = a.n;
    const int nthreads = host_threads();
    if (level <= 1 && n >= 65536 && (nthreads > 1 || numeric) && !std::getenv("SFV_ILU_SERIAL") &&
        iluk_factor_parallel(a, level, out, nthreads, numeric))
        return "";
    // symbolic phase: level-of-fill row merge in ascending column order (linalg.cpp:252-269)
    out.n = n;
    out.rp.assign(n + 1, 0);
    out.col.clear();
    std::vector<int> levs;
    out.col.reserve(a.col.size() * 2);
    levs.reserve(a.col.size() * 2);
    std::vector<int> pos(n, 0), wcol, wlev;
    for (int i = 0; i < n; ++i) {
        wcol.clear();
        wlev.clear();
        for (int p = a.rp[i]; p < a.rp[i + 1]; ++p) {
            wcol.push_back(a.col[p]);
            wlev.push_back(0);
        }
        if (!std::binary_search(a.col.begin() + a.rp[i], a.col.begin() + a.rp[i + 1], i)) {
            wcol.insert(std::lower_bound(wcol.begin(), wcol.end(), i), i);
            wlev.push_back(0);
        }
        for (std::size_t x = 0; x < wcol.size(); ++x) pos[wcol[x]] = static_cast<int>(x) + 1;
        for (std::size_t it = 0; it < wcol.size() && wcol[it] < i; ++it) {
            const int k = wcol[it], lev_ik = wlev[it];
            if (lev_ik >= level) continue;
            for (int q = out.rp[k]; q < out.rp[k + 1]; ++q) {
                const int j = out.col[q];
                if (j <= k) continue;
                const int lev = lev_ik + levs[q] + 1;
                if (lev > level) continue;
                if (pos[j]) {
                    if (wlev[pos[j] - 1] > lev) wlev[pos[j] - 1] = lev;
                } else {
                    const std::size_t at = static_cast<std::size_t>(
                        std::lower_bound(wcol.begin() + it + 1, wcol.end(), j) - wcol.begin());
                    wcol.insert(wcol.begin() + at, j);
                    wlev.insert(wlev.begin() + at, lev);
                    for (std::size_t y = at; y < wcol.size(); ++y) pos[wcol[y]] = static_cast<int>(y) + 1;
                }
            }
        }
        for (std::size_t x = 0; x < wcol.size(); ++x) {
            out.col.push_back(wcol[x]);
            levs.push_back(wlev[x]);
            pos[wcol[x]] = 0;
        }
        out.rp[i + 1] = static_cast<int>(out.col.size());
    }
    out.val.assign(out.col.size(), 0.0);
    std::vector<int> diag(n, -1);
    for (int i = 0; i < n; ++i) {
        for (int q = out.rp[i]; q < out.rp[i + 1]; ++q) {
            pos[out.col[q]] = q + 1;
            if (out.col[q] == i) diag[i] = q;
        }
        for (int p = a.rp[i]; p < a.rp[i + 1]; ++p) out.val[pos[a.col[p]] - 1] = a.val[p];
        for (int q = out.rp[i]; q < out.rp[i + 1]; ++q) pos[out.col[q]] = 0;
    }
    // numeric phase, IKJ on the fixed pattern (linalg.cpp:283-299)
    for (int i = 0; i < n; ++i) {
        for (int q = out.rp[i]; q < out.rp[i + 1]; ++q) pos[out.col[q]] = q + 1;
        for (int p = out.rp[i]; p < out.rp[i + 1] && out.col[p] < i; ++p) {
            const int k = out.col[p];
            const double pivot = out.val[diag[k]];
            if (pivot == 0.0 || !std::isfinite(pivot)) {
                for (int q = out.rp[i]; q < out.rp[i + 1]; ++q) pos[out.col[q]] = 0;
                return "ilu: zero pivot in row " + std::to_string(k);
            }
            const double lik = (out.val[p] /= pivot);
            for (int q = out.rp[k]; q < out.rp[k + 1]; ++q) {
                if (out.col[q] <= k) continue;
                if (pos[out.col[q]]) out.val[pos[out.col[q]] - 1] -= lik * out.val[q];
            }
        }
        for (int q = out.rp[i]; q < out.rp[i + 1]; ++q) pos[out.col[q]] = 0;
        const double d = out.val[diag[i]];
        if (d == 0.0 || !std::isfinite(d)) return "ilu: zero pivot in row " + std::to_string(i);
    }
    return "";
}

namespace {

// rows grouped by dependency level, each level padded to a multiple of 32 positions
void pack(const std::vector<int>& level, int n_levels, TriSchedule& t,
          const std::function<void(int, std::vector<int>&, std::vector<double>&, double&)>& row_entries) {
    const int n = static_cast<int>(level.size());
    std::vector<int> count(n_levels, 0);
    for (int i = 0; i < n; ++i) ++count[level[i]];
    std::vector<int> start(n_levels + 1, 0);
    for (int l = 0; l < n_levels; ++l) start[l + 1] = start[l] + (count[l] + 31) / 32 * 32;
    t.n_pos = start[n_levels];
    t.n_levels = n_levels;
    t.level_ptr = start;
    t.order.assign(t.n_pos, -1);
    std::vector<int> fill(start.begin(), start.end() - 1);
    for (int i = 0; i < n; ++i) t.order[fill[level[i]]++] = i;
    t.rp.assign(t.n_pos + 1, 0);
    t.diag.assign(t.n_pos, 1.0);
    // rows gathered by position ranges in parallel, then concatenated in position order
    const int nthr = host_threads();
    const int pchunk = (t.n_pos + nthr - 1) / nthr;
    std::vector<std::vector<int>> pc(nthr);
    std::vector<std::vector<double>> pv(nthr);
    {
        std::vector<std::thread> th;
        for (int k = 0; k < nthr; ++k)
            th.emplace_back([&, k] {
                std::vector<int> c;
                std::vector<double> v;
                for (int p = std::min(t.n_pos, k * pchunk); p < std::min(t.n_pos, (k + 1) * pchunk); ++p) {
                    const int i = t.order[p];
                    if (i >= 0) {
                        c.clear();
                        v.clear();
                        double d = 1.0;
                        row_entries(i, c, v, d);
                        pc[k].insert(pc[k].end(), c.begin(), c.end());
                        pv[k].insert(pv[k].end(), v.begin(), v.end());
                        t.diag[p] = d;
                        t.rp[p + 1] = static_cast<int>(c.size());
                    }
                }
            });
        for (auto& x : th) x.join();
    }
    StageClock sc;
    for (int p = 0; p < t.n_pos; ++p) t.rp[p + 1] += t.rp[p];
    t.col.resize(t.rp[t.n_pos]);
    t.val.resize(t.rp[t.n_pos]);
    t.pos.assign(n, -1);
    std::vector<int> maxd(nthr, 0);
    {  // each thread places its own position range (and its rows' positions)
        std::vector<std::thread> th;
        for (int k = 0; k < nthr; ++k)
            th.emplace_back([&, k] {
                const int p0 = std::min(t.n_pos, k * pchunk), p1 = std::min(t.n_pos, (k + 1) * pchunk);
                std::copy(pc[k].begin(), pc[k].end(), t.col.begin() + t.rp[p0]);
                std::copy(pv[k].begin(), pv[k].end(), t.val.begin() + t.rp[p0]);
                std::vector<int>().swap(pc[k]);
                std::vector<double>().swap(pv[k]);
                for (int p = p0; p < p1; ++p) {
                    maxd[k] = std::max(maxd[k], t.rp[p + 1] - t.rp[p]);
                    if (t.order[p] >= 0) t.pos[t.order[p]] = p;
                }
            });
        for (auto& x : th) x.join();
    }
    t.maxd = *std::max_element(maxd.begin(), maxd.end());
    const size_t ne = static_cast<size_t>(t.maxd) * t.n_pos;
    // ELL transposition: entry k of position p at k * n_pos + p (padding -1 / 0); threads own
    // position ranges and write every slot of them, so the arrays need no prior fill
    t.ell_col.resize(ne);
    t.ell_val.resize(ne);
    t.ell_pcol.resize(ne);
    sc.mark("pack concat + pos");
    const int nth = host_threads();
    auto ell = [&](int p0, int p1) {
        for (int p = p0; p < p1; ++p) {
            const int b = t.rp[p], len = t.rp[p + 1] - b;
            for (int k = 0; k < t.maxd; ++k) {
                const size_t x = static_cast<size_t>(k) * t.n_pos + p;
                if (k < len) {
                    t.ell_col[x] = t.col[b + k];
                    t.ell_val[x] = t.val[b + k];
                    t.ell_pcol[x] = t.pos[t.col[b + k]];
                } else {
                    t.ell_col[x] = -1;
                    t.ell_val[x] = 0.0;
                    t.ell_pcol[x] = -1;
                }
            }
        }
    };
    std::vector<std::thread> th;
    const int chunk = (t.n_pos + nth - 1) / nth;
    for (int k = 0; k < nth; ++k) th.emplace_back(ell, std::min(t.n_pos, k * chunk), std::min(t.n_pos, (k + 1) * chunk));
    for (auto& x : th) x.join();
    sc.mark("pack ell");
}

}  // namespace

void schedule_lower(const ScalarCsr& lu, TriSchedule& t) {
    StageClock sc;
    const int n = lu.n;
    std::vector<int> level(n, 0);
    int n_levels = 0;
    for (int i = 0; i < n; ++i) {
        int l = 0;
        for (int p = lu.rp[i]; p < lu.rp[i + 1] && lu.col[p] < i; ++p) l = std::max(l, level[lu.col[p]] + 1);
        level[i] = l;
        n_levels = std::max(n_levels, l + 1);
    }
    sc.mark("lower levels");
    // forward row: entries col < i in ascending column order (linalg.cpp:304-306)
    pack(level, n_levels, t, [&](int i, std::vector<int>& c, std::vector<double>& v, double&) {
        for (int p = lu.rp[i]; p < lu.rp[i + 1] && lu.col[p] < i; ++p) {
            c.push_back(lu.col[p]);
            v.push_back(lu.val[p]);
        }
    });
}

bool ic0_factor(const ScalarCsr& a, ScalarCsr& L) {
    const int n = a.n;
    L.n = n;
    L.rp.assign(n + 1, 0);
    L.col.clear();
    L.val.clear();
    for (int i = 0; i < n; ++i) {
        for (int p = a.rp[i]; p < a.rp[i + 1]; ++p)
            if (a.col[p] <= i) {
                L.col.push_back(a.col[p]);
                L.val.push_back(a.val[p]);
            }
        L.rp[i + 1] = static_cast<int>(L.col.size());
    }
    const std::vector<int>& rp = L.rp;
    const auto& col = L.col;
    auto& val = L.val;
    for (int i = 0; i < n; ++i) {
        const int diag_p = rp[i + 1] - 1;
        if (diag_p < rp[i] || col[diag_p] != i) return false;
        for (int p = rp[i]; p < diag_p; ++p) {
            const int j = col[p];
            double s = val[p];
            int pi = rp[i], pj = rp[j];
            while (pi < p && pj < rp[j + 1] - 1) {
                if (col[pi] == col[pj]) s -= val[pi++] * val[pj++];
                else if (col[pi] < col[pj]) ++pi;
                else ++pj;
            }
            val[p] = s / val[rp[j + 1] - 1];
        }
        double s = val[diag_p];
        for (int p = rp[i]; p < diag_p; ++p) s -= val[p] * val[p];
        if (!(s > 0.0)) return false;
        val[diag_p] = std::sqrt(s);
    }
    return true;
}

void schedule_ic0(const ScalarCsr& L, TriSchedule& fwd, TriSchedule& bwd) {
    const int n = L.n;
    // forward: level of row i from its columns j < i
    std::vector<int> level(n, 0);
    int nl = 0;
    for (int i = 0; i < n; ++i) {
        int l = 0;
        for (int p = L.rp[i]; p < L.rp[i + 1] - 1; ++p) l = std::max(l, level[L.col[p]] + 1);
        level[i] = l;
        nl = std::max(nl, l + 1);
    }
    pack(level, nl, fwd, [&](int i, std::vector<int>& c, std::vector<double>& v, double& d) {
        for (int p = L.rp[i]; p < L.rp[i + 1] - 1; ++p) {
            c.push_back(L.col[p]);
            v.push_back(L.val[p]);
        }
        d = L.val[L.rp[i + 1] - 1];
    });
    // backward: row i of L^T holds L_ji for j > i; the saxpy loop subtracts them from z_i in
    // descending j, then divides by L_ii (linalg.cpp:213-216)
    std::vector<int> tp(n + 1, 0);
    for (int j = 0; j < n; ++j)
        for (int p = L.rp[j]; p < L.rp[j + 1] - 1; ++p) ++tp[L.col[p] + 1];
    for (int i = 0; i < n; ++i) tp[i + 1] += tp[i];
    std::vector<int> tcol(tp[n]);
    std::vector<double> tval(tp[n]);
    {
        std::vector<int> fill(tp.begin(), tp.end() - 1);
        for (int j = n - 1; j >= 0; --j)  // descending j within each row of L^T
            for (int p = L.rp[j]; p < L.rp[j + 1] - 1; ++p) {
                const int i = L.col[p];
                tcol[fill[i]] = j;
                tval[fill[i]++] = L.val[p];
            }
    }
    std::vector<int> lev2(n, 0);
    int nl2 = 0;
    for (int i = n - 1; i >= 0; --i) {
        int l = 0;
        for (int q = tp[i]; q < tp[i + 1]; ++q) l = std::max(l, lev2[tcol[q]] + 1);
        lev2[i] = l;
        nl2 = std::max(nl2, l + 1);
    }
    pack(lev2, nl2, bwd, [&](int i, std::vector<int>& c, std::vector<double>& v, double& d) {
        for (int q = tp[i]; q < tp[i + 1]; ++q) {
            c.push_back(tcol[q]);
            v.push_back(tval[q]);
        }
        d = L.val[L.rp[i + 1] - 1];
    });
}

void schedule_upper(const ScalarCsr& lu, TriSchedule& t) {
    const int n = lu.n;
    std::vector<int> level(n, 0);
    int n_levels = 0;
    for (int i = n - 1; i >= 0; --i) {
        int l = 0;
        for (int p = lu.rp[i + 1] - 1; p >= lu.rp[i] && lu.col[p] > i; --p) l = std::max(l, level[lu.col[p]] + 1);
        level[i] = l;
        n_levels = std::max(n_levels, l + 1);
    }
    // backward row: entries col > i in descending column order, then the pivot (linalg.cpp:307-314)
    pack(level, n_levels, t, [&](int i, std::vector<int>& c, std::vector<double>& v, double& d) {
        d = 0.0;
        for (int p = lu.rp[i + 1] - 1; p >= lu.rp[i] && lu.col[p] >= i; --p) {
            if (lu.col[p] == i)
                d = lu.val[p];
            else {
                c.push_back(lu.col[p]);
                v.push_back(lu.val[p]);
            }
        }
    });
}

std::string band_cholesky_neg(const ScalarCsr& a, BandChol& out, bool factor) {
    const int n = a.n;
    // reverse Cuthill-McKee ordering of the symmetric pattern
    std::vector<int> deg(n);
    for (int i = 0; i < n; ++i) deg[i] = a.rp[i + 1] - a.rp[i];
    std::vector<int> by_deg(n);
    std::iota(by_deg.begin(), by_deg.end(), 0);
    std::stable_sort(by_deg.begin(), by_deg.end(), [&](int x, int y) { return deg[x] < deg[y]; });
    std::vector<char> seen(n, 0);
    std::vector<int> order;
    order.reserve(n);
    std::vector<int> nb;
    for (int s0 : by_deg) {
        if (seen[s0]) continue;
        const std::size_t base = order.size();
        order.push_back(s0);
        seen[s0] = 1;
        for (std::size_t h = base; h < order.size(); ++h) {
            const int u = order[h];
            nb.clear();
            for (int p = a.rp[u]; p < a.rp[u + 1]; ++p)
                if (!seen[a.col[p]] && a.val[p] != 0.0) {
                    seen[a.col[p]] = 1;
                    nb.push_back(a.col[p]);
                }
            std::stable_sort(nb.begin(), nb.end(), [&](int x, int y) { return deg[x] < deg[y]; });
            order.insert(order.end(), nb.begin(), nb.end());
        }
    }
    std::reverse(order.begin(), order.end());
    auto bandwidth = [&](const std::vector<int>& inv_) {
        int b = 0;
        for (int i = 0; i < n; ++i)
            for (int p = a.rp[i]; p < a.rp[i + 1]; ++p)
                if (a.val[p] != 0.0) b = std::max(b, std::abs(inv_[i] - inv_[a.col[p]]));
        return b;
    };
    std::vector<int> inv(n), ident(n);
    for (int i = 0; i < n; ++i) inv[order[i]] = i;
    std::iota(ident.begin(), ident.end(), 0);
    int bw = bandwidth(inv);
    if (const int bw0 = bandwidth(ident); bw0 <= bw) {  // keep the natural order when it is as narrow
        bw = bw0;
        order = ident;
        inv = ident;
    }
    out.n = n;
    out.bw = bw;
    out.perm = order;
    const int w = bw + 1;
    out.l.assign(static_cast<std::size_t>(n) * w, 0.0);
    auto L = [&](int i, int j) -> double& { return out.l[static_cast<std::size_t>(i) * w + (j - i + bw)]; };
    for (int i = 0; i < n; ++i)
        for (int p = a.rp[i]; p < a.rp[i + 1]; ++p) {
            const int bi = inv[i], bj = inv[a.col[p]];
            // -A is symmetric positive definite (explicit zeros of an expanded block pattern are
            // outside the band computed above and stay out)
            if (bj <= bi && a.val[p] != 0.0) L(bi, bj) = -a.val[p];
        }
    if (!factor) return "";
    for (int i = 0; i < n; ++i) {
        const int j0 = std::max(0, i - bw);
        for (int j = j0; j < i; ++j) {
            double s = L(i, j);
            const int k0 = std::max(j0, std::max(0, j - bw));
            for (int k = k0; k < j; ++k) s -= L(i, k) * L(j, k);
            L(i, j) = s / L(j, j);
        }
        double d = L(i, i);
        for (int k = j0; k < i; ++k) d -= L(i, k) * L(i, k);
        if (!(d > 0.0) || !std::isfinite(d)) return "lu: factorisation failed";
        L(i, i) = std::sqrt(d);
    }
    return "";
}

}  // namespace sfv

namespace sfv {

bool build_stream_records(const TriSchedule& t, int cs, int ring, int max_rows, rawvec<unsigned char>& packed,
                          const std::vector<int>* out_pos) {
    StageClock sc;
    if (t.maxd > 8 || ring > 4095) return false;  // slot index ring (12 bits) is the +0.0 slot
    const int np = t.n_pos;
    std::vector<int> owner(np, 0), ordinal(np, 0), level_of(np, 0);
    std::vector<int> count(cs, 0);
    std::vector<std::vector<int>> ord_level(cs);  // per CTA: level of its k-th position
    for (int l = 0; l < t.n_levels; ++l) {
        const int a = t.level_ptr[l], b = t.level_ptr[l + 1];
        const int nch = (b - a) / 32, per = (nch + cs - 1) / cs;
        if (per * 32 > max_rows) return false;
        for (int p = a; p < b; ++p) {
            const int r = ((p - a) / 32) / std::max(per, 1);
            owner[p] = r;
            ordinal[p] = count[r]++;
            ord_level[r].push_back(l);
            level_of[p] = l;
        }
    }
    sc.mark("records owners");
    // device chunk layout (device.h kStream*): per 32 positions val[8][32], diag[32], dep[8][32],
    // own[32], out[32]; positions are whole chunks (levels padded to 32), every byte written below
    const size_t nchunk = (static_cast<size_t>(np) + 31) / 32;
    packed.resize(nchunk * kChunkBytes);
    sc.mark("records alloc");
    long long n_dep = 0, n_local = 0, n_near = 0, n_near_remote = 0;
    // positions are independent: threads own position ranges; statistics only when asked
    const bool stats = std::getenv("SFV_STREAM_STATS") != nullptr;
    const int nthr = stats ? 1 : host_threads();
    std::atomic<bool> bad{false};
    auto body = [&](int c0, int c1) {  // chunk ranges
    for (int ch = c0; ch < c1 && !bad; ++ch) {
        unsigned char* cb = packed.data() + static_cast<size_t>(ch) * kChunkBytes;
        double* cval = reinterpret_cast<double*>(cb);
        double* cdiag = reinterpret_cast<double*>(cb + kStreamOffDiag);
        uint32_t* cdep = reinterpret_cast<uint32_t*>(cb + kStreamOffDep);
        uint16_t* cown = reinterpret_cast<uint16_t*>(cb + kStreamOffOwn);
        int32_t* cout = reinterpret_cast<int32_t*>(cb + kStreamOffOut);
        std::memset(cb + kStreamOffEnd, 0, kChunkBytes - kStreamOffEnd);
    for (int l = 0; l < 32; ++l) {
        const int p = ch * 32 + l;
        if (p >= np) {  // tail: no dependencies
            for (int k = 0; k < 8; ++k) {
                cval[k * 32 + l] = 0.0;
                cdep[k * 32 + l] = stream_dep(0, ring);  // rank 0's +0.0 slot
            }
            cdiag[l] = 0.0;
            cown[l] = 0;
            cout[l] = -1;
            continue;
        }
        cown[l] = static_cast<uint16_t>(ordinal[p] % ring);
        // where the sweep stores this position's value: the row (backward sweep), or the row's
        // backward-sweep position (forward sweep, out_pos = that schedule's row -> position)
        cout[l] = t.order[p] < 0 ? -1 : out_pos ? (*out_pos)[t.order[p]] : t.order[p];
        cdiag[l] = t.diag[p];
        for (int k = 0; k < 8; ++k) {
            // an absent dependency reads the +0.0 slot of the reading CTA's ring
            cdep[k * 32 + l] = stream_dep(owner[p], ring);
            cval[k * 32 + l] = 0.0;
            if (k >= t.maxd) continue;
            const int q = t.ell_pcol[static_cast<size_t>(k) * np + p];
            if (q < 0) continue;
            // the slot of q is rewritten by its owner's (ordinal + ring)-th position: that
            // position must lie in a strictly later level than the reader p
            const int r = owner[q], o = ordinal[q] + ring;
            if (o < static_cast<int>(ord_level[r].size()) && ord_level[r][o] <= level_of[p]) {
                bad = true;
                return;
            }
            cdep[k * 32 + l] = stream_dep(r, ordinal[q] % ring);
            cval[k * 32 + l] = t.ell_val[static_cast<size_t>(k) * np + p];
            if (stats) {
                ++n_dep;
                if (r == owner[p]) ++n_local;
                if (level_of[q] == level_of[p] - 1) {
                    ++n_near;
                    if (r != owner[p]) ++n_near_remote;
                }
            }
        }
    }
    }
    };
    {
        std::vector<std::thread> th;
        const int nch = static_cast<int>(nchunk);
        const int ch = (nch + nthr - 1) / nthr;
        for (int k = 0; k < nthr; ++k) th.emplace_back(body, std::min(nch, k * ch), std::min(nch, (k + 1) * ch));
        for (auto& x : th) x.join();
    }
    if (bad) return false;
    if (std::getenv("SFV_STREAM_STATS"))
        std::fprintf(stderr,
                     "stream records: %d positions, %d levels, %lld deps, %.1f%% in the reading CTA, %.1f%% from the "
                     "previous level (%.1f%% of all deps: previous level and another CTA)\n",
                     np, t.n_levels, n_dep, 100.0 * n_local / std::max(1LL, n_dep),
                     100.0 * n_near / std::max(1LL, n_dep), 100.0 * n_near_remote / std::max(1LL, n_dep));
    return true;
}

bool build_pipe(const ScalarCsr& lu, bool upper, int blocks, int ring, PipeSchedule& out, std::string* why) {
    auto fail = [&](const char* m) {
        if (why) *why = m;
        return false;
    };
    const int n = lu.n;
    if (n < blocks || ring <= 0 || (ring & (ring - 1))) return fail("pipe: bad size");
    // dependencies of row i in the reference's order (linalg.cpp:302-316)
    auto entries = [&](int i, std::vector<int>& c, std::vector<double>& v, double& d) {
        c.clear();
        v.clear();
        d = 1.0;
        if (!upper) {
            for (int p = lu.rp[i]; p < lu.rp[i + 1] && lu.col[p] < i; ++p) {
                c.push_back(lu.col[p]);
                v.push_back(lu.val[p]);
            }
        } else {
            d = 0.0;
            for (int p = lu.rp[i + 1] - 1; p >= lu.rp[i] && lu.col[p] >= i; --p) {
                if (lu.col[p] == i)
                    d = lu.val[p];
                else {
                    c.push_back(lu.col[p]);
                    v.push_back(lu.val[p]);
                }
            }
        }
    };
    // sweep order k -> row, global dependency levels, blocks
    auto row_at = [&](int k) { return upper ? n - 1 - k : k; };
    std::vector<int> level(n, 0), blk(n);
    std::vector<int> c;
    std::vector<double> v;
    double d;
    for (int k = 0; k < n; ++k) {
        const int i = row_at(k);
        blk[i] = static_cast<int>(static_cast<long long>(k) * blocks / n);
        entries(i, c, v, d);
        if (c.size() > 8) return fail("pipe: more than 8 dependencies in a row");
        int l = 0;
        for (int j : c) {
            l = std::max(l, level[j] + 1);
            if (blk[j] != blk[i] && blk[j] != blk[i] - 1) return fail("pipe: dependency beyond the previous block");
        }
        level[i] = l;
    }
    // per block: rows by (level, sweep order); steps = distinct levels
    out = PipeSchedule{};
    out.blocks = blocks;
    out.ring = ring;
    std::vector<std::vector<int>> rows_of(blocks);
    for (int k = 0; k < n; ++k) rows_of[blk[row_at(k)]].push_back(row_at(k));
    std::vector<int> step(n, 0);
    out.step_off.assign(blocks + 1, 0);
    std::vector<int> block_start(blocks + 1, 0);
    int npos = 0;
    for (int b = 0; b < blocks; ++b) {
        std::vector<int>& rs = rows_of[b];
        std::stable_sort(rs.begin(), rs.end(), [&](int x, int y) { return level[x] < level[y]; });
        block_start[b] = npos;
        int nsteps = 0;
        for (size_t x = 0; x < rs.size();) {
            size_t y = x;
            while (y < rs.size() && level[rs[y]] == level[rs[x]]) ++y;
            out.step_ptr.push_back(npos);
            for (size_t q = x; q < y; ++q) step[rs[q]] = nsteps;
            const int cnt = static_cast<int>(y - x);
            out.max_rows = std::max(out.max_rows, cnt);
            for (size_t q = x; q < y; ++q) out.order.push_back(rs[q]);
            const int padded = (cnt + 31) / 32 * 32;
            for (int q = cnt; q < padded; ++q) out.order.push_back(-1);
            npos += padded;
            ++nsteps;
            x = y;
        }
        out.step_ptr.push_back(npos);
        out.step_off[b + 1] = out.step_off[b] + nsteps;
    }
    block_start[blocks] = npos;
    out.n_pos = npos;
    if (out.max_rows > ring / 2) return fail("pipe: ring smaller than two steps");
    out.pos.assign(n, -1);
    std::vector<int> pblk(npos), pstep(npos);
    for (int b = 0; b < blocks; ++b)
        for (int s = 0; s < out.step_off[b + 1] - out.step_off[b]; ++s) {
            const int i0 = out.step_off[b] + b + s;
            for (int p = out.step_ptr[i0]; p < out.step_ptr[i0 + 1]; ++p) {
                pblk[p] = b;
                pstep[p] = s;
            }
        }
    for (int p = 0; p < npos; ++p)
        if (out.order[p] >= 0) out.pos[out.order[p]] = p;
    const int total = out.step_off[blocks];
    out.need.assign(total, 0);
    out.guard.assign(total, 0);
    // last reader step (in block b + 1) of every position read remotely
    std::vector<int> last_remote(npos, -1);
    out.rec.assign(static_cast<size_t>(npos / 32) * kPipeChunkBytes, 0);
    for (int p = 0; p < npos; ++p) {
        unsigned char* ch = out.rec.data() + static_cast<size_t>(p / 32) * kPipeChunkBytes;
        const int ln = p % 32;
        const uint32_t none = 0xffffffffu;
        for (int q = 0; q < 8; ++q) std::memcpy(ch + 2304 + (q * 32 + ln) * 4, &none, 4);
        const int i = out.order[p];
        if (i < 0) continue;
        entries(i, c, v, d);
        std::memcpy(ch + 2048 + ln * 8, &d, 8);
        const int b = pblk[p], s = pstep[p];
        for (size_t q = 0; q < c.size(); ++q) {
            const int pj = out.pos[c[q]];
            const int bj = pblk[pj];
            const uint32_t slot = static_cast<uint32_t>(pj - block_start[bj]) & static_cast<uint32_t>(ring - 1);
            // local reuse: the slot is rewritten by position pj + ring of block bj
            const int over = pj + ring;
            if (over < block_start[bj + 1] && bj == b && pstep[over] <= s) return fail("pipe: ring too small (local)");
            const uint32_t dep = bj == b ? slot : (slot | 0x80000000u);
            std::memcpy(ch + 2304 + (q * 32 + ln) * 4, &dep, 4);
            std::memcpy(ch + (q * 32 + ln) * 8, &v[q], 8);
            if (bj != b) {
                out.need[out.step_off[b] + s] = std::max(out.need[out.step_off[b] + s], pstep[pj] + 1);
                last_remote[pj] = std::max(last_remote[pj], s);
            }
        }
    }
    for (int b = 0; b + 1 < blocks; ++b)
        for (int p = block_start[b]; p < block_start[b + 1]; ++p) {
            if (last_remote[p] < 0) continue;
            const int over = p + ring;  // rewritten by this position of block b
            if (over >= block_start[b + 1]) continue;
            int& g = out.guard[out.step_off[b] + pstep[over]];
            g = std::max(g, last_remote[p] + 1);
        }
    for (int b = 0; b < blocks; ++b)
        for (int s = out.step_off[b] + 1; s < out.step_off[b + 1]; ++s) {
            out.need[s] = std::max(out.need[s], out.need[s - 1]);
            out.guard[s] = std::max(out.guard[s], out.guard[s - 1]);
        }
    return true;
}


}  // namespace sfv
