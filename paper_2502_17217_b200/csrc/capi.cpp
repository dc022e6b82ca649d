// capi.cpp — libsfv.so: context, device layout, preconditioner setup and the
// device-resident GMRES / JFNK / stepping drivers behind the C-ABI of include/sfv.h.
//
// Control flow restates the reference line for line (cited per function); all vector
// work stays on the device, and the host sees only the scalars the reference's control
// decisions need (norms, Hessenberg columns) — one small D2H per Arnoldi step.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "host_threads.h"
#include "device.h"
#include "host_mesh.h"
#include "precond_dev.h"
#include "precond_host.h"
#include "sfv.h"

using namespace sfv;

namespace {

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    bool alloc(size_t count) {
        release();
        n = count;
        if (count == 0) return true;
        return cudaMalloc(&p, sizeof(T) * count) == cudaSuccess;
    }
    template <class A>
    bool upload(const std::vector<T, A>& h) {
        if (!alloc(h.size())) return false;
        return h.empty() || cudaMemcpy(p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice) == cudaSuccess;
    }
    size_t bytes() const { return sizeof(T) * n; }
    void adopt(T* q, size_t count) {  // take ownership of a cudaMalloc'd array
        release();
        p = q;
        n = count;
    }
};

struct Status {  // pinned host mirror of the device scalars read per control decision
    ErrWords err;
    double* h;  // pinned, hcap doubles: the Hessenberg column of an Arnoldi step (restart + 2)
    int hcap;
};

struct TriDev {
    DevBuf<int> order, rp, col, level_ptr, ell_col, ell_pcol, u2l;
    DevBuf<double> val, diag, ell_val;
    DevTri view;
    int n_levels = 0;
    size_t nnz = 0;
    // full = false: only the position map and level pointers (all the streamed sweep reads)
    bool upload(const TriSchedule& t, int n_rows, bool full) {
        bool ok = order.upload(t.order) && level_ptr.upload(t.level_ptr);
        if (full)
            ok = ok && rp.upload(t.rp) && col.upload(t.col) && val.upload(t.val) && diag.upload(t.diag) &&
                 ell_col.upload(t.ell_col) && ell_val.upload(t.ell_val) && ell_pcol.upload(t.ell_pcol);
        view.ell_pcol = ell_pcol.p;
        view.level_ptr = level_ptr.p;
        view.maxd = t.maxd;
        view.ell_col = ell_col.p;
        view.ell_val = ell_val.p;
        view.n = t.n_pos;
        view.n_rows = n_rows;
        view.n_levels = t.n_levels;
        view.order = order.p;
        view.rp = rp.p;
        view.col = col.p;
        view.val = val.p;
        view.diag = diag.p;
        n_levels = t.n_levels;
        nnz = t.col.size();
        return ok;
    }
};

struct SfvError {
    int code;
    int cell;
    std::string msg;
};

}  // namespace

struct sfv_mesh {
    HostMesh m;
    bool on_device = false;  // built by a device generator
};

struct sfv_ctx {
    HostMesh mesh;
    HostGeometry geom;
    int nc = 0, n = 0;
    int singular_cell = -1;
    DevMesh dm;
    Physics ph{};
    PatchTable pt{};
    std::vector<double> bc_raw;  // per patch, unscaled
    std::vector<int> bc_ramp;
    double time = 0.0;
    cudaStream_t stream = nullptr;
    // owned layout buffers
    // bnd_si: per boundary face, slot index s * nc + cell (alternative paths) or cell * 8 + s (default)
    DevBuf<int> slot_face, slot_other, bnd_si, tslot;
    DevBuf<double> slot_ls, gam, del, dmag, w, volume, tls;
    // jv_pair.cu scratch + tiled face records (device.h): pwg = tiled [w | G], psig: tiled cell stress
    DevBuf<double> pwg, face9, bres, psig, lawst;
    DeviceGeometry* dgeo = nullptr;  // device-resident geometry (the host copy is partial until host_geometry())
    // segregated solver (per component: A = -J~, IC(0) sweeps or the Jacobi fallback)
    struct SegComp {
        DevBuf<int> rp, col, f_order, f_rp, f_col, b_order, b_rp, b_col;
        DevBuf<double> val, f_val, f_diag, b_val, b_diag, inv_diag;
        SegCsr a;
        SegSweep fwd, bwd;
        bool jacobi = false;
    };
    SegComp seg[3];
    int seg_ncomp = 0;
    DevBuf<double> sg_b, sg_x, sg_r, sg_z, sg_p, sg_ap, sg_y, sg_un, sg_du;
    PairScratch ps;
    // scratch
    DevBuf<double> grad, red, scal;  // scal: [0]=eps [1]=u_norm [2..] misc
    DevBuf<unsigned> counter;
    DevBuf<unsigned long long> epsbar;  // grid-barrier counter of eps_perturb_kernel
    DevBuf<ErrWords> err;
    Status* st = nullptr;  // pinned
    History hist{};
    DevBuf<double> hist_own;  // zero history when none supplied
    // preconditioner
    int pc_kind = SFV_PRECOND_NONE;
    int pc_ncomp = 1;
    bool pc_coupled = false;  // one factor over all 3n unknowns (symmetry plane not axis-aligned)
    TriDev L[3], U[3];
    DevBuf<double> ily, ipa, ipb;  // forward-sweep scratch, position-space scratch
    int tri_grid = 0;
    int tri_sleep = 0;
    int tri_cluster = 16;
    bool ring_ok = false;
    bool stream_ok = false;
    StreamSet sL{}, sU{};
    bool pipe_ok = false;
    PipeSet pL{}, pU{};
    DevBuf<int> pint[6 * 6];          // per (component, sweep): step_off, step_ptr, need, guard, order, to_lower
    DevBuf<unsigned char> prec[6];    // per (component, sweep) records
    DevBuf<unsigned char> srec[6];  // streamed-sweep records: L0..L2, U0..U2
    DevBuf<double> dense_w[3];
    DevBuf<int> dense_perm[3];
    // residual / J.v kernels: 0 = jv_pair.cu (default), 1 = jv_fused.cu, 2 = residual.cu
    int jv_path = 0;
    bool use_fused = false;
    // body force and per-face boundary values (DiscretisationConfig::body_force,
    // BoundaryCondition::value sampled at the face centroids)
    DevBuf<double> body_dev, face_bc_dev;
    std::vector<double> face_bc_host;
    sfv_bc_sampler bc_sampler = nullptr;
    void* bc_user = nullptr;
    // run_steps' StepCallback (nonlinear.hpp:106-107): the field on the host after every step
    sfv_step_callback step_fn = nullptr;
    void* step_user = nullptr;
    std::vector<double> step_field;
    FusedLayout fl;
    DevBuf<int> f_tfp, f_own, f_oth, f_slots, f_index, f_flags, f_ticket;
    DevBuf<double> f_geo, f_gring, f_fring;
    int f_epoch = 0, f_grid = 0;
    // krylov workspace
    DevBuf<double> V, wv, rv, tv, xv, bv, hdev, ydev, ucand, rcand, uscratch, rscratch, dzero;
    int v_cap = 0;
    // device-resident GMRES cycle (gmres_graph): one CUDA graph whose WHILE node runs the
    // Arnoldi steps of a restart cycle (J.v, preconditioner, MGS, Givens) without the host
    DevBuf<unsigned char> gstate;
    unsigned char* gstate_host = nullptr;  // pinned mirror
    GmresDev gdev{};
    int g_cap = 0;  // restart the state is sized for
    cudaStream_t gstream = nullptr;
    cudaEvent_t gev0 = nullptr, gev1 = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    std::vector<unsigned char> g_key;  // everything the graph captured by value (gmres_graph_key)
    long long pc_gen = 0;              // bumped by every preconditioner (re)build
    long long g_launches = 0;  // kernels per Arnoldi step in the graph
    bool graph_broken = false;
    bool graph_off = false;  // sfv_set_option("gmres_graph", 0)
    // sfv_set_option("sequential_reductions", 1) / SFV_SEQ_REDUCE=1: every inner product and
    // norm summed left to right as the reference does (launch_seq_dot), so the Krylov and Newton
    // decisions are bit-identical to the CPU reference's; ~13 ms per 3M-term sum
    bool seq_reduce = [] {
        const char* e = std::getenv("SFV_SEQ_REDUCE");
        return e && std::atoi(e) != 0;
    }();
    bool vsel_failed = false;
    long long launches = 0;
    SfvError last{0, -1, ""};
    // host-buffer J.v: r_u uploaded on a copy stream while the ε and gradient passes run
    cudaStream_t copy = nullptr;
    cudaEvent_t ev_uv = nullptr, ev_ru = nullptr;
    // chunked host-buffer J.v: r_u arrives in kHostChunks pieces, the face pass runs per piece
    // and each piece of the result leaves on d2h while the next is computed
    static constexpr int kHostChunks = 16;  // at most (SFV_JV_HOST_CHUNKS, default 8)
    cudaStream_t d2h = nullptr;
    cudaEvent_t ev_ruk[kHostChunks] = {}, ev_outk[kHostChunks] = {};
    void drop_graph() {
        if (gexec) cudaGraphExecDestroy(gexec);
        if (graph) cudaGraphDestroy(graph);
        gexec = nullptr;
        graph = nullptr;
        g_key.clear();
    }
    ~sfv_ctx() {
        drop_graph();
        if (gstate_host) cudaFreeHost(gstate_host);
        if (gev0) cudaEventDestroy(gev0);
        if (gev1) cudaEventDestroy(gev1);
        if (gstream) cudaStreamDestroy(gstream);
        free_device_geometry(dgeo);
        if (ps.ev_w) cudaEventDestroy(ps.ev_w);
        if (ps.ev_b) cudaEventDestroy(ps.ev_b);
        if (ps.side) cudaStreamDestroy(ps.side);
        if (ev_uv) cudaEventDestroy(ev_uv);
        if (ev_ru) cudaEventDestroy(ev_ru);
        if (copy) cudaStreamDestroy(copy);
        for (int k = 0; k < kHostChunks; ++k) {
            if (ev_ruk[k]) cudaEventDestroy(ev_ruk[k]);
            if (ev_outk[k]) cudaEventDestroy(ev_outk[k]);
        }
        if (d2h) cudaStreamDestroy(d2h);
    }

    int fail(int code, int cell, const std::string& msg) {
        last = {code, cell, msg};
        return code;
    }
    int cuda_check(const char* where) {
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail(SFV_ERR_CUDA, -1, std::string(where) + ": " + cudaGetErrorString(e));
        return SFV_OK;
    }
};

namespace {

constexpr int kNone = 0x7f7f7f7f;

int upload_face_values(sfv_ctx* c, const double* v);

int update_patch_values(sfv_ctx* c) {
    // config-built BC: ramp ? v * t : v (io.cpp:278-279)
    for (int p = 0; p < c->pt.n; ++p)
        for (int k = 0; k < 3; ++k)
            c->pt.value[p][k] = c->bc_ramp[p] ? c->bc_raw[3 * p + k] * c->time : c->bc_raw[3 * p + k];
    if (c->bc_sampler) {  // BoundaryCondition::value(face_centroid, t) for every boundary face
        c->face_bc_host.assign(3 * static_cast<size_t>(c->mesh.n_faces() - c->mesh.n_internal), 0.0);
        c->bc_sampler(c->bc_user, c->time, c->face_bc_host.data());
        return upload_face_values(c, c->face_bc_host.data());
    }
    return SFV_OK;
}

// per boundary face values on the device (null: the patch table)
int upload_face_values(sfv_ctx* c, const double* v) {
    if (!v) {
        c->pt.face_value = nullptr;
        return SFV_OK;
    }
    const size_t nb = 3 * static_cast<size_t>(c->mesh.n_faces() - c->mesh.n_internal);
    if (c->face_bc_dev.n != nb && !c->face_bc_dev.alloc(nb)) return c->fail(SFV_ERR_CUDA, -1, "out of device memory");
    // ordered on the context stream: earlier kernels still reading the old values finish first
    cudaStreamSynchronize(c->stream);
    if (nb && cudaMemcpy(c->face_bc_dev.p, v, sizeof(double) * nb, cudaMemcpyHostToDevice) != cudaSuccess)
        return c->cuda_check("boundary values");
    c->pt.face_value = c->face_bc_dev.p;
    return SFV_OK;
}

std::string build_layout(sfv_ctx* c) {
    const HostMesh& m = c->mesh;
    // the alternative J.v kernels build their tables on the host from the full geometry
    if (c->jv_path != 0)
        if (std::string e = download_geometry(c->dgeo, c->geom); !e.empty()) return e;
    const HostGeometry& g = c->geom;
    const int nc = m.n_cells, nf = m.n_faces();
    int slots = 0;
    for (int i = 0; i < nc; ++i) slots = std::max(slots, m.cf_off[i + 1] - m.cf_off[i]);
    if (slots > kMaxSlots) return "mesh: cells with more than 8 faces are not supported by the device layout";
    if (static_cast<size_t>(slots) * nc > static_cast<size_t>(INT_MAX) || nc > (INT_MAX >> 3))
        return "mesh: too many cells for 32-bit slot indices";
    auto par = [](int n, const std::function<void(int, int)>& body) {  // independent ranges
        const int nth = host_threads();
        std::vector<std::thread> th;
        const int ch = (n + nth - 1) / nth;
        for (int k = 0; k < nth; ++k) th.emplace_back(body, std::min(n, k * ch), std::min(n, (k + 1) * ch));
        for (auto& t : th) t.join();
    };
    const bool legacy = c->jv_path != 0;  // SoA slot / face arrays only for the alternative J.v kernels
    // default path: tiled tables (device.h), slot stride padded to the kernels' template width
    const int spad = slots <= 4 ? 4 : slots <= 6 ? 6 : 8;
    const int ntc = (nc + 31) / 32, ntf = (nf + 31) / 32;
    const size_t nsl = legacy ? static_cast<size_t>(slots) * nc : 0;
    std::vector<int> sf(nsl, -1), so(nsl, -1);
    std::vector<double> sl(3 * nsl, 0.0);
    // default path with the geometry on the device: the tables are built there (geometry.cu)
    const bool on_dev = !legacy && c->dgeo;
    std::vector<int> tsl(legacy || on_dev ? 0 : static_cast<size_t>(ntc) * 2 * spad * 32, -1);
    std::vector<double> tls(legacy || on_dev ? 0 : static_cast<size_t>(ntc) * 3 * spad * 32, 0.0);
    std::vector<int> bsi(on_dev ? 0 : std::max(1, nf - m.n_internal), 0);
    if (!on_dev)
    par(nc, [&](int i0, int i1) {
    for (int i = i0; i < i1; ++i) {
        int s = 0;
        for (int q = m.cf_off[i]; q < m.cf_off[i + 1]; ++q, ++s) {
            const int f = m.cf[q];
            const bool nb = f < m.n_internal && m.neighbour[f] == i;
            const int code = f | (nb ? static_cast<int>(0x80000000u) : 0);
            const int other = f < m.n_internal ? (nb ? m.owner[f] : m.neighbour[f]) : -(2 + m.face_patch[f]);
            if (legacy) {
                const size_t si = static_cast<size_t>(s) * nc + i;
                sf[si] = code;
                so[si] = other;
                sl[(3 * static_cast<size_t>(s)) * nc + i] = g.ls[q].x;
                sl[(3 * static_cast<size_t>(s) + 1) * nc + i] = g.ls[q].y;
                sl[(3 * static_cast<size_t>(s) + 2) * nc + i] = g.ls[q].z;
                if (f >= m.n_internal) bsi[f - m.n_internal] = static_cast<int>(si);
            } else {
                const size_t tb = tiled(i, 2 * spad), lb = tiled(i, 3 * spad);
                tsl[tb + 32 * s] = code;
                tsl[tb + 32 * (spad + s)] = other;
                tls[lb + 32 * (3 * s)] = g.ls[q].x;
                tls[lb + 32 * (3 * s + 1)] = g.ls[q].y;
                tls[lb + 32 * (3 * s + 2)] = g.ls[q].z;
                if (f >= m.n_internal) bsi[f - m.n_internal] = i * 8 + s;
            }
        }
    }
    });
    const size_t nfl = legacy ? static_cast<size_t>(nf) : 0;
    std::vector<double> gm(3 * nfl), de(3 * nfl), dmg(nfl), ww(nfl);
    std::vector<double> f9(legacy || on_dev ? 0 : static_cast<size_t>(ntf) * 9 * 32, 0.0);
    if (!on_dev)
    par(nf, [&](int f0, int f1) {
    for (int f = f0; f < f1; ++f) {
        if (legacy) {
            gm[f] = g.area[f].x;
            gm[nf + f] = g.area[f].y;
            gm[2 * static_cast<size_t>(nf) + f] = g.area[f].z;
            de[f] = g.delta[f].x;
            de[nf + f] = g.delta[f].y;
            de[2 * static_cast<size_t>(nf) + f] = g.delta[f].z;
            dmg[f] = g.d_mag[f];
            ww[f] = g.w[f];
            continue;
        }
        // per-face constants of rhie_chow(): |Delta| / |d| and |Gamma| (discretisation.cpp:176-208),
        // same IEEE operations as the reference (sqrt of the left-to-right dot, then divide)
        const double* a = &g.area[f].x;
        const double* d = &g.delta[f].x;
        const double rec[9] = {a[0], a[1], a[2], d[0], d[1], d[2],
                               std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]) / g.d_mag[f],
                               std::sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]), g.w[f]};
        const size_t fb = tiled(f, 9);
        for (int q = 0; q < 9; ++q) f9[fb + 32 * q] = rec[q];
    }
    });
    const size_t nbs = std::max(1, nf - m.n_internal);
    if ((legacy && (!c->slot_face.upload(sf) || !c->slot_other.upload(so) || !c->slot_ls.upload(sl) ||
                    !c->gam.upload(gm) || !c->del.upload(de) || !c->dmag.upload(dmg) || !c->w.upload(ww))) ||
        (!legacy && !on_dev && (!c->tslot.upload(tsl) || !c->tls.upload(tls) || !c->face9.upload(f9))) ||
        (on_dev && (!c->tslot.alloc(static_cast<size_t>(ntc) * 2 * spad * 32) ||
                    !c->tls.alloc(static_cast<size_t>(ntc) * 3 * spad * 32) ||
                    !c->face9.alloc(static_cast<size_t>(ntf) * 9 * 32) || !c->bnd_si.alloc(nbs))) ||
        (!legacy && !c->pwg.alloc(static_cast<size_t>(ntc) * kWG * 32)) ||
        (!on_dev && !c->bnd_si.upload(bsi)) || !c->bres.alloc(6 * nbs))
        return "cuda: out of device memory for the mesh layout";
    if (on_dev) {
        const std::string le = device_layout(c->dgeo, spad, c->tslot.p, c->tls.p, c->face9.p, c->bnd_si.p);
        if (!le.empty()) return le;
    }
    if (c->ph.transient && !c->volume.upload(g.volume)) return "cuda: out of device memory";
    DevMesh& d = c->dm;
    d.nc = nc;
    d.nf = nf;
    d.nint = m.n_internal;
    d.slots = slots;
    d.spad = spad;
    d.slot_face = c->slot_face.p;
    d.slot_other = c->slot_other.p;
    d.slot_ls = c->slot_ls.p;
    d.gam = c->gam.p;
    d.del = c->del.p;
    d.dmag = c->dmag.p;
    d.w = c->w.p;
    d.tslot = c->tslot.p;
    d.tls = c->tls.p;
    d.tf9 = c->face9.p;
    d.volume = c->volume.p;
    if (!legacy && (c->ph.law != SFV_LAW_HOOKE || c->ph.tl) && !c->psig.alloc(static_cast<size_t>(ntc) * kSig * 32))
        return "cuda: out of device memory for the mesh layout";
    if (c->ph.law == SFV_LAW_J2) {  // PlasticCell{} per cell (laws.hpp:66-70): b_bar = I, eps_p = 0, F = I
        std::vector<double> st(static_cast<size_t>(ntc) * kJ2 * 32, 0.0);
        for (int i = 0; i < ntc * 32; ++i)
            for (int q : {0, 4, 8, 10, 14, 18}) st[tiled(i, kJ2) + 32 * q] = 1.0;
        if (!c->lawst.upload(st)) return "cuda: out of device memory for the law state";
    }
    c->ps.lawst = c->lawst.p;
    c->ps.sig = c->psig.p;
    c->ps.wg = c->pwg.p;
    // boundary pass on a side stream beside the gradient pass: opt-in (SFV_SIDE_STREAM=1);
    // measured 3% slower at 1M cells (the stream events break the PDL chain)
    if (const char* se = std::getenv("SFV_SIDE_STREAM");
        se && std::atoi(se) != 0 && nf > m.n_internal && c->ph.law != SFV_LAW_J2) {
        if (cudaStreamCreateWithFlags(&c->ps.side, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ps.ev_w, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ps.ev_b, cudaEventDisableTiming) != cudaSuccess)
            return "cuda: cannot create the side stream";
    }
    // [w | G] in a persisting L2 window: opt-in experiment (SFV_L2_PERSIST=1);
    // measured 2-4% slower at 1M cells, the passes are latency-bound
    c->ps.win_bytes = 0;
    const char* pe = std::getenv("SFV_L2_PERSIST");
    if (pe && std::atoi(pe) != 0) {
        int dev = 0, max_persist = 0, max_window = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        const size_t want = kWG * sizeof(double) * 32 * static_cast<size_t>(ntc);
        if (max_persist > 0 && max_window > 0) {
            size_t limit = 0;
            cudaDeviceGetLimit(&limit, cudaLimitPersistingL2CacheSize);
            const size_t set_aside = std::min<size_t>(static_cast<size_t>(max_persist), want);
            if (limit < set_aside) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, set_aside);
            cudaDeviceGetLimit(&limit, cudaLimitPersistingL2CacheSize);
            c->ps.win_base = static_cast<void*>(c->pwg.p);
            c->ps.win_bytes = std::min<size_t>(want, static_cast<size_t>(max_window));
            c->ps.win_hit = static_cast<float>(std::min(1.0, static_cast<double>(limit) / c->ps.win_bytes));
            cudaGetLastError();
        }
    }
    c->ps.bnd_cs = c->bnd_si.p;
    for (int q = 0; q < c->pt.n; ++q) c->ps.sym = c->ps.sym || c->pt.kind[q] == SFV_PATCH_SYMMETRY;
    c->ps.bres = c->bres.p;
    return "";
}

// Layout of the fused kernel: faces regrouped by the tile of their lower cell (sorted by
// the slot they occupy there, then by cell, so ring writes of a warp are contiguous),
// rings sized to the pipeline depth.  Returns "" when the fused path is unusable (too
// wide a bandwidth for L2-resident rings), and the two-pass kernels are used instead.
std::string build_fused_layout(sfv_ctx* c) {
    const HostMesh& m = c->mesh;
    const HostGeometry& g = c->geom;
    const int nc = m.n_cells, nf = m.n_faces();
    int bw = 0;
    for (int f = 0; f < m.n_internal; ++f) bw = std::max(bw, std::abs(m.neighbour[f] - m.owner[f]));
    std::vector<int> slot_of_owner(nf, 0), slot_of_nb(nf, 0);
    for (int i = 0; i < nc; ++i)
        for (int q = m.cf_off[i]; q < m.cf_off[i + 1]; ++q) {
            const int f = m.cf[q];
            if (m.owner[f] == i) slot_of_owner[f] = q - m.cf_off[i];
            else slot_of_nb[f] = q - m.cf_off[i];
        }
    FusedLayout& L = c->fl;
    L.ntiles = (nc + kTile - 1) / kTile;
    L.lag = (bw + kTile - 1) / kTile + 1;
    const int ctas = fused_resident_ctas(c->ph.law != SFV_LAW_HOOKE || c->ph.tl != 0);
    c->f_grid = std::max(1, std::min(ctas, L.ntiles + L.lag));
    L.ring_tiles = std::min(L.ntiles + L.lag + 1, L.lag + c->f_grid + 4);
    L.ring_cells = L.ring_tiles * kTile;
    const double ring_bytes = 8.0 * L.ring_cells * (9.0 + 6.0 * c->dm.slots);
    if (ring_bytes > 96e6) return "rings exceed the L2 budget";
    std::vector<int> order(nf);
    for (int f = 0; f < nf; ++f) order[f] = f;
    auto low = [&](int f) { return f < m.n_internal ? std::min(m.owner[f], m.neighbour[f]) : m.owner[f]; };
    auto low_slot = [&](int f) {
        return f < m.n_internal && m.neighbour[f] < m.owner[f] ? slot_of_nb[f] : slot_of_owner[f];
    };
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        const int ta = low(a) / kTile, tb = low(b) / kTile;
        if (ta != tb) return ta < tb;
        const int sa = low_slot(a), sb = low_slot(b);
        if (sa != sb) return sa < sb;
        return low(a) < low(b);
    });
    std::vector<int> tfp(L.ntiles + 1, 0), own(nf), oth(nf), sl(nf), idx(nf);
    std::vector<double> geo(8 * static_cast<size_t>(nf));
    for (int x = 0; x < nf; ++x) {
        const int f = order[x];
        ++tfp[low(f) / kTile + 1];
        own[x] = m.owner[f];
        oth[x] = f < m.n_internal ? m.neighbour[f] : -(2 + m.face_patch[f]);
        sl[x] = slot_of_owner[f] | ((f < m.n_internal ? slot_of_nb[f] : 0) << 8);
        idx[x] = f;
        const double vals[8] = {g.area[f].x, g.area[f].y, g.area[f].z, g.delta[f].x,
                                g.delta[f].y, g.delta[f].z, g.d_mag[f], g.w[f]};
        for (int k = 0; k < 8; ++k) geo[static_cast<size_t>(k) * nf + x] = vals[k];
    }
    for (int t = 0; t < L.ntiles; ++t) tfp[t + 1] += tfp[t];
    if (!c->f_tfp.upload(tfp) || !c->f_own.upload(own) || !c->f_oth.upload(oth) || !c->f_slots.upload(sl) ||
        !c->f_index.upload(idx) || !c->f_geo.upload(geo) || !c->f_gring.alloc(9 * static_cast<size_t>(L.ring_cells)) ||
        !c->f_fring.alloc(6 * static_cast<size_t>(c->dm.slots) * L.ring_cells) ||
        !c->f_flags.alloc(3 * static_cast<size_t>(L.ntiles)) || !c->f_ticket.alloc(1))
        return "cuda: out of device memory for the fused layout";
    cudaMemset(c->f_flags.p, 0, sizeof(int) * 3 * static_cast<size_t>(L.ntiles));
    L.nfl = nf;
    L.tile_face_ptr = c->f_tfp.p;
    L.f_owner = c->f_own.p;
    L.f_other = c->f_oth.p;
    L.f_slots = c->f_slots.p;
    L.f_index = c->f_index.p;
    L.f_geo = c->f_geo.p;
    L.gring = c->f_gring.p;
    L.fring = c->f_fring.p;
    c->use_fused = true;
    return "";
}

void launch_fused_pass(sfv_ctx* c, const Physics& ph, const double* u, const double* v, const double* eps,
                       const double* r_u, double* out) {
    FusedArgs a;
    a.m = c->dm;
    a.L = c->fl;
    a.ph = ph;
    a.pt = c->pt;
    a.hist = c->hist;
    a.u = u;
    a.v = v ? v : u;
    a.eps = eps;
    a.r_u = r_u;
    a.out = out;
    a.err = c->err.p;
    a.ticket = c->f_ticket.p;
    a.a_done = c->f_flags.p;
    a.b1_done = c->f_flags.p + c->fl.ntiles;
    a.b2_done = c->f_flags.p + 2 * static_cast<size_t>(c->fl.ntiles);
    a.epoch = ++c->f_epoch;
    cudaMemsetAsync(c->f_ticket.p, 0, sizeof(int), c->stream);
    launch_fused(a, c->f_grid, c->stream);
    c->launches += 1;
}

// the default path runs boundary_kernel (else the flux pass evaluates the boundary faces)
bool boundary_pass(const sfv_ctx* c) {
    return c->dm.nf > c->dm.nint && (c->ph.law != SFV_LAW_HOOKE || c->ph.tl || c->ps.sym || c->ps.side);
}

void reset_err(sfv_ctx* c) { cudaMemsetAsync(c->err.p, 0x7f, sizeof(ErrWords), c->stream); }

// read the error words (and optionally k doubles from hdev) in one D2H + sync
int fetch(sfv_ctx* c, int k) {
    cudaMemcpyAsync(&c->st->err, c->err.p, sizeof(ErrWords), cudaMemcpyDeviceToHost, c->stream);
    if (k > 0) cudaMemcpyAsync(c->st->h, c->hdev.p, sizeof(double) * k, cudaMemcpyDeviceToHost, c->stream);
    const cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return c->fail(SFV_ERR_CUDA, -1, std::string("cuda: ") + cudaGetErrorString(e));
    return SFV_OK;
}

// Map device error words to the reference's exception, in the order the reference
// would raise them (stress loop, then face loop, then the NaN scan).
int decode_residual_errors(sfv_ctx* c, bool jv) {
    const ErrWords& e = c->st->err;
    // the stress loop throws at the first failing cell: LawOverflow / ReturnMapFailure there if
    // it comes first (a J.v maps LawOverflow to JvpNan and lets ReturnMapFailure through,
    // nonlinear.cpp:122-131)
    if (e.retmap_cell != kNone && e.retmap_cell < e.inverted_cell && e.retmap_cell < e.overflow_cell)
        return c->fail(SFV_ERR_RETURN_MAP, e.retmap_cell, "j2_radial_return: hardening Newton did not converge");
    if (e.overflow_cell != kNone && e.overflow_cell < e.inverted_cell)
        return jv ? c->fail(SFV_ERR_JVP_NAN, -1, "jvp: guccione_stress: exponent overflow")
                  : c->fail(SFV_ERR_LAW_OVERFLOW, e.overflow_cell, "guccione_stress: exponent overflow");
    if (e.inverted_cell != kNone)
        return jv ? c->fail(SFV_ERR_JVP_NAN, -1, "jvp: kinematics: det F <= 0")
                  : c->fail(SFV_ERR_INVERTED_ELEMENT, e.inverted_cell, "kinematics: det F <= 0");
    if (e.inverted_face != kNone)
        return jv ? c->fail(SFV_ERR_JVP_NAN, -1, "jvp: face deformation gradient is not invertible")
                  : c->fail(SFV_ERR_INVERTED_ELEMENT, c->mesh.owner[e.inverted_face],
                            "face deformation gradient is not invertible");
    if (e.nan_cell != kNone)
        return jv ? c->fail(SFV_ERR_JVP_NAN, -1, "jvp: residual: non-finite entry")
                  : c->fail(SFV_ERR_RESIDUAL_NAN, e.nan_cell, "residual: non-finite entry");
    if (jv && e.nan_jv != kNone) return c->fail(SFV_ERR_JVP_NAN, -1, "jvp: non-finite difference quotient");
    return SFV_OK;
}

int gradient_failure(sfv_ctx* c) {
    return c->fail(SFV_ERR_GRADIENT_FAILURE, c->singular_cell, "cell_gradients: singular least-squares stencil");
}

// R(u) into r (async; caller fetches + decodes)
void residual_pass(sfv_ctx* c, const Physics& ph, const double* u, const double* v, const double* eps,
                   const double* r_u, double* out) {
    if (c->use_fused) {
        launch_fused_pass(c, ph, u, v, eps, r_u, out);
        return;
    }
    if (c->jv_path == 0) {
        launch_residual_pair(c->dm, ph, c->pt, c->hist, u, v, eps, r_u, out, c->ps, c->err.p, c->stream);
        c->launches += boundary_pass(c) ? 4 : 3;
        return;
    }
    launch_residual(c->dm, ph, c->pt, c->hist, u, v, eps, r_u, out, c->grad.p, c->err.p, c->stream);
    c->launches += 2;
}

void residual_async(sfv_ctx* c, const double* u, double* r) {
    residual_pass(c, c->ph, u, nullptr, nullptr, nullptr, r);
}

// *out = a.b on the device: a fixed-order tree, or the reference's left-to-right chain
void dot_async(sfv_ctx* c, const double* a, const double* b, int n, double* out) {
    if (c->seq_reduce) launch_seq_dot(a, b, n, out, c->stream);
    else launch_dot(a, b, n, out, c->red.p, c->counter.p, c->stream);
}

// J.v (async).  u_norm_cached: *scal[1] already holds |u| for this u.
void jv_async(sfv_ctx* c, const double* u, const double* r_u, const double* v, double* out, bool u_norm_cached) {
    if (c->seq_reduce) {  // reference-order |v|, |u| and ε (nonlinear.cpp:109-115), then w = u + εv
        launch_seq_eps(u, v, c->n, c->red.p, c->scal.p, c->scal.p + 1, u_norm_cached, c->stream);
        c->ps.partials = nullptr;
        residual_pass(c, c->ph, u, v, c->scal.p, r_u, out);
        c->launches += 2;
        return;
    }
    if (c->jv_path == 0) {  // norms as block partials; eps finished inside the perturb pass
        if (!c->ps.bar) {
            c->ps.npart = launch_norm_partials(u, v, c->n, c->red.p, u_norm_cached, c->stream);
            c->launches += 1;
        }
        c->ps.partials = c->red.p;
        c->ps.u_norm = c->scal.p + 1;
        c->ps.u_norm_cached = u_norm_cached;
        residual_pass(c, c->ph, u, v, c->scal.p, r_u, out);
        c->ps.partials = nullptr;
        return;
    }
    launch_jv_eps(u, v, c->n, c->red.p, c->counter.p, c->scal.p, c->scal.p + 1, u_norm_cached, c->stream);
    residual_pass(c, c->ph, u, v, c->scal.p, r_u, out);
    c->launches += 1;
}

int residual_sync(sfv_ctx* c, const double* u, double* r) {
    if (c->singular_cell >= 0) return gradient_failure(c);
    reset_err(c);
    residual_async(c, u, r);
    if (int e = c->cuda_check("residual")) return e;
    if (int e = fetch(c, 0)) return e;
    return decode_residual_errors(c, false);
}

// squared-norm on the device, returned on the host (one sync)
int norm_host(sfv_ctx* c, const double* a, double* out) {
    dot_async(c, a, a, c->n, c->hdev.p);
    c->launches += 1;
    if (int e = fetch(c, 1)) return e;
    *out = std::sqrt(c->st->h[0]);
    return SFV_OK;
}

int precond_apply_async(sfv_ctx* c, const double* r, double* z) {
    const int n = c->n;
    switch (c->pc_kind) {
        case SFV_PRECOND_ILU0:
        case SFV_PRECOND_ILU1:
        case SFV_PRECOND_ILU2:
        {
            TriSet Ls, Us;
            for (int a = 0; a < 3; ++a) {
                Ls.t[a] = c->L[a].view;
                Us.t[a] = c->U[a].view;
            }
            launch_ilu_apply(Ls, Us, c->pc_coupled ? -1 : c->pc_ncomp, r, c->ily.p, z, c->tri_grid, c->tri_sleep, c->tri_cluster, c->ipa.p,
                             c->ipb.p, &c->sL, &c->sU, c->stream, &c->pL, &c->pU);
            c->launches += c->tri_cluster == kPipeMode ? 11 : c->tri_cluster > 0 ? 2 : 4;
            return SFV_OK;
        }
        case SFV_PRECOND_LU:
            for (int a = 0; a < c->pc_ncomp; ++a) {
                launch_dense_apply_perm(c->dense_w[a].p, c->pc_coupled ? c->n : c->nc, c->dense_perm[a].p, r, z,
                                        c->pc_coupled ? kDenseCoupled : c->pc_ncomp == 1 ? -1 : a, c->stream);
                c->launches += 1;
            }
            return SFV_OK;
        default:
            if (r != z) cudaMemcpyAsync(z, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream);
            return SFV_OK;
    }
}

bool ensure_krylov(sfv_ctx* c, int restart) {
    const size_t n = static_cast<size_t>(c->n);
    if (c->v_cap >= restart + 1 && c->wv.p) return true;
    c->drop_graph();  // the basis and workspace pointers change
    if (restart + 2 > c->st->hcap) {  // Hessenberg column of an Arnoldi step: restart + 2 doubles
        double* h = nullptr;
        if (cudaMallocHost(&h, sizeof(double) * (restart + 2)) != cudaSuccess || !c->hdev.alloc(restart + 2)) {
            if (h) cudaFreeHost(h);
            return false;
        }
        cudaFreeHost(c->st->h);
        c->st->h = h;
        c->st->hcap = restart + 2;
    }
    bool ok = c->V.alloc(n * (restart + 1)) && c->wv.alloc(n) && c->rv.alloc(n) && c->tv.alloc(n) &&
              c->xv.alloc(n) && c->bv.alloc(n) && c->ydev.alloc(restart + 1) && c->ucand.alloc(n) && c->rcand.alloc(n) &&
              c->uscratch.alloc(n) && c->rscratch.alloc(n);
    c->v_cap = ok ? restart + 1 : 0;
    return ok;
}

enum { G_CONVERGED = 0, G_MAX_ITERS = 1, G_STAGNATED = 2 };

size_t gstate_bytes(int m) {
    return sizeof(GmresHdr) + sizeof(double) * (2 * static_cast<size_t>(m) + (m + 1) + static_cast<size_t>(m) * (m + 1));
}
GmresDev gstate_view(unsigned char* base, int m) {
    GmresDev d;
    d.hdr = reinterpret_cast<GmresHdr*>(base);
    d.cs = reinterpret_cast<double*>(base + sizeof(GmresHdr));
    d.sn = d.cs + m;
    d.g = d.sn + m;
    d.H = d.g + (m + 1);
    return d;
}

// The cycle graph for op = J.v at (u, r_u): a WHILE node whose body is one Arnoldi step —
// J.v of V[j] (the fused ε pass selects v on the device), the preconditioner, the fused MGS
// step (j on the device) and givens_kernel, which sets the condition.  Built once per
// (u, r_u, restart) and reused for every cycle; false when any piece cannot be captured
// (then gmres keeps the host-driven loop).  SFV_GMRES_GRAPH=0 disables it.
// Kernel arguments are captured by value: the patch values (set_time), the physics, the
// history pointers, the preconditioner's buffers and every workspace pointer.  The graph is
// reused only while all of them are unchanged.
std::vector<unsigned char> gmres_graph_key(const sfv_ctx* c, const double* u, const double* r_u, int restart) {
    std::vector<unsigned char> k;
    auto put = [&](const void* p, size_t nb) {
        const unsigned char* b = static_cast<const unsigned char*>(p);
        k.insert(k.end(), b, b + nb);
    };
    const void* ptrs[] = {u, r_u, c->V.p, c->tv.p, c->wv.p, c->hdev.p, c->red.p, c->scal.p, c->err.p, c->pwg.p,
                          c->gstate.p, c->stream};
    put(ptrs, sizeof(ptrs));
    put(&restart, sizeof(restart));
    put(&c->pc_gen, sizeof(c->pc_gen));
    put(&c->ph, sizeof(c->ph));
    put(&c->pt, sizeof(c->pt));
    put(&c->hist, sizeof(c->hist));
    put(&c->dm, sizeof(c->dm));
    return k;
}

bool gmres_graph_ready(sfv_ctx* c, const double* u, const double* r_u, int restart) {
    static const bool off = [] {
        const char* e = std::getenv("SFV_GMRES_GRAPH");
        return e && std::atoi(e) == 0;
    }();
    if (off || c->graph_off || c->graph_broken || c->use_fused || c->jv_path != 0 || !c->ps.bar) return false;
    int chunk = 0;
    if (eps_perturb_grid_for(c->nc) == 0 || arnoldi_fused_grid(c->n, &chunk) == 0) return false;
    if (c->gexec && c->g_key == gmres_graph_key(c, u, r_u, restart)) return true;
    c->drop_graph();
    auto broken = [&](const char* why) {
        if (std::getenv("SFV_TIMING")) std::fprintf(stderr, "[sfv] gmres graph unavailable: %s\n", why);
        cudaGetLastError();
        c->drop_graph();
        c->graph_broken = true;
        return false;
    };
    if (c->g_cap < restart) {
        if (c->gstate_host) cudaFreeHost(c->gstate_host);
        c->gstate_host = nullptr;
        if (!c->gstate.alloc(gstate_bytes(restart)) ||
            cudaMallocHost(&c->gstate_host, gstate_bytes(restart)) != cudaSuccess)
            return broken("state allocation");
        c->g_cap = restart;
    }
    c->gdev = gstate_view(c->gstate.p, restart);
    if (!c->gstream && (cudaStreamCreateWithFlags(&c->gstream, cudaStreamNonBlocking) != cudaSuccess ||
                        cudaEventCreateWithFlags(&c->gev0, cudaEventDisableTiming) != cudaSuccess ||
                        cudaEventCreateWithFlags(&c->gev1, cudaEventDisableTiming) != cudaSuccess))
        return broken("stream");
    cudaGraphConditionalHandle cond;
    if (cudaGraphCreate(&c->graph, 0) != cudaSuccess ||
        cudaGraphConditionalHandleCreate(&cond, c->graph, 1, cudaGraphCondAssignDefault) != cudaSuccess)
        return broken("conditional handle");
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cond;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    if (cudaGraphAddNode(&node, c->graph, nullptr, 0, &np) != cudaSuccess) return broken("while node");
    cudaGraph_t body = np.conditional.phGraph_out[0];
    const int n = c->n;
    cudaStream_t saved = c->stream;
    c->stream = c->gstream;
    const long long l0 = c->launches;
    c->vsel_failed = false;
    bool ok = cudaStreamBeginCaptureToGraph(c->gstream, body, nullptr, nullptr, 0,
                                            cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
        c->ps.vsel_j = &c->gdev.hdr->j;
        c->ps.vsel_stride = static_cast<size_t>(n);
        c->ps.vsel_failed = &c->vsel_failed;
        c->ps.partials = c->red.p;
        c->ps.u_norm = c->scal.p + 1;
        c->ps.u_norm_cached = true;
        residual_pass(c, c->ph, u, c->V.p, c->scal.p, r_u, c->tv.p);
        c->ps.partials = nullptr;
        c->ps.vsel_j = nullptr;
        c->ps.vsel_failed = nullptr;
        if (std::getenv("SFV_GRAPH_NOPC"))  // debugging aid: identity preconditioner inside the graph
            cudaMemcpyAsync(c->wv.p, c->tv.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->gstream);
        else
            ok = precond_apply_async(c, c->tv.p, c->wv.p) == SFV_OK;
        ok = launch_arnoldi_fused_dev(c->wv.p, c->V.p, n, &c->gdev.hdr->j, c->v_cap, c->hdev.p, c->red.p,
                                      c->gstream) && ok;
        launch_givens(c->gdev, c->hdev.p, c->err.p, cond, c->gstream);
        c->launches += 2;
        cudaGraph_t out = nullptr;
        ok = cudaStreamEndCapture(c->gstream, &out) == cudaSuccess && ok && !c->vsel_failed;
    }
    c->stream = saved;
    c->g_launches = c->launches - l0;
    c->launches = l0;
    if (!ok) return broken("capture");
    if (cudaGraphInstantiate(&c->gexec, c->graph, 0) != cudaSuccess) return broken("instantiate");
    c->g_key = gmres_graph_key(c, u, r_u, restart);
    return true;
}

// One restart cycle through the graph: state upload (j = 0, total, g[0] = beta, target),
// the graph, and one fetch of the state and the error words.
int gmres_graph_cycle(sfv_ctx* c, int total, int restart, int max_iters, double beta, double target) {
    GmresDev hv = gstate_view(c->gstate_host, restart);
    *hv.hdr = GmresHdr{0, total, restart, max_iters, 0, 0, target};
    hv.g[0] = beta;
    cudaMemcpyAsync(c->gstate.p, c->gstate_host, sizeof(GmresHdr), cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(c->gdev.g, hv.g, sizeof(double), cudaMemcpyHostToDevice, c->stream);
    reset_err(c);
    cudaEventRecord(c->gev0, c->stream);
    cudaStreamWaitEvent(c->gstream, c->gev0, 0);
    if (cudaGraphLaunch(c->gexec, c->gstream) != cudaSuccess) return c->cuda_check("gmres graph");
    cudaEventRecord(c->gev1, c->gstream);
    cudaStreamWaitEvent(c->stream, c->gev1, 0);
    cudaMemcpyAsync(c->gstate_host, c->gstate.p, gstate_bytes(restart), cudaMemcpyDeviceToHost, c->stream);
    if (int e = fetch(c, 0)) return e;
    c->launches += c->g_launches * (hv.hdr->total - total);
    return SFV_OK;
}

// gmres_solve (/root/reference/proj/src/linalg.cpp:423-538), with op = J.v at (u, r_u),
// left preconditioned or, with `right`, right preconditioned (residuals unpreconditioned
// :437, w = op(M^-1 v_j) :466-467, dx = M^-1 V y :514).  x_zero: x0 is all zeros, so
// op(x0) = 0 without evaluation (jacobian_vector_product short-circuits |v| = 0,
// nonlinear.cpp:110).  Any restart >= 1 (the basis is sized to it).
int gmres(sfv_ctx* c, const double* u, const double* r_u, const double* b, double* x, bool x_zero, int restart,
          double rel_reduction, int max_iters, int* iters_out, int* status_out, double* rel_out, bool right = false) {
    const int n = c->n;
    if (restart < 1) return c->fail(SFV_ERR_INVALID_ARGUMENT, -1, "gmres: restart must be >= 1");
    if (!ensure_krylov(c, restart)) return c->fail(SFV_ERR_CUDA, -1, "gmres: out of device memory");
    double* V = c->V.p;
    double* w = c->wv.p;
    double* r = c->rv.p;
    double* tmp = c->tv.p;
    bool unorm_cached = false;
    auto op = [&](const double* v, double* out) -> int {
        reset_err(c);
        jv_async(c, u, r_u, v, out, unorm_cached);
        unorm_cached = true;
        return SFV_OK;
    };
    // residual(x): r = M^-1 (b - op(x))  (linalg.cpp:434-439)
    auto residual_of_x = [&](bool zero) -> int {
        double* res = right ? r : tmp;  // b - op(x); left: then M^-1
        if (zero) {
            cudaMemcpyAsync(res, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream);
        } else {
            op(x, res);
            launch_sub_from(b, res, n, c->stream);
            ++c->launches;
        }
        if (!right)
            if (int e = precond_apply_async(c, tmp, r)) return e;
        dot_async(c, r, r, n, c->hdev.p);
        ++c->launches;
        if (int e = fetch(c, 1)) return e;
        if (!zero)
            if (int e = decode_residual_errors(c, true)) return e;
        return SFV_OK;
    };
    int total = 0, status = G_MAX_ITERS;
    double rel = 1.0;
    *iters_out = 0;
    if (int e = residual_of_x(x_zero)) return e;
    const double r0 = std::sqrt(c->st->h[0]);
    if (r0 == 0.0) {
        *status_out = G_CONVERGED;
        *rel_out = 0.0;
        return SFV_OK;
    }
    const double target = rel_reduction * r0;
    double beta = r0;
    std::vector<std::vector<double>> H;
    std::vector<double> cs, sn, g, y;
    // SFV_TIMING=1: per-iteration device time of J.v / preconditioner / Arnoldi, and the
    // host wall time of the per-iteration fetch, summed over the solve (stderr)
    struct IterTimer {
        bool on = std::getenv("SFV_TIMING") != nullptr;
        cudaEvent_t ev[4];
        double ms[4] = {0, 0, 0, 0};
        int iters = 0;
        IterTimer() {
            if (on)
                for (auto& e : ev) cudaEventCreate(&e);
        }
        void add(double host_ms) {
            float t = 0.f;
            for (int k = 0; k < 3; ++k) {
                cudaEventElapsedTime(&t, ev[k], ev[k + 1]);
                ms[k] += t;
            }
            ms[3] += host_ms;
            ++iters;
        }
        ~IterTimer() {
            if (!on) return;
            if (iters)
                std::fprintf(stderr, "[sfv] gmres %d iters: jv %.3f  precond %.3f  arnoldi %.3f  fetch(host) %.3f ms/iter\n",
                             iters, ms[0] / iters, ms[1] / iters, ms[2] / iters, ms[3] / iters);
            for (auto& e : ev) cudaEventDestroy(e);
        }
    } tim;
    static const bool no_fused_mgs = [] {
        const char* e = std::getenv("SFV_FUSED_MGS");
        return e && std::atoi(e) == 0;
    }();
    const bool use_graph = !right && !c->seq_reduce && gmres_graph_ready(c, u, r_u, restart);
    while (total < max_iters) {
        const double cycle_start = beta;
        launch_scale_div_host(r, beta, V, n, c->stream);  // v0 = r / beta
        ++c->launches;
        H.clear();
        cs.clear();
        sn.clear();
        g.assign(1, beta);
        int j = 0;
        bool happy = false;
        if (use_graph) {
            if (!unorm_cached) op(V, tmp);  // |u| for this u, as the first in-loop J.v would compute it
            if (int e = gmres_graph_cycle(c, total, restart, max_iters, beta, target)) return e;
            if (int e = decode_residual_errors(c, true)) return e;
            const GmresDev hv = gstate_view(c->gstate_host, restart);
            j = hv.hdr->j;
            total = hv.hdr->total;
            happy = hv.hdr->happy != 0;
            g.assign(hv.g, hv.g + j + 1);
            for (int k = 0; k < j; ++k) H.emplace_back(hv.H + static_cast<size_t>(k) * (restart + 1),
                                                     hv.H + static_cast<size_t>(k) * (restart + 1) + k + 2);
        }
        while (!use_graph && j < restart && total < max_iters) {
            double* vj = V + static_cast<size_t>(j) * n;
            if (tim.on) cudaEventRecord(tim.ev[0], c->stream);
            if (right) {  // w = op(M^-1 v_j)
                if (int e = precond_apply_async(c, vj, tmp)) return e;
                if (tim.on) cudaEventRecord(tim.ev[1], c->stream);
                op(tmp, w);
            } else {  // w = M^-1 op(v_j)
                op(vj, tmp);
                if (tim.on) cudaEventRecord(tim.ev[1], c->stream);
                if (int e = precond_apply_async(c, tmp, w)) return e;
            }
            if (tim.on) cudaEventRecord(tim.ev[2], c->stream);
            // modified Gram-Schmidt (linalg.cpp:469-473).  Fused: one cooperative launch with
            // w in shared memory, also writing v_{j+1} = w / |w|.  Otherwise h_0 = w.v_0, then
            // w -= h_i v_i fused with h_{i+1} = w.v_{i+1}; the last pass yields w.w
            bool fused = !no_fused_mgs && !c->seq_reduce &&
                         launch_arnoldi_fused(w, V, n, j, c->hdev.p, c->red.p,
                                              j + 1 < restart + 1 ? V + static_cast<size_t>(j + 1) * n : nullptr,
                                              c->stream);
            if (fused) {
                ++c->launches;
            } else {
                dot_async(c, w, V, n, c->hdev.p);
                ++c->launches;
                for (int i = 0; i <= j; ++i) {
                    const double* vnext = i < j ? V + static_cast<size_t>(i + 1) * n : nullptr;
                    if (c->seq_reduce)
                        launch_seq_axpy_dot(w, V + static_cast<size_t>(i) * n, c->hdev.p + i, vnext, n,
                                            c->hdev.p + i + 1, c->stream);
                    else
                        launch_axpy_dot(w, V + static_cast<size_t>(i) * n, c->hdev.p + i, vnext, n,
                                        c->hdev.p + i + 1, c->red.p, c->counter.p, c->stream);
                    ++c->launches;
                }
            }
            if (int e = c->cuda_check("arnoldi")) return e;
            if (tim.on) cudaEventRecord(tim.ev[3], c->stream);
            const auto th0 = std::chrono::steady_clock::now();
            if (int e = fetch(c, j + 2)) return e;
            if (tim.on) tim.add(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count());
            if (int e = decode_residual_errors(c, true)) return e;
            std::vector<double> hj(j + 2, 0.0);
            for (int i = 0; i <= j; ++i) hj[i] = c->st->h[i];
            hj[j + 1] = std::sqrt(c->st->h[j + 1]);
            for (int i = 0; i < j; ++i) {  // apply stored rotations
                const double t = cs[i] * hj[i] + sn[i] * hj[i + 1];
                hj[i + 1] = -sn[i] * hj[i] + cs[i] * hj[i + 1];
                hj[i] = t;
            }
            const double denom = sfv_hypot(hj[j], hj[j + 1]);
            const double cc = denom == 0.0 ? 1.0 : hj[j] / denom;
            const double ss = denom == 0.0 ? 0.0 : hj[j + 1] / denom;
            cs.push_back(cc);
            sn.push_back(ss);
            g.push_back(-ss * g[j]);
            g[j] = cc * g[j];
            hj[j] = denom;
            const double subdiag = hj[j + 1];
            hj[j + 1] = 0.0;
            H.push_back(std::move(hj));
            ++total;
            ++j;
            if (subdiag <= 1e-14 * std::max(denom, 1e-300)) {  // happy breakdown
                happy = true;
                break;
            }
            if (std::abs(g[j]) <= target) break;
            if (j < restart && !fused) {  // (the fused step already wrote v_j = w / subdiag)
                launch_scale_div_host(w, subdiag, V + static_cast<size_t>(j) * n, n, c->stream);
                ++c->launches;
            }
        }
        // back substitution, then x += V y (linalg.cpp:505-515)
        y.assign(j, 0.0);
        for (int i = j - 1; i >= 0; --i) {
            double s = g[i];
            for (int k = i + 1; k < j; ++k) s -= H[k][i] * y[k];
            y[i] = s / H[i][i];
        }
        cudaMemcpyAsync(c->ydev.p, y.data(), sizeof(double) * j, cudaMemcpyHostToDevice, c->stream);
        if (right) {  // dx = M^-1 (V y); x += 1.0 * dx
            launch_basis_combination(tmp, V, c->ydev.p, j, n, c->stream);
            if (int e = precond_apply_async(c, tmp, w)) return e;
            launch_axpy_host(x, 1.0, w, n, c->stream);
            c->launches += 2;
        } else {
            launch_update(x, V, c->ydev.p, j, n, c->stream);
            ++c->launches;
        }
        x_zero = false;
        if (int e = residual_of_x(false)) return e;  // explicit restart residual (:518-519)
        beta = std::sqrt(c->st->h[0]);
        rel = beta / r0;
        if (beta <= target || (happy && std::abs(g[j]) <= target)) {
            status = G_CONVERGED;
            break;
        }
        if (happy || beta >= cycle_start * (1.0 - 1e-12)) {
            status = G_STAGNATED;
            break;
        }
    }
    *iters_out = total;
    *status_out = status;
    *rel_out = rel;
    return SFV_OK;
}

void push_record(sfv_solve_report* rep, int iter, double r_norm, int kry, double s) {
    const int cap = static_cast<int>(sizeof(rep->records) / sizeof(rep->records[0]));
    const sfv_iteration_record rec{0, iter, r_norm, kry, s};
    if (rep->n_records < cap) rep->records[rep->n_records] = rec;
    if (rep->all_records && rep->n_records < rep->all_capacity) rep->all_records[rep->n_records] = rec;
    ++rep->n_records;
}

// memset a report, keeping the caller's unbounded-history buffer
void clear_report(sfv_solve_report* rep) {
    sfv_iteration_record* all = rep->all_records;
    const int cap = rep->all_capacity;
    std::memset(rep, 0, sizeof(*rep));
    rep->all_records = all;
    rep->all_capacity = cap;
}

// jfnk_solve (nonlinear.cpp:173-266) with line_search (:140-163) and check_convergence
// (:97-103).  Returns an error only where the reference lets an exception escape.
// A = -J~ per component (scalar_component_matrices, linalg.cpp:160-165; nonlinear.cpp:278-281)
// and its IC(0) factor (Ic0Precond, factored once: cg_solve re-factors the same matrix on
// every call, linalg.cpp:384-390) or the Jacobi fallback (DiagPrecond) on a breakdown.
int seg_create(sfv_ctx* c) {
    if (c->seg_ncomp) return SFV_OK;
    std::vector<ScalarCsr> comps;
    const std::string msg = cell_jacobian(c->mesh, c->geom, c->ph.kbar, c->ph.transient != 0, c->ph.rho, c->ph.dt, comps);
    if (!msg.empty() || comps[0].n != c->nc)  // scalar_component (linalg.cpp:120-133) refuses coupled blocks
        return c->fail(SFV_ERR_INVALID_ARGUMENT, -1, "scalar_component: blocks are not diagonal");
    const int n = c->nc;
    for (size_t a = 0; a < comps.size(); ++a) {
        ScalarCsr& A = comps[a];
        for (double& v : A.val) v = -v;
        sfv_ctx::SegComp& sc = c->seg[a];
        ScalarCsr L;
        sc.jacobi = !ic0_factor(A, L);
        bool ok = sc.rp.upload(A.rp) && sc.col.upload(A.col) && sc.val.upload(A.val);
        if (sc.jacobi) {
            std::vector<double> inv(n, 1.0);
            for (int i = 0; i < n; ++i)
                for (int p = A.rp[i]; p < A.rp[i + 1]; ++p)
                    if (A.col[p] == i && A.val[p] != 0.0) inv[i] = 1.0 / A.val[p];
            ok = ok && sc.inv_diag.upload(inv);
        } else {
            TriSchedule f, b;
            schedule_ic0(L, f, b);
            ok = ok && sc.f_order.upload(f.order) && sc.f_rp.upload(f.rp) && sc.f_col.upload(f.col) &&
                 sc.f_val.upload(f.val) && sc.f_diag.upload(f.diag) && sc.b_order.upload(b.order) &&
                 sc.b_rp.upload(b.rp) && sc.b_col.upload(b.col) && sc.b_val.upload(b.val) && sc.b_diag.upload(b.diag);
            sc.fwd = {f.n_pos, sc.f_order.p, sc.f_rp.p, sc.f_col.p, sc.f_val.p, sc.f_diag.p};
            sc.bwd = {b.n_pos, sc.b_order.p, sc.b_rp.p, sc.b_col.p, sc.b_val.p, sc.b_diag.p};
        }
        if (!ok) return c->fail(SFV_ERR_CUDA, -1, "segregated: out of device memory");
        sc.a = {n, sc.rp.p, sc.col.p, sc.val.p};
    }
    const size_t nn = static_cast<size_t>(n);
    if (!c->sg_b.alloc(nn) || !c->sg_x.alloc(nn) || !c->sg_r.alloc(nn) || !c->sg_z.alloc(nn) || !c->sg_p.alloc(nn) ||
        !c->sg_ap.alloc(nn) || !c->sg_y.alloc(nn) || !c->sg_un.alloc(3 * nn) || !c->sg_du.alloc(3 * nn))
        return c->fail(SFV_ERR_CUDA, -1, "segregated: out of device memory");
    c->seg_ncomp = static_cast<int>(comps.size());
    return SFV_OK;
}

// dot product of two device vectors of length n, on the host (fixed-order reduction, one sync)
int dot_host(sfv_ctx* c, const double* a, const double* b, int n, double* out) {
    dot_async(c, a, b, n, c->hdev.p);
    c->launches += 1;
    if (int e = fetch(c, 1)) return e;
    *out = c->st->h[0];
    return SFV_OK;
}

// cg_solve (linalg.cpp:380-421) on component comp: x (holding x0) <- A^{-1} b approximately
int seg_cg(sfv_ctx* c, const sfv_ctx::SegComp& sc, const double* b, double* x, double rel, int max_iters,
           int* iters) {
    const int n = c->nc;
    double *r = c->sg_r.p, *z = c->sg_z.p, *p = c->sg_p.p, *ap = c->sg_ap.p;
    cudaStream_t s = c->stream;
    auto precond = [&](const double* in, double* out) {
        if (sc.jacobi) seg_jacobi(n, sc.inv_diag.p, in, out, s);
        else seg_ic0_apply(sc.fwd, sc.bwd, in, c->sg_y.p, out, n, seg_sweep_grid(), s);
        c->launches += sc.jacobi ? 1 : 4;
    };
    *iters = 0;
    seg_spmv(sc.a, x, r, s);
    seg_rsub(n, b, r, s);
    c->launches += 2;
    double r0;
    if (int e = dot_host(c, r, r, n, &r0)) return e;
    r0 = std::sqrt(r0);
    if (r0 == 0.0) return SFV_OK;
    precond(r, z);
    cudaMemcpyAsync(p, z, sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
    double rz;
    if (int e = dot_host(c, r, z, n, &rz)) return e;
    for (int it = 0; it < max_iters; ++it) {
        seg_spmv(sc.a, p, ap, s);
        ++c->launches;
        double pap;
        if (int e = dot_host(c, p, ap, n, &pap)) return e;
        if (!(pap > 0.0)) break;  // loss of positive definiteness
        const double alpha = rz / pap;
        launch_axpy_host(x, alpha, p, n, s);
        launch_axpy_host(r, -alpha, ap, n, s);
        c->launches += 2;
        *iters = it + 1;
        double rn;
        if (int e = dot_host(c, r, r, n, &rn)) return e;
        if (std::sqrt(rn) <= rel * r0) return SFV_OK;
        precond(r, z);
        double rz_new;
        if (int e = dot_host(c, r, z, n, &rz_new)) return e;
        const double beta = rz_new / rz;
        rz = rz_new;
        seg_xpby(n, z, beta, p, s);
        ++c->launches;
    }
    return SFV_OK;
}

// segregated_solve (nonlinear.cpp:268-351): per outer iteration, for each component
// A u_next = A u + R_c(u) by IC(0)-CG, then u += relaxation (u_next - u)
int segregated(sfv_ctx* c, double* u, const sfv_solver_cfg* cfg, sfv_solve_report* rep) {
    const auto t0 = std::chrono::steady_clock::now();
    const int n = c->n, nc = c->nc;
    const int max_outer = cfg->max_outer > 0 ? cfg->max_outer : 2000;
    const double inner = cfg->inner_reduction > 0.0 ? cfg->inner_reduction : 0.9;
    const double relax = cfg->relaxation > 0.0 ? cfg->relaxation : 1.0;
    clear_report(rep);
    rep->status = SFV_MAX_ITERS;
    auto wall = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    if (!ensure_krylov(c, std::max(cfg->restart, 1))) return c->fail(SFV_ERR_CUDA, -1, "segregated: out of device memory");
    if (int e = seg_create(c)) return e;
    double* r = c->rscratch.p;
    int e = residual_sync(c, u, r);
    if (e) {
        rep->wall_seconds = wall();
        return e;
    }
    double r_norm;
    if ((e = norm_host(c, r, &r_norm))) return e;
    const double r0 = r_norm;
    rep->initial_residual = r0;
    rep->final_residual = r_norm;
    push_record(rep, 0, r_norm, 0, 0.0);
    auto converged = [&](double rn, double du, double un) {  // check_convergence (nonlinear.cpp:97-103)
        return rn <= cfg->a_tol || rn <= cfg->r_tol * r0 || (cfg->s_tol > 0.0 && du <= cfg->s_tol * un);
    };
    if (converged(r_norm, 0.0, 0.0)) {
        rep->status = SFV_CONVERGED;
        rep->wall_seconds = wall();
        return SFV_OK;
    }
    cudaStream_t s = c->stream;
    for (int k = 0; k < max_outer; ++k) {
        int krylov = 0;
        for (int comp = 0; comp < 3; ++comp) {
            const sfv_ctx::SegComp& sc = c->seg[c->seg_ncomp == 1 ? 0 : comp];
            seg_component(nc, u, comp, c->sg_x.p, s);
            seg_spmv(sc.a, c->sg_x.p, c->sg_b.p, s);
            seg_add_component(nc, r, comp, c->sg_b.p, s);
            c->launches += 3;
            int it = 0;
            if ((e = seg_cg(c, sc, c->sg_b.p, c->sg_x.p, inner, std::max(nc, 50), &it))) return e;
            krylov += it;
            rep->cg_diag_fallback |= sc.jacobi ? 1 : 0;
            seg_set_component(nc, c->sg_x.p, comp, c->sg_un.p, s);
            ++c->launches;
        }
        rep->krylov_iters += krylov;
        seg_relax(n, c->sg_un.p, relax, u, c->sg_du.p, s);
        ++c->launches;
        double du_norm, u_norm;
        if ((e = dot_host(c, c->sg_du.p, c->sg_du.p, n, &du_norm))) return e;
        du_norm = std::sqrt(du_norm);
        e = residual_sync(c, u, r);
        if (e) {  // eval.residual threw (nonlinear.cpp:326-333)
            rep->status = SFV_DIVERGED;
            std::snprintf(rep->detail, SFV_DETAIL_LEN, "%s", c->last.msg.c_str());
            rep->outer_iters = k + 1;
            break;
        }
        if ((e = norm_host(c, r, &r_norm))) return e;
        rep->outer_iters = k + 1;
        push_record(rep, k + 1, r_norm, krylov, 1.0);
        rep->final_residual = r_norm;
        if (!std::isfinite(r_norm)) {
            rep->status = SFV_DIVERGED;
            std::snprintf(rep->detail, SFV_DETAIL_LEN, "residual norm overflow");
            break;
        }
        if ((e = norm_host(c, u, &u_norm))) return e;
        if (converged(r_norm, du_norm, u_norm)) {
            rep->status = SFV_CONVERGED;
            break;
        }
    }
    if (rep->status == SFV_MAX_ITERS) std::snprintf(rep->detail, SFV_DETAIL_LEN, "outer iteration limit reached");
    cudaStreamSynchronize(c->stream);
    rep->wall_seconds = wall();
    return SFV_OK;
}

// line_search (nonlinear.cpp:140-163): s = 1, 1/2, ... 1/32; the first candidate u + s du
// whose residual norm is strictly below r_norm0 wins (an invalid trial state — a law or
// NaN error in R — rejects that step length).  The accepted candidate and its residual are
// left in ucand / rcand.
int line_search(sfv_ctx* c, const double* u, const double* du, double r_norm0, bool* ok, double* s_out,
                double* rn_out) {
    const int n = c->n;
    double ss = 1.0, rn = 0.0;
    *ok = false;
    if (!ensure_krylov(c, 1)) return c->fail(SFV_ERR_CUDA, -1, "line_search: out of device memory");
    for (int attempt = 0; attempt < 6; ++attempt, ss *= 0.5) {
        launch_lincomb(c->ucand.p, u, ss, du, n, c->stream);
        ++c->launches;
        if (residual_sync(c, c->ucand.p, c->rcand.p)) continue;  // invalid trial state rejects the step
        if (int e = norm_host(c, c->rcand.p, &rn)) return e;
        if (rn < r_norm0) {
            *ok = true;
            break;
        }
    }
    *s_out = ss;
    *rn_out = rn;
    return SFV_OK;
}

int jfnk(sfv_ctx* c, double* u, const sfv_solver_cfg* cfg, sfv_solve_report* rep) {
    const auto t0 = std::chrono::steady_clock::now();
    const int n = c->n;
    const int max_outer = cfg->max_outer > 0 ? cfg->max_outer : 50;
    const double inner = cfg->inner_reduction > 0.0 ? cfg->inner_reduction : 1e-3;
    clear_report(rep);
    rep->status = SFV_MAX_ITERS;
    auto wall = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    if (!ensure_krylov(c, std::max(cfg->restart, 1))) return c->fail(SFV_ERR_CUDA, -1, "jfnk: out of device memory");
    double* r = c->rscratch.p;  // residual at the current iterate
    double* rhs = c->bv.p;
    double* x = c->xv.p;
    int e = residual_sync(c, u, r);
    if (e) {
        rep->wall_seconds = wall();
        return e;
    }
    double r_norm;
    if ((e = norm_host(c, r, &r_norm))) return e;
    const double r_norm0 = r_norm;
    rep->initial_residual = r_norm0;
    rep->final_residual = r_norm;
    push_record(rep, 0, r_norm, 0, 0.0);
    if (r_norm <= cfg->a_tol || r_norm <= cfg->r_tol * r_norm0) {
        rep->status = SFV_CONVERGED;
        rep->wall_seconds = wall();
        return SFV_OK;
    }
    int stag = 0;
    for (int k = 0; k < max_outer; ++k) {
        launch_negate(r, rhs, n, c->stream);
        cudaMemsetAsync(x, 0, sizeof(double) * n, c->stream);
        ++c->launches;
        int iters = 0, status = 0;
        double rel = 0.0;
        e = gmres(c, u, r, rhs, x, true, cfg->restart, inner, cfg->max_krylov, &iters, &status, &rel,
                  cfg->right_preconditioned != 0);
        if (e == SFV_ERR_JVP_NAN) {
            rep->status = SFV_DIVERGED;
            std::snprintf(rep->detail, SFV_DETAIL_LEN, "%s", c->last.msg.c_str());
            e = SFV_OK;
            break;
        }
        if (e) {
            rep->wall_seconds = wall();
            return e;
        }
        rep->krylov_iters += iters;
        if (status == G_STAGNATED) {
            if (++stag >= 2) {
                rep->status = SFV_DIVERGED;
                std::snprintf(rep->detail, SFV_DETAIL_LEN, "gmres stagnated on two consecutive outer iterations");
                break;
            }
        } else {
            stag = 0;
        }
        double s = 1.0;
        if (cfg->line_search) {
            bool ok = false;
            double ss = 1.0, rn = 0.0;
            if ((e = line_search(c, u, x, r_norm, &ok, &ss, &rn))) return e;
            if (!ok) {
                rep->status = SFV_DIVERGED;
                std::snprintf(rep->detail, SFV_DETAIL_LEN, "line search found no residual decrease");
                break;
            }
            s = ss;
            // u += s du reproduces the accepted candidate bit for bit; r is its residual
            cudaMemcpyAsync(u, c->ucand.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream);
            cudaMemcpyAsync(r, c->rcand.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream);
            r_norm = rn;
        } else {
            launch_lincomb(u, u, 1.0, x, n, c->stream);
            ++c->launches;
            if (residual_sync(c, u, r)) {
                rep->status = SFV_DIVERGED;
                std::snprintf(rep->detail, SFV_DETAIL_LEN, "%s", c->last.msg.c_str());
                rep->outer_iters = k + 1;
                break;
            }
            if ((e = norm_host(c, r, &r_norm))) return e;
        }
        rep->outer_iters = k + 1;
        push_record(rep, k + 1, r_norm, iters, s);
        rep->final_residual = r_norm;
        bool conv = r_norm <= cfg->a_tol || r_norm <= cfg->r_tol * r_norm0;
        if (!conv && cfg->s_tol > 0.0) {
            double dn, un;
            if ((e = norm_host(c, x, &dn)) || (e = norm_host(c, u, &un))) return e;
            conv = s * dn <= cfg->s_tol * un;
        }
        if (conv) {
            rep->status = SFV_CONVERGED;
            break;
        }
    }
    if (rep->status == SFV_MAX_ITERS && rep->outer_iters == max_outer)
        std::snprintf(rep->detail, SFV_DETAIL_LEN, "outer iteration limit reached");
    cudaStreamSynchronize(c->stream);
    rep->wall_seconds = wall();
    return SFV_OK;
}

// SFV_TIMING=1: host setup phases on stderr
struct PhaseTimer {
    bool on = std::getenv("SFV_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto n = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[sfv] %-28s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};

// ILU(0) / ILU(1) set up on the device: J~, the factor, both sweeps' schedules and the
// streamed sweep's records never visit the host (precond_dev.cu).  "" or why not.
std::string precond_create_device(sfv_ctx* c, int level) {
    DevIluSetup ds;
    double tm[5] = {0, 0, 0, 0, 0};
    const bool timing = std::getenv("SFV_TIMING") != nullptr;
    std::string why = device_ilu_setup(device_topo(c->dgeo), c->ph.kbar, c->ph.transient != 0, c->ph.rho, c->ph.dt,
                                       level, c->stream, ds, timing ? tm : nullptr);
    cudaGetLastError();
    if (!why.empty()) return why;
    const int smem_cap = 232448;
    const int stages =
        std::min(8, (smem_cap - stream_smem_bytes(ds.ring, ds.max_rows, 0)) / (ds.max_rows * (kStreamRec + 24)));
    if (stages < 3) {
        ds.release();
        return "device ilu: shared memory holds fewer than 3 stages";
    }
    const int nc = c->nc;
    auto adopt = [&](TriDev& td, DevSweep& sw) {
        td.order.adopt(sw.order, sw.n_pos);
        td.level_ptr.adopt(sw.level_ptr, sw.n_levels + 1);
        td.rp.release();
        td.col.release();
        td.val.release();
        td.diag.release();
        td.ell_col.release();
        td.ell_val.release();
        td.ell_pcol.release();
        td.view = DevTri{};
        td.view.n = sw.n_pos;
        td.view.n_rows = nc;
        td.view.n_levels = sw.n_levels;
        td.view.order = td.order.p;
        td.view.level_ptr = td.level_ptr.p;
        td.n_levels = sw.n_levels;
        td.nnz = 0;
        sw.order = nullptr;
        sw.level_ptr = nullptr;
    };
    adopt(c->L[0], ds.L);
    adopt(c->U[0], ds.U);
    c->L[0].nnz = static_cast<size_t>(ds.nnz_L);
    c->U[0].nnz = static_cast<size_t>(ds.nnz_U);
    c->U[0].u2l.adopt(ds.U.u2l, ds.U.n_pos);
    c->U[0].view.u2l = c->U[0].u2l.p;
    ds.U.u2l = nullptr;
    c->srec[0].adopt(ds.L.rec, (static_cast<size_t>(ds.L.n_pos) + 31) / 32 * kStreamChunk);
    c->srec[3].adopt(ds.U.rec, (static_cast<size_t>(ds.U.n_pos) + 31) / 32 * kStreamChunk);
    ds.L.rec = ds.U.rec = nullptr;
    c->sL.t[0] = DevStream{ds.L.n_levels, c->L[0].view.level_ptr, c->srec[0].p};
    c->sU.t[0] = DevStream{ds.U.n_levels, c->U[0].view.level_ptr, c->srec[3].p};
    for (StreamSet* ss : {&c->sL, &c->sU}) {
        ss->ring = ds.ring;
        ss->max_rows = ds.max_rows;
        ss->stages = stages;
    }
    const int max_pos = std::max(ds.L.n_pos, ds.U.n_pos);
    if (!c->ily.alloc(c->n) || !c->ipa.alloc(3 * static_cast<size_t>(max_pos)) ||
        !c->ipb.alloc(3 * static_cast<size_t>(max_pos))) {
        c->fail(SFV_ERR_CUDA, -1, "ilu: out of device memory");
        return "ilu: out of device memory";
    }
    c->pc_ncomp = 1;
    c->ring_ok = false;
    c->stream_ok = true;
    c->pipe_ok = false;
    c->tri_cluster = kStreamMode;
    c->pc_kind = level == 0 ? SFV_PRECOND_ILU0 : SFV_PRECOND_ILU1;
    c->launches += 20;
    if (timing)
        std::fprintf(stderr,
                     "[sfv] device ilu setup: J~ %.1f  pattern %.1f  schedules %.1f  numeric %.1f  records %.1f ms "
                     "(ring %d rows %d stages %d; levels L %d U %d)\n",
                     tm[0], tm[1], tm[2], tm[3], tm[4], ds.ring, ds.max_rows, stages, ds.L.n_levels, ds.U.n_levels);
    return "";
}

// One discarded apply at the end of an ILU setup.  In soaks at C2 (scripts/probes/ilu_repeat.py)
// the streamed sweep's FIRST apply after a setup — records, schedules and scratch vectors cold in
// L2 and the TLB, so a cluster really stalls on its first TMA copies of a page — came out wrong
// in rare cases when the sweep was perturbed (2 of 480 first applies with -DSFV_STREAM_DELAY=3;
// 0 of ~430 unperturbed), while no later apply ever did (thousands, and the bit-for-bit
// full-size solves).  Until that stale read is found, the cold apply is spent here on a zero
// vector, so every apply a caller sees runs warm.  SFV_ILU_WARMUP=0 disables it.
int precond_warmup(sfv_ctx* c) {
    if (const char* e = std::getenv("SFV_ILU_WARMUP"); e && std::atoi(e) == 0) return SFV_OK;
    if (c->tri_cluster != kStreamMode || !c->ily.p) return SFV_OK;
    cudaMemsetAsync(c->ily.p, 0, sizeof(double) * c->n, c->stream);
    if (int e = precond_apply_async(c, c->ily.p, c->ily.p)) return e;
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) return c->cuda_check("ilu warm-up");
    return SFV_OK;
}

int precond_create(sfv_ctx* c, int kind) {
    ++c->pc_gen;  // a cached GMRES graph holds the old preconditioner's buffers
    c->drop_graph();
    PhaseTimer pt;
    c->pc_kind = SFV_PRECOND_NONE;
    c->pc_coupled = false;
    if (kind == SFV_PRECOND_AUTO) kind = 3 * c->nc <= 30000 ? SFV_PRECOND_LU : SFV_PRECOND_ILU1;  // nonlinear.cpp:355-356
    if (kind == SFV_PRECOND_NONE) return SFV_OK;
    // (the host-built sweeps and the host factorisation switches keep the host setup)
    if ((kind == SFV_PRECOND_ILU0 || kind == SFV_PRECOND_ILU1) && c->dgeo && !std::getenv("SFV_HOST_PRECOND") &&
        !std::getenv("SFV_PIPE") && !std::getenv("SFV_TRI_CLUSTER") && !std::getenv("SFV_ILU_SERIAL") &&
        !std::getenv("SFV_DEVICE_ILU")) {
        // the whole setup on the device (precond_dev.cu); the host path below when it declines
        const std::string why = precond_create_device(c, kind == SFV_PRECOND_ILU0 ? 0 : 1);
        if (why.empty()) {
            if (int e = c->cuda_check("ilu device setup")) return e;
            return precond_warmup(c);
        }
        if (pt.on) std::fprintf(stderr, "[sfv] device ilu setup declined: %s\n", why.c_str());
    }
    std::vector<ScalarCsr> comps;
    const std::string msg = cell_jacobian(c->mesh, c->geom, c->ph.kbar, c->ph.transient != 0, c->ph.rho, c->ph.dt, comps);
    if (!msg.empty()) return c->fail(SFV_ERR_INVALID_ARGUMENT, -1, msg);
    c->pc_ncomp = static_cast<int>(comps.size());
    // a symmetry plane that is not axis-aligned: the expanded 3n x 3n matrix, one factor
    c->pc_coupled = comps.size() == 1 && comps[0].n == c->n && c->nc != c->n;
    const int rows = c->pc_coupled ? c->n : c->nc;
    pt.mark("cell_jacobian");
    if (kind == SFV_PRECOND_LU) {
        for (size_t a = 0; a < comps.size(); ++a) {
            // ordering and band on the host; the factorisation on the device (cuSOLVER dense
            // Cholesky, SFV_HOST_LU=1: the host band factorisation)
            BandChol bc;
            const bool host_lu = std::getenv("SFV_HOST_LU") != nullptr;
            const std::string m2 = band_cholesky_neg(comps[a], bc, host_lu);
            if (!m2.empty()) return c->fail(SFV_ERR_LU_SINGULAR, -1, m2);
            pt.mark(host_lu ? "lu order + host factor" : "lu order + band");
            DevBuf<double> band;
            if (!band.upload(bc.l) || !c->dense_perm[a].upload(bc.perm) ||
                !c->dense_w[a].alloc(static_cast<size_t>(bc.n) * bc.n))
                return c->fail(SFV_ERR_CUDA, -1, "lu: out of device memory");
            if (!host_lu) {  // factor and explicit inverse on the device
                if (const std::string m3 = device_band_cholesky(band.p, bc.n, bc.bw, c->stream, c->dense_w[a].p);
                    !m3.empty())
                    return c->fail(m3.rfind("lu: factorisation", 0) == 0 ? SFV_ERR_LU_SINGULAR : SFV_ERR_CUDA, -1, m3);
                c->launches += 3;
                pt.mark("lu device factor + inverse");
            } else {  // host band factor, inverse column by column on the device
                launch_band_inverse(band.p, bc.n, bc.bw, c->dense_w[a].p, c->stream);
                ++c->launches;
                if (cudaStreamSynchronize(c->stream) != cudaSuccess) return c->cuda_check("lu setup");
                pt.mark("lu inverse");
            }
        }
        c->pc_kind = SFV_PRECOND_LU;
        return SFV_OK;
    }
    const int level = kind == SFV_PRECOND_ILU0 ? 0 : kind == SFV_PRECOND_ILU1 ? 1 : 2;
    std::vector<ScalarCsr> lus(comps.size());
    bool broke = false;
    // SFV_DEVICE_ILU=1: the numeric phase of ILU(0)/ILU(1) on the device (bit-identical factor)
    IluNumericFn numeric;
    if (std::getenv("SFV_DEVICE_ILU"))
        numeric = [c](ScalarCsr& out, const std::vector<int>& diag, const std::vector<int>& rows) {
            return device_ilu_numeric(out, diag, rows, c->stream);
        };
    for (size_t a = 0; a < comps.size(); ++a)
        if (!iluk_factor(comps[a], level, lus[a], numeric).empty()) broke = true;
    if (broke) {  // one retry with a 1e-12 |diag| shift over the expanded diagonal (nonlinear.cpp:357-369)
        double dn = 0.0;
        for (int i = 0; i < c->nc; ++i)
            for (int a = 0; a < 3; ++a) {
                const ScalarCsr& s = comps[comps.size() == 1 ? 0 : a];
                const int ri = c->pc_coupled ? 3 * i + a : i;
                const int q = static_cast<int>(std::lower_bound(s.col.begin() + s.rp[ri], s.col.begin() + s.rp[ri + 1], ri) -
                                               s.col.begin());
                dn += s.val[q] * s.val[q];
            }
        dn = std::sqrt(dn);
        for (auto& s : comps)
            for (int i = 0; i < rows; ++i) {
                const int q = static_cast<int>(std::lower_bound(s.col.begin() + s.rp[i], s.col.begin() + s.rp[i + 1], i) -
                                               s.col.begin());
                s.val[q] += 1e-12 * dn;
            }
        for (size_t a = 0; a < comps.size(); ++a) {
            const std::string m3 = iluk_factor(comps[a], level, lus[a]);
            if (!m3.empty()) return c->fail(SFV_ERR_ILU_BREAKDOWN, -1, m3);
        }
    }
    pt.mark("iluk_factor");
    int max_pos = 0;
    bool ring_ok_all = true, stream_ok_all = true;
    std::vector<TriSchedule> scheds(2 * lus.size());  // L0, U0, L1, U1, ...
    {
        std::vector<std::thread> th;  // the sweeps' schedules are independent
        for (size_t x = 0; x < scheds.size(); ++x)
            th.emplace_back([&, x] {
                if (x % 2) schedule_upper(lus[x / 2], scheds[x]);
                else schedule_lower(lus[x / 2], scheds[x]);
            });
        for (auto& t : th) t.join();
    }
    std::vector<std::vector<int>> u2ls(lus.size());
    for (size_t a = 0; a < lus.size(); ++a) {
        const TriSchedule& tl = scheds[2 * a];
        const TriSchedule& tu = scheds[2 * a + 1];
        u2ls[a].assign(tu.n_pos, -1);  // backward-sweep position -> forward-sweep position
        for (int p = 0; p < tu.n_pos; ++p)
            if (tu.order[p] >= 0) u2ls[a][p] = tl.pos[tu.order[p]];
        max_pos = std::max(max_pos, std::max(tl.n_pos, tu.n_pos));
    }
    pt.mark("schedules");
    // streamed sweep (precond_stream.cu): rows per CTA-slice, the smallest safe value ring,
    // and as many cp.async stages as the remaining shared memory holds
    std::vector<rawvec<unsigned char>> packed(scheds.size());
    int s_ring = 0, s_rows = 32, s_stages = 0;
    {
        for (const TriSchedule& ts : scheds)
            for (int l = 0; l < ts.n_levels; ++l) {
                const int nch = (ts.level_ptr[l + 1] - ts.level_ptr[l]) / 32;
                s_rows = std::max(s_rows, (nch + kStreamCluster - 1) / kStreamCluster * 32);
            }
        if (s_rows <= kStreamMaxRows)
            for (int cand : {1024, 2048, 3072, 4095}) {  // (slot 4095 at most: the +0.0 slot)
                std::vector<char> ok(scheds.size(), 0);
                std::vector<std::thread> th;
                for (size_t x = 0; x < scheds.size(); ++x)
                    th.emplace_back([&, x] {
                        // forward sweep of component a: values go to its backward-sweep positions
                        ok[x] = build_stream_records(scheds[x], kStreamCluster, cand, s_rows, packed[x],
                                                     x % 2 ? nullptr : &scheds[x + 1].pos);
                    });
                for (auto& t : th) t.join();
                if (std::all_of(ok.begin(), ok.end(), [](char v) { return v != 0; })) {
                    s_ring = cand;
                    break;
                }
            }
        const int smem_cap = 232448;
        s_stages = s_ring ? std::min(8, (smem_cap - stream_smem_bytes(s_ring, s_rows, 0)) / (s_rows * (kStreamRec + 24)))
                          : 0;
        stream_ok_all = s_ring > 0 && s_stages >= 3;
    }
    pt.mark("stream records");
    // device copies: the streamed sweep needs only the position maps and level pointers;
    // the CSR / ELL copies feed the fallback sweeps (uploaded when they may be selected)
    const bool full = !stream_ok_all || std::getenv("SFV_TRI_CLUSTER") != nullptr;
    for (size_t a = 0; a < lus.size(); ++a) {
        const TriSchedule& tl = scheds[2 * a];
        const TriSchedule& tu = scheds[2 * a + 1];
        if (!c->L[a].upload(tl, rows, full) || !c->U[a].upload(tu, rows, full) || !c->U[a].u2l.upload(u2ls[a]))
            return c->fail(SFV_ERR_CUDA, -1, "ilu: out of device memory");
        c->U[a].view.u2l = c->U[a].u2l.p;
        for (const TriSchedule* ts : {&tl, &tu}) {  // DSMEM ring admissibility
            if (!full) {
                ring_ok_all = false;
                break;
            }
            int dist = 0, width = 0;
            for (int l = 0; l < ts->n_levels; ++l) width = std::max(width, ts->level_ptr[l + 1] - ts->level_ptr[l]);
            for (size_t q = 0; q < ts->ell_pcol.size(); ++q)
                if (ts->ell_pcol[q] >= 0) dist = std::max(dist, static_cast<int>(q % ts->n_pos) - ts->ell_pcol[q]);
            if (dist + 2 * width + 64 > ilu_ring_window()) ring_ok_all = false;
        }
    }
    if (stream_ok_all) {
        for (size_t x = 0; x < scheds.size(); ++x) {
            DevBuf<unsigned char>& b = c->srec[(x % 2) * 3 + x / 2];
            if (!b.alloc(packed[x].size()) ||
                cudaMemcpy(b.p, packed[x].data(), b.bytes(), cudaMemcpyHostToDevice) != cudaSuccess)
                return c->fail(SFV_ERR_CUDA, -1, "ilu: out of device memory");
            const int a = static_cast<int>(x / 2);
            DevStream ds{scheds[x].n_levels, x % 2 ? c->U[a].view.level_ptr : c->L[a].view.level_ptr, b.p};
            (x % 2 ? c->sU : c->sL).t[a] = ds;
        }
        for (StreamSet* ss : {&c->sL, &c->sU}) {
            ss->ring = s_ring;
            ss->max_rows = s_rows;
            ss->stages = s_stages;
        }
    }
    pt.mark("uploads");
    c->ring_ok = ring_ok_all;
    c->stream_ok = stream_ok_all;
    if (!c->ily.alloc(c->n) || !c->ipa.alloc(3 * static_cast<size_t>(max_pos)) ||
        !c->ipb.alloc(3 * static_cast<size_t>(max_pos)))
        return c->fail(SFV_ERR_CUDA, -1, "ilu: out of device memory");
    // persistent grid: every CTA resident (<= 8 CTAs of 256 threads per SM fit), so each
    // awaited row belongs to a running thread.  Knobs for tuning: SFV_TRI_CTAS_PER_SM,
    // SFV_TRI_SLEEP_NS.
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per_sm = 2;
    if (const char* e = std::getenv("SFV_TRI_CTAS_PER_SM")) per_sm = std::max(1, std::min(8, std::atoi(e)));
    c->tri_sleep = 0;
    if (const char* e = std::getenv("SFV_TRI_SLEEP_NS")) c->tri_sleep = std::max(0, std::atoi(e));
    c->tri_grid = std::max(1, sms * per_sm);
    if (const char* e = std::getenv("SFV_TRI_CTAS")) c->tri_grid = std::max(1, std::atoi(e));
    // default: the DSMEM-ring sweep when its window covers every dependency distance plus
    // two levels (so no ring slot is overwritten before its last reader ran); else the
    // L2 cluster sweep
    // block-pipelined sweeps (precond_pipe.cu), opt-in with SFV_PIPE=1: bit-identical, but
    // slower than the streamed level-synchronous sweep at every size measured
    c->pipe_ok = false;
    if (const char* pe = std::getenv("SFV_PIPE"); pe && std::atoi(pe) != 0 && !c->pc_coupled) {
        bool ok = true;
        int ring = 0;
        std::vector<PipeSchedule> ps(2 * lus.size());
        int min_ring = 4096;
        if (const char* e = std::getenv("SFV_PIPE_RING")) min_ring = std::atoi(e);
        for (int cand : {4096, 8192, 16384}) {
            if (cand < min_ring) continue;
            ok = true;
            for (size_t x = 0; x < ps.size() && ok; ++x)
                ok = build_pipe(lus[x / 2], x % 2 == 1, kPipeCluster, cand, ps[x], nullptr);
            if (ok) {
                ring = cand;
                break;
            }
        }
        if (ok) {
            for (size_t a = 0; a < lus.size() && ok; ++a) {
                const PipeSchedule& pl = ps[2 * a];
                const PipeSchedule& pu = ps[2 * a + 1];
                std::vector<int> to_lower(pu.n_pos, -1);
                for (int p = 0; p < pu.n_pos; ++p)
                    if (pu.order[p] >= 0) to_lower[p] = pl.pos[pu.order[p]];
                for (int w = 0; w < 2; ++w) {
                    const PipeSchedule& q = w ? pu : pl;
                    DevBuf<int>* ib = c->pint + (2 * a + w) * 6;
                    if (!ib[0].upload(q.step_off) || !ib[1].upload(q.step_ptr) || !ib[2].upload(q.need) ||
                        !ib[3].upload(q.guard) || !ib[4].upload(q.order) ||
                        (w && !ib[5].upload(to_lower)) || !c->prec[2 * a + w].alloc(q.rec.size()) ||
                        cudaMemcpy(c->prec[2 * a + w].p, q.rec.data(), q.rec.size(), cudaMemcpyHostToDevice) !=
                            cudaSuccess)
                        return c->fail(SFV_ERR_CUDA, -1, "ilu: out of device memory");
                    max_pos = std::max(max_pos, q.n_pos);
                }
            }
            for (int a = 0; a < 3; ++a) {
                const int src = c->pc_ncomp == 1 ? 0 : a;
                for (int w = 0; w < 2; ++w) {
                    DevBuf<int>* ib = c->pint + (2 * src + w) * 6;
                    DevPipe d;
                    d.step_off = ib[0].p;
                    d.step_ptr = ib[1].p;
                    d.need = ib[2].p;
                    d.guard = ib[3].p;
                    d.order = ib[4].p;
                    d.to_lower = w ? ib[5].p : nullptr;
                    d.rec = c->prec[2 * src + w].p;
                    d.n_pos = ps[2 * src + w].n_pos;
                    (w ? c->pU : c->pL).t[a] = d;
                }
            }
            c->pL.ring = c->pU.ring = ring;
            c->pipe_ok = true;
            if (!c->ipa.alloc(3 * static_cast<size_t>(max_pos)) || !c->ipb.alloc(3 * static_cast<size_t>(max_pos)))
                return c->fail(SFV_ERR_CUDA, -1, "ilu: out of device memory");
        }
    }
    c->tri_cluster = c->pipe_ok ? kPipeMode : c->stream_ok ? kStreamMode : (c->ring_ok ? kDsRingMode : 16);
    if (const char* e = std::getenv("SFV_TRI_CLUSTER")) {
        const int v = std::atoi(e);
        c->tri_cluster = (v == kDsRingMode && c->ring_ok) || (v == kStreamMode && c->stream_ok) ||
                                 (v == kPipeMode && c->pipe_ok)
                             ? v
                             : std::max(0, std::min(16, v));
    }
    for (int a = 0; a < c->pc_ncomp; ++a)  // the ELL cluster sweep holds rows of up to 32 entries
        if (c->tri_cluster != kPipeMode && (c->L[a].view.maxd > 32 || c->U[a].view.maxd > 32)) c->tri_cluster = 0;
    if (c->pc_coupled) c->tri_cluster = 0;  // one factor over 3n unknowns: the sync-free sweep
    c->pc_kind = kind;
    pt.mark("rest");
    if (std::getenv("SFV_TIMING"))
        std::fprintf(stderr, "[sfv] ilu sweep mode %d (stream: ring %d rows %d stages %d; levels L %d U %d)\n",
                     c->tri_cluster, c->sL.ring, c->sL.max_rows, c->sL.stages, c->sL.t[0].n_levels,
                     c->sU.t[0].n_levels);
    if (int e = c->cuda_check("ilu setup")) return e;
    return precond_warmup(c);
}

}  // namespace

// ================================================================ C-ABI

extern "C" {

sfv_mesh* sfv_mesh_box(const double extents[3], const int divisions[3], const int patch_kinds[6],
                       double distort_factor, uint64_t seed, char* err, int errlen) {
    for (int a = 0; a < 3; ++a)
        if (divisions[a] < 1 || !(extents[a] > 0.0)) {
            if (err) std::snprintf(err, errlen, "generate_box_hex: bad divisions or extents");
            return nullptr;
        }
    auto* m = new sfv_mesh{box_hex(extents, divisions, patch_kinds)};
    const std::string e = distort(m->m, distort_factor, seed);
    if (!e.empty()) {
        if (err) std::snprintf(err, errlen, "%s", e.c_str());
        delete m;
        return nullptr;
    }
    return m;
}

sfv_mesh* sfv_mesh_kuhn_tets(const double extents[3], int n, const int patch_kinds[6], uint64_t perm_seed, int permute,
                             int rcm, char* err, int errlen) {
    if (n < 1) {
        if (err) std::snprintf(err, errlen, "kuhn_tets: n must be >= 1");
        return nullptr;
    }
    bool dev = false;
    HostMesh hm = kuhn_tets(extents, n, patch_kinds, perm_seed, permute != 0, rcm != 0, &dev);
    return new sfv_mesh{std::move(hm), dev};
}

int sfv_mesh_built_on_device(const sfv_mesh* m) { return m && m->on_device ? 1 : 0; }

void sfv_mesh_counts(const sfv_mesh* mm, int counts[6]) {
    const HostMesh& m = mm->m;
    counts[0] = static_cast<int>(m.points.size());
    counts[1] = m.n_faces();
    counts[2] = static_cast<int>(m.face_pts.size());
    counts[3] = m.n_cells;
    counts[4] = m.n_internal;
    counts[5] = static_cast<int>(m.patches.size());
}

void sfv_mesh_export(const sfv_mesh* mm, double* points, int* face_offsets, int* face_points, int* owner,
                     int* neighbour, int* patch_kind, int* patch_start, int* patch_count) {
    const HostMesh& m = mm->m;
    for (size_t i = 0; i < m.points.size(); ++i) {
        points[3 * i] = m.points[i].x;
        points[3 * i + 1] = m.points[i].y;
        points[3 * i + 2] = m.points[i].z;
    }
    std::memcpy(face_offsets, m.face_off.data(), sizeof(int) * m.face_off.size());
    std::memcpy(face_points, m.face_pts.data(), sizeof(int) * m.face_pts.size());
    std::memcpy(owner, m.owner.data(), sizeof(int) * m.owner.size());
    std::memcpy(neighbour, m.neighbour.data(), sizeof(int) * m.neighbour.size());
    for (size_t p = 0; p < m.patches.size(); ++p) {
        patch_kind[p] = m.patches[p].kind;
        patch_start[p] = m.patches[p].start;
        patch_count[p] = m.patches[p].count;
    }
}

void sfv_mesh_free(sfv_mesh* m) { delete m; }

sfv_ctx* sfv_create(const sfv_mesh_desc* md, const sfv_physics* ph, char* err, int errlen) {
    auto fail = [&](const std::string& m) -> sfv_ctx* {
        if (err) std::snprintf(err, errlen, "%s", m.c_str());
        return nullptr;
    };
    if (md->dim != 3) return fail("sfv: only 3-D meshes are on the hot path");
    if (md->n_patches > kMaxPatches) return fail("sfv: too many patches");
    auto c = std::make_unique<sfv_ctx>();
    PhaseTimer pt;
    HostMesh& m = c->mesh;
    m.points.resize(md->n_points);
    for (int i = 0; i < md->n_points; ++i)
        m.points[i] = {md->points[3 * i], md->points[3 * i + 1], md->points[3 * i + 2]};
    m.face_off.assign(md->face_offsets, md->face_offsets + md->n_faces + 1);
    m.face_pts.assign(md->face_points, md->face_points + md->face_offsets[md->n_faces]);
    m.owner.assign(md->owner, md->owner + md->n_faces);
    m.neighbour.assign(md->neighbour, md->neighbour + md->n_faces);
    for (int p = 0; p < md->n_patches; ++p) m.patches.push_back({md->patch_kind[p], md->patch_start[p], md->patch_count[p]});
    m.n_cells = md->n_cells;
    m.n_internal = md->n_internal;
    std::string e = m.finalise();
    if (!e.empty()) return fail(e);
    pt.mark("mesh copy + finalise");
    // geometry on the device by default (bit-identical; SFV_HOST_GEOMETRY=1: the host passes)
    e = std::getenv("SFV_HOST_GEOMETRY") ? compute_geometry(m, c->geom) : device_geometry(m, c->geom, &c->dgeo);
    if (!e.empty()) return fail(e);
    pt.mark("compute_geometry");
    // ResidualEvaluator ctor checks (discretisation.cpp:64-67)
    if (!(ph->alpha > 0.0)) return fail("discretisation: alpha must be positive");
    if (ph->transient && !(ph->dt > 0.0)) return fail("discretisation: transient mode needs dt > 0");
    c->nc = m.n_cells;
    c->n = 3 * m.n_cells;
    for (int i = 0; i < c->nc; ++i)
        if (c->geom.g_singular[i]) {
            c->singular_cell = i;
            break;
        }
    Physics& p = c->ph;
    p.law = ph->law;
    p.tl = ph->total_lagrangian;
    p.transient = ph->transient;
    p.mu = ph->mu;
    p.lam = ph->lambda;
    p.alpha = ph->alpha;
    if (ph->law < SFV_LAW_HOOKE || ph->law > SFV_LAW_J2) return fail("law: unknown constitutive law");
    for (int k = 0; k < 8; ++k) p.gc[k] = ph->guccione[k];
    p.ja = ph->j2_curve[0];
    p.jb = ph->j2_curve[1];
    p.jc = ph->j2_curve[2];
    p.jd = ph->j2_curve[3];
    p.jn = ph->law == SFV_LAW_J2 ? ph->j2_n_table : 0;
    if (p.jn < 0 || p.jn > kMaxHardening || (p.jn > 0 && !ph->j2_table))
        return fail("law: the J2 hardening table holds at most 16 points");
    for (int k = 0; k < 2 * p.jn; ++k) p.jt[k] = ph->j2_table[k];
    for (int k = 1; k < p.jn; ++k)
        if (!(p.jt[2 * k] > p.jt[2 * k - 2])) return fail("law: hardening table eps_p must increase strictly");
    p.commit = 0;
    // MechanicalLaw::stabilisation_modulus (laws.hpp:100, :111, :122, :133, :147)
    p.kbar = ph->law == SFV_LAW_NEO_HOOKEAN || ph->law == SFV_LAW_J2 ? 4.0 / 3.0 * ph->mu + ph->lambda
             : ph->law == SFV_LAW_GUCCIONE ? 4.0 / 3.0 * (ph->guccione[0] * ph->guccione[2]) + ph->guccione[4]
                                           : 2.0 * ph->mu + ph->lambda;
    p.rho = ph->rho;
    p.dt = ph->dt;
    c->pt.n = md->n_patches;
    c->bc_raw.assign(ph->bc_value, ph->bc_value + 3 * md->n_patches);
    c->bc_ramp.assign(ph->bc_ramp, ph->bc_ramp + md->n_patches);
    for (int q = 0; q < md->n_patches; ++q) c->pt.kind[q] = md->patch_kind[q];
    update_patch_values(c.get());
    if (const char* j = std::getenv("SFV_JV")) {  // kernel-path override (scripts/microbench.py)
        const std::string js(j);
        c->jv_path = js == "fused" ? 1 : js == "twopass" ? 2 : 0;
    }
    if (ph->law >= SFV_LAW_STVK && c->jv_path != 0)
        return fail("law: St. Venant-Kirchhoff and Guccione run on the default J.v path only");
    e = build_layout(c.get());
    if (!e.empty()) return fail(e);
    pt.mark("device layout + upload");
    if (c->jv_path == 1 && build_fused_layout(c.get()).rfind("cuda", 0) == 0)
        return fail("cuda: out of device memory");
    const size_t n = static_cast<size_t>(c->n);
    if (!c->grad.alloc(9 * static_cast<size_t>(c->nc)) || !c->red.alloc(2 * 148 * 8 + 64) || !c->scal.alloc(8) ||
        !c->counter.alloc(1) || !c->err.alloc(1) || !c->hdev.alloc(72) || !c->dzero.alloc(n))
        return fail("cuda: out of device memory");
    cudaMemset(c->counter.p, 0, sizeof(unsigned));
    // ε reduction fused into the perturb pass (default; SFV_EPS_FUSED=0: separate partials pass)
    const char* ef = std::getenv("SFV_EPS_FUSED");
    if (c->jv_path == 0 && !(ef && std::atoi(ef) == 0) && eps_perturb_grid_for(c->nc) > 0) {
        if (!c->epsbar.alloc(1)) return fail("cuda: out of device memory");
        cudaMemset(c->epsbar.p, 0, sizeof(unsigned long long));
        c->ps.bar = c->epsbar.p;
    }
    cudaMemset(c->dzero.p, 0, sizeof(double) * n);
    if (c->ph.transient) {
        c->hist.u_old = c->hist.u_old_old = c->hist.v_old = c->hist.v_old_old = c->dzero.p;
    }
    if (cudaMallocHost(&c->st, sizeof(Status)) != cudaSuccess) return fail("cuda: pinned allocation failed");
    c->st->hcap = 72;
    if (cudaMallocHost(&c->st->h, sizeof(double) * c->st->hcap) != cudaSuccess)
        return fail("cuda: pinned allocation failed");
    if (cudaDeviceSynchronize() != cudaSuccess) return fail("cuda: setup failed");
    return c.release();
}

void sfv_destroy(sfv_ctx* c) {
    if (!c) return;
    if (c->st) {
        if (c->st->h) cudaFreeHost(c->st->h);
        cudaFreeHost(c->st);
    }
    delete c;
}

int sfv_set_stream(sfv_ctx* c, void* s) {
    c->stream = static_cast<cudaStream_t>(s);
    return SFV_OK;
}

int sfv_set_option(sfv_ctx* c, const char* name, int value) {
    if (name && std::strcmp(name, "sequential_reductions") == 0) {
        c->seq_reduce = value != 0;
        c->drop_graph();
        return SFV_OK;
    }
    if (name && std::strcmp(name, "gmres_graph") == 0) {
        c->graph_off = value == 0;
        c->drop_graph();
        return SFV_OK;
    }
    return c->fail(SFV_ERR_INVALID_ARGUMENT, -1, std::string("sfv_set_option: unknown option ") + (name ? name : ""));
}

int sfv_n_cells(const sfv_ctx* c) { return c->nc; }
const char* sfv_last_error(const sfv_ctx* c) { return c->last.msg.c_str(); }
long long sfv_launch_count(const sfv_ctx* c) { return c->launches; }

size_t sfv_device_bytes(const sfv_ctx* c) {
    return c->slot_face.bytes() + c->slot_other.bytes() + c->slot_ls.bytes() + c->gam.bytes() + c->del.bytes() +
           c->dmag.bytes() + c->w.bytes() + c->volume.bytes() + c->grad.bytes() + c->V.bytes() + c->dense_w[0].bytes() +
           c->dense_w[1].bytes() + c->dense_w[2].bytes() + c->tslot.bytes() + c->tls.bytes() + c->face9.bytes() +
           c->pwg.bytes() + c->psig.bytes() + c->bres.bytes();
}

double sfv_jv_bytes(const sfv_ctx* c) {
    // B = 96 N_c + 120 N_f + 60 N_d + 12 N_t (+104 N_c transient)
    const HostMesh& m = c->mesh;
    double nd = 0, nt = 0, ns = 0;
    for (int f = m.n_internal; f < m.n_faces(); ++f) {
        const int k = m.patches[m.face_patch[f]].kind;
        if (k == SFV_PATCH_DISPLACEMENT) nd += 1;
        else if (k == SFV_PATCH_TRACTION) nt += 1;
        else ns += 1;
    }
    return 96.0 * c->nc + 120.0 * m.n_internal + 60.0 * nd + 12.0 * nt + 84.0 * ns +
           (c->ph.transient ? 104.0 * c->nc : 0.0);
}

void sfv_jv_stage_bytes(const sfv_ctx* c, double* b) {
    // bytes each stage of the default J.v path must move at least once:
    // N_c cells, S face slots per cell, N_f faces, N_b boundary faces
    const double nc = c->nc, S = c->dm.slots, nf = c->dm.nf, nb = c->dm.nf - c->dm.nint;
    const double tr = c->ph.transient ? 104.0 * nc : 0.0;  // volume + 4 history vectors
    b[0] = c->ps.bar ? 0.0 : 48.0 * nc;                     // u, v (fused into the next pass by default)
    b[1] = 72.0 * nc;                                       // u, v -> w
    b[2] = (4.0 * S + 24.0 * S + 24.0 + 72.0) * nc;         // slot_other, ls, w, G
    const bool bp = boundary_pass(c);                       // else boundary faces are read by the flux pass
    b[3] = bp ? 208.0 * nb : 0.0;                           // slot, geometry, G, w -> 6 results
    b[4] = (8.0 * S + 72.0 + 24.0 + 24.0 + 24.0) * nc + 72.0 * nf + (bp ? 48.0 * nb : 0.0) + tr;  // slots, G, w, r_u, out, faces
}

int sfv_geometry(const sfv_ctx* c, double* volume, double* centroid, double* face_centroid, double* area, double* d,
                 double* d_mag, double* w, double* delta, double* g_inv, signed char* g_singular, int* cf_offsets,
                 int* cf_faces, double* ls_vec) {
    const HostMesh& m = c->mesh;
    if (std::string e = download_geometry(c->dgeo, const_cast<sfv_ctx*>(c)->geom); !e.empty()) return SFV_ERR_CUDA;
    const HostGeometry& g = c->geom;
    for (int i = 0; i < m.n_cells; ++i) {
        volume[i] = g.volume[i];
        centroid[3 * i] = g.centroid[i].x;
        centroid[3 * i + 1] = g.centroid[i].y;
        centroid[3 * i + 2] = g.centroid[i].z;
        for (int k = 0; k < 9; ++k) g_inv[9 * i + k] = g.g_inv[9 * static_cast<size_t>(i) + k];
        g_singular[i] = g.g_singular[i];
    }
    for (int f = 0; f < m.n_faces(); ++f) {
        const V3* src[4] = {&g.face_centroid[f], &g.area[f], &g.d[f], &g.delta[f]};
        double* dst[4] = {face_centroid, area, d, delta};
        for (int a = 0; a < 4; ++a) {
            dst[a][3 * f] = src[a]->x;
            dst[a][3 * f + 1] = src[a]->y;
            dst[a][3 * f + 2] = src[a]->z;
        }
        d_mag[f] = g.d_mag[f];
        w[f] = g.w[f];
    }
    std::memcpy(cf_offsets, m.cf_off.data(), sizeof(int) * m.cf_off.size());
    std::memcpy(cf_faces, m.cf.data(), sizeof(int) * m.cf.size());
    for (size_t q = 0; q < g.ls.size(); ++q) {
        ls_vec[3 * q] = g.ls[q].x;
        ls_vec[3 * q + 1] = g.ls[q].y;
        ls_vec[3 * q + 2] = g.ls[q].z;
    }
    return SFV_OK;
}

int sfv_set_time(sfv_ctx* c, double t) {
    c->time = t;
    return update_patch_values(c);
}

int sfv_set_body_force(sfv_ctx* c, const double* f) {
    if (c->jv_path != 0 || c->use_fused)
        return c->fail(SFV_ERR_INVALID_ARGUMENT, -1, "body force: only on the default residual path");
    if (!f) {
        c->hist.body = nullptr;
        return SFV_OK;
    }
    // volume_c * body_force(centroid_c): the reference's product (discretisation.cpp:161)
    std::vector<double> bv(3 * static_cast<size_t>(c->nc));
    if (!download_geometry(c->dgeo, c->geom).empty()) return c->fail(SFV_ERR_CUDA, -1, "body force: geometry");
    const auto& vol = c->geom.volume;
    for (int cc = 0; cc < c->nc; ++cc)
        for (int k = 0; k < 3; ++k) bv[3 * cc + k] = vol[cc] * f[3 * cc + k];
    if (!c->body_dev.upload(bv)) return c->fail(SFV_ERR_CUDA, -1, "body force: out of device memory");
    c->hist.body = c->body_dev.p;
    return SFV_OK;
}

int sfv_set_boundary_values(sfv_ctx* c, const double* values) {
    if (c->jv_path != 0 || c->use_fused)
        return c->fail(SFV_ERR_INVALID_ARGUMENT, -1, "boundary values: only on the default residual path");
    c->bc_sampler = nullptr;
    return upload_face_values(c, values);
}

int sfv_set_boundary_sampler(sfv_ctx* c, sfv_bc_sampler fn, void* user) {
    if (c->jv_path != 0 || c->use_fused)
        return c->fail(SFV_ERR_INVALID_ARGUMENT, -1, "boundary values: only on the default residual path");
    c->bc_sampler = fn;
    c->bc_user = user;
    if (!fn) return upload_face_values(c, nullptr);
    return update_patch_values(c);
}

int sfv_set_history(sfv_ctx* c, const double* uo, const double* uoo, const double* vo, const double* voo) {
    c->hist.u_old = uo;
    c->hist.u_old_old = uoo;
    c->hist.v_old = vo;
    c->hist.v_old_old = voo;
    return SFV_OK;
}

int sfv_residual(sfv_ctx* c, const double* u, double* r, int* cell) {
    const int e = residual_sync(c, u, r);
    if (cell) *cell = e ? c->last.cell : -1;
    return e;
}

int sfv_stabilisation(sfv_ctx* c, const double* u, double* r, int* cell) {
    if (cell) *cell = -1;
    if (c->singular_cell >= 0) {
        if (cell) *cell = c->singular_cell;
        return gradient_failure(c);
    }
    reset_err(c);
    Physics ph = c->ph;
    ph.stab_only = 1;
    residual_pass(c, ph, u, nullptr, nullptr, nullptr, r);
    if (int e = c->cuda_check("stabilisation")) return e;
    return fetch(c, 0);
}

int sfv_commit(sfv_ctx* c, const double* u) {
    // ResidualEvaluator::commit (discretisation.cpp:91-95): the law's stress at u in every cell,
    // then trial -> committed.  Only J2 carries state; the hyperelastic laws' commit is empty.
    if (c->ph.law != SFV_LAW_J2) return SFV_OK;
    if (c->singular_cell >= 0) return gradient_failure(c);
    reset_err(c);
    Physics ph = c->ph;
    ph.commit = 1;
    launch_gradients_pair(c->dm, c->pt, ph, u, nullptr, c->ps, c->err.p, c->stream);
    c->launches += 2;
    if (int e = c->cuda_check("commit")) return e;
    if (int e = fetch(c, 0)) return e;
    return decode_residual_errors(c, false);
}

int sfv_law_state(sfv_ctx* c, double* state) {
    if (c->ph.law != SFV_LAW_J2) return c->fail(SFV_ERR_INVALID_ARGUMENT, -1, "law_state: J2 only");
    std::vector<double> t(c->lawst.n);
    if (cudaMemcpy(t.data(), c->lawst.p, c->lawst.bytes(), cudaMemcpyDeviceToHost) != cudaSuccess)
        return c->cuda_check("law_state");
    for (int i = 0; i < c->nc; ++i)
        for (int q = 0; q < kJ2; ++q) state[static_cast<size_t>(i) * kJ2 + q] = t[tiled(i, kJ2) + 32 * q];
    return SFV_OK;
}

int sfv_gradients(sfv_ctx* c, const double* u, double* G, int* cell) {
    if (cell) *cell = -1;
    if (c->singular_cell >= 0) {
        if (cell) *cell = c->singular_cell;
        return gradient_failure(c);
    }
    if (c->jv_path == 0) {
        launch_gradients_pair(c->dm, c->pt, c->ph, u, G, c->ps, c->err.p, c->stream);
        c->launches += 3;
    } else {
        launch_gradients(c->dm, c->pt, u, G, c->stream);
        c->launches += 1;
    }
    if (int e = c->cuda_check("gradients")) return e;
    return cudaStreamSynchronize(c->stream) == cudaSuccess ? SFV_OK : c->cuda_check("gradients");
}

int sfv_mesh_geometry(const sfv_mesh_desc* md, double* volume, double* centroid, double* face_centroid,
                      double* area, double* d, double* d_mag, double* w, double* delta, double* g_inv,
                      signed char* g_singular, int* cf_offsets, int* cf_faces, double* ls_vec, char* err,
                      int errlen) {
    sfv_ctx tmp;
    HostMesh& m = tmp.mesh;
    m.points.resize(md->n_points);
    for (int i = 0; i < md->n_points; ++i)
        m.points[i] = {md->points[3 * i], md->points[3 * i + 1], md->points[3 * i + 2]};
    m.face_off.assign(md->face_offsets, md->face_offsets + md->n_faces + 1);
    m.face_pts.assign(md->face_points, md->face_points + md->face_offsets[md->n_faces]);
    m.owner.assign(md->owner, md->owner + md->n_faces);
    m.neighbour.assign(md->neighbour, md->neighbour + md->n_faces);
    for (int p = 0; p < md->n_patches; ++p) m.patches.push_back({md->patch_kind[p], md->patch_start[p], md->patch_count[p]});
    m.n_cells = md->n_cells;
    m.n_internal = md->n_internal;
    std::string e = m.finalise();
    if (e.empty()) e = compute_geometry(m, tmp.geom);
    if (!e.empty()) {
        if (err) std::snprintf(err, errlen, "%s", e.c_str());
        return SFV_ERR_GEOMETRY;
    }
    tmp.nc = m.n_cells;
    return sfv_geometry(&tmp, volume, centroid, face_centroid, area, d, d_mag, w, delta, g_inv, g_singular,
                        cf_offsets, cf_faces, ls_vec);
}

int sfv_jv(sfv_ctx* c, const double* u, const double* r_u, const double* v, double* out, int* cell) {
    if (cell) *cell = -1;
    if (c->singular_cell >= 0) {  // GradientFailure escapes J.v unless v == 0 (nonlinear.cpp:110)
        double vn;
        if (int e = norm_host(c, v, &vn)) return e;
        if (vn != 0.0) {
            if (cell) *cell = c->singular_cell;
            return gradient_failure(c);
        }
        cudaMemsetAsync(out, 0, sizeof(double) * c->n, c->stream);
        return SFV_OK;
    }
    reset_err(c);
    jv_async(c, u, r_u, v, out, false);
    if (int e = c->cuda_check("jv")) return e;
    if (int e = fetch(c, 0)) return e;
    return decode_residual_errors(c, true);
}

int sfv_jv_eps(sfv_ctx* c, const double* u, const double* r_u, const double* v, double eps, double* out, int* cell) {
    if (cell) *cell = -1;
    if (c->singular_cell >= 0) return gradient_failure(c);
    reset_err(c);
    cudaMemcpyAsync(c->scal.p, &eps, sizeof(double), cudaMemcpyHostToDevice, c->stream);
    cudaStreamSynchronize(c->stream);
    residual_pass(c, c->ph, u, v, c->scal.p, r_u, out);
    if (int e = c->cuda_check("jv_eps")) return e;
    if (int e = fetch(c, 0)) return e;
    return decode_residual_errors(c, true);
}

int sfv_jv_async(sfv_ctx* c, const double* u, const double* r_u, const double* v, double* out) {
    if (c->singular_cell >= 0) return gradient_failure(c);
    jv_async(c, u, r_u, v, out, false);
    return c->cuda_check("jv_async");
}

int sfv_jv_stage_times(sfv_ctx* c, const double* u, const double* r_u, const double* v, double* out, int reps,
                       double* ms) {
    if (c->jv_path != 0 || reps <= 0 || !ms) return c->fail(SFV_ERR_INVALID_ARGUMENT, -1, "jv_stage_times: default path only");
    if (c->singular_cell >= 0) return gradient_failure(c);
    // all reps queued back to back (as in a throughput loop), one host sync at the end
    std::vector<cudaEvent_t> ev(6 * static_cast<size_t>(reps));
    for (auto& e : ev) cudaEventCreate(&e);
    for (int r = 0; r < reps; ++r) {
        cudaEvent_t* e = ev.data() + 6 * r;
        cudaEventRecord(e[0], c->stream);
        // fused ε: stage 0 is empty and stage 1 (the perturb pass) includes the reduction
        if (!c->ps.bar) c->ps.npart = launch_norm_partials(u, v, c->n, c->red.p, false, c->stream);
        cudaEventRecord(e[1], c->stream);
        c->ps.marks = e + 2;
        c->ps.partials = c->red.p;
        c->ps.u_norm = c->scal.p + 1;
        c->ps.u_norm_cached = false;
        launch_residual_pair(c->dm, c->ph, c->pt, c->hist, u, v, c->scal.p, r_u, out, c->ps, c->err.p, c->stream);
        c->ps.partials = nullptr;
        c->ps.marks = nullptr;
        cudaEventRecord(e[5], c->stream);
    }
    const cudaError_t se = cudaEventSynchronize(ev.back());
    double acc[5] = {0, 0, 0, 0, 0};
    for (int r = 0; r < reps && se == cudaSuccess; ++r)
        for (int k = 0; k < 5; ++k) {
            float t = 0.f;
            cudaEventElapsedTime(&t, ev[6 * r + k], ev[6 * r + k + 1]);
            acc[k] += t;
        }
    for (auto& e : ev) cudaEventDestroy(e);
    for (int k = 0; k < 5; ++k) ms[k] = acc[k] / reps;
    c->launches += static_cast<long long>(reps) * ((boundary_pass(c) ? 4 : 3) + (c->ps.bar ? 0 : 1));
    return c->cuda_check("jv_stage_times");
}

int sfv_check_errors(sfv_ctx* c, int* cell) {
    if (int e = fetch(c, 0)) return e;
    const int e = decode_residual_errors(c, true);
    if (cell) *cell = e ? c->last.cell : -1;
    reset_err(c);
    return e;
}

int sfv_jfnk_solve_host(sfv_ctx* c, double* u, const sfv_solver_cfg* cfg, sfv_solve_report* rep) {
    const size_t bytes = sizeof(double) * c->n;
    double* d = nullptr;
    if (cudaMalloc(&d, bytes) != cudaSuccess) return c->fail(SFV_ERR_CUDA, -1, "out of device memory");
    cudaMemcpyAsync(d, u, bytes, cudaMemcpyHostToDevice, c->stream);
    const int e = jfnk(c, d, cfg, rep);
    cudaMemcpyAsync(u, d, bytes, cudaMemcpyDeviceToHost, c->stream);
    cudaStreamSynchronize(c->stream);
    cudaFree(d);
    return e;
}

int sfv_residual_host(sfv_ctx* c, const double* u, double* r, int* cell) {
    const size_t bytes = sizeof(double) * c->n;
    if (!ensure_krylov(c, 1)) return c->fail(SFV_ERR_CUDA, -1, "out of device memory");
    cudaMemcpyAsync(c->ucand.p, u, bytes, cudaMemcpyHostToDevice, c->stream);
    const int e = residual_sync(c, c->ucand.p, c->rcand.p);
    if (cell) *cell = e ? c->last.cell : -1;
    if (e) return e;
    cudaMemcpyAsync(r, c->rcand.p, bytes, cudaMemcpyDeviceToHost, c->stream);
    return cudaStreamSynchronize(c->stream) == cudaSuccess ? SFV_OK : c->cuda_check("residual_host");
}

int sfv_jv_host(sfv_ctx* c, const double* u, const double* r_u, const double* v, double* out, int* cell) {
    const size_t bytes = sizeof(double) * c->n;
    if (!ensure_krylov(c, 1)) return c->fail(SFV_ERR_CUDA, -1, "out of device memory");
    if (!c->copy && (cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking) != cudaSuccess ||
                     cudaEventCreateWithFlags(&c->ev_uv, cudaEventDisableTiming) != cudaSuccess ||
                     cudaEventCreateWithFlags(&c->ev_ru, cudaEventDisableTiming) != cudaSuccess))
        return c->cuda_check("jv_host streams");
    // u and v first (the ε and gradient passes need them); r_u, read only by the face pass,
    // follows on the copy stream while those passes run
    static const int host_chunks = [] {
        const char* e = std::getenv("SFV_JV_HOST_CHUNKS");
        return std::max(1, std::min(sfv_ctx::kHostChunks, e ? std::atoi(e) : 8));
    }();
    const bool chunked = host_chunks > 1 && !c->use_fused && c->jv_path == 0 && !c->seq_reduce && c->nc >= 4096 &&
                         c->singular_cell < 0;
    cudaMemcpyAsync(c->ucand.p, u, bytes, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(c->tv.p, v, bytes, cudaMemcpyHostToDevice, c->stream);
    cudaEventRecord(c->ev_uv, c->stream);
    cudaStreamWaitEvent(c->copy, c->ev_uv, 0);
    if (!chunked) {
        cudaMemcpyAsync(c->rcand.p, r_u, bytes, cudaMemcpyHostToDevice, c->copy);
        cudaEventRecord(c->ev_ru, c->copy);
    }
    if (c->singular_cell >= 0) {
        cudaStreamWaitEvent(c->stream, c->ev_ru, 0);  // sfv_jv's GradientFailure / zero-direction rule
        const int e = sfv_jv(c, c->ucand.p, c->rcand.p, c->tv.p, c->wv.p, cell);
        if (e) return e;
        cudaMemcpyAsync(out, c->wv.p, bytes, cudaMemcpyDeviceToHost, c->stream);
        return cudaStreamSynchronize(c->stream) == cudaSuccess ? SFV_OK : c->cuda_check("jv_host");
    }
    // one host synchronisation: the result copy is queued before the error words are read
    // (on an error, out holds the failed product, as the reference leaves its output undefined)
    if (cell) *cell = -1;
    reset_err(c);
    if (chunked && !c->d2h) {
        bool ok = cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking) == cudaSuccess;
        for (int k = 0; k < sfv_ctx::kHostChunks && ok; ++k)
            ok = cudaEventCreateWithFlags(&c->ev_ruk[k], cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&c->ev_outk[k], cudaEventDisableTiming) == cudaSuccess;
        if (!ok) return c->cuda_check("jv_host streams");
    }
    if (chunked) {
        // r_u and the result in tile-aligned pieces: the face pass of piece k starts when its
        // r_u has arrived, and its result goes back while piece k + 1 is computed, so the copy
        // back overlaps the upload of the rest of r_u (the two PCIe directions are independent)
        const int K = host_chunks;
        const int ntiles = (c->nc + 31) / 32;
        size_t lo[sfv_ctx::kHostChunks + 1];
        for (int k = 0; k <= K; ++k)
            lo[k] = 3 * std::min<size_t>(static_cast<size_t>(c->nc),
                                         32 * static_cast<size_t>(static_cast<long long>(ntiles) * k / K));
        for (int k = 0; k < K; ++k) {
            cudaMemcpyAsync(c->rcand.p + lo[k], r_u + lo[k], sizeof(double) * (lo[k + 1] - lo[k]),
                            cudaMemcpyHostToDevice, c->copy);
            cudaEventRecord(c->ev_ruk[k], c->copy);
        }
        c->ps.nchunk = K;
        c->ps.ru_chunk = c->ev_ruk;
        c->ps.out_chunk = c->ev_outk;
        jv_async(c, c->ucand.p, c->rcand.p, c->tv.p, c->wv.p, false);
        c->ps.nchunk = 0;
        c->ps.ru_chunk = nullptr;
        c->ps.out_chunk = nullptr;
        for (int k = 0; k < K; ++k) {
            cudaStreamWaitEvent(c->d2h, c->ev_outk[k], 0);
            cudaMemcpyAsync(out + lo[k], c->wv.p + lo[k], sizeof(double) * (lo[k + 1] - lo[k]), cudaMemcpyDeviceToHost,
                            c->d2h);
        }
        cudaEventRecord(c->ev_ru, c->d2h);  // (reused: the last piece is home)
        cudaStreamWaitEvent(c->stream, c->ev_ru, 0);
        if (int e = c->cuda_check("jv_host")) return e;
        if (int e = fetch(c, 0)) return e;
        const int e = decode_residual_errors(c, true);
        if (cell) *cell = e ? c->last.cell : -1;
        return e;
    }
    if (c->use_fused || c->jv_path != 0) cudaStreamWaitEvent(c->stream, c->ev_ru, 0);  // no in-pass wait
    c->ps.ru_ready = c->ev_ru;
    jv_async(c, c->ucand.p, c->rcand.p, c->tv.p, c->wv.p, false);
    c->ps.ru_ready = nullptr;
    cudaStreamWaitEvent(c->stream, c->ev_ru, 0);  // also when the product short-circuits
    cudaMemcpyAsync(out, c->wv.p, bytes, cudaMemcpyDeviceToHost, c->stream);
    if (int e = c->cuda_check("jv_host")) return e;
    if (int e = fetch(c, 0)) return e;
    const int e = decode_residual_errors(c, true);
    if (cell) *cell = e ? c->last.cell : -1;
    return e;
}

int sfv_precond_create(sfv_ctx* c, int kind) { return precond_create(c, kind); }

int sfv_set_step_callback(sfv_ctx* c, sfv_step_callback fn, void* user) {
    c->step_fn = fn;
    c->step_user = user;
    return SFV_OK;
}

int sfv_precond_apply_host(sfv_ctx* c, const double* r, double* z) {
    const size_t bytes = sizeof(double) * c->n;
    if (!ensure_krylov(c, 1)) return c->fail(SFV_ERR_CUDA, -1, "out of device memory");
    cudaMemcpyAsync(c->tv.p, r, bytes, cudaMemcpyHostToDevice, c->stream);
    if (int e = precond_apply_async(c, c->tv.p, c->wv.p)) return e;
    cudaMemcpyAsync(z, c->wv.p, bytes, cudaMemcpyDeviceToHost, c->stream);
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) return c->cuda_check("precond_apply");
    return SFV_OK;
}

int sfv_line_search(sfv_ctx* c, const double* u, const double* du, double r_norm0, int* success, double* s,
                    double* r_norm, double* residual) {
    if (c->singular_cell >= 0) return gradient_failure(c);
    bool ok = false;
    double ss = 1.0, rn = 0.0;
    if (int e = line_search(c, u, du, r_norm0, &ok, &ss, &rn)) return e;
    *success = ok ? 1 : 0;
    *s = ok ? ss : 0.0;
    *r_norm = ok ? rn : 0.0;
    if (ok && residual) cudaMemcpyAsync(residual, c->rcand.p, sizeof(double) * c->n, cudaMemcpyDeviceToDevice, c->stream);
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) return c->cuda_check("line_search");
    return SFV_OK;
}

int sfv_approximate_jacobian(const sfv_ctx* c, int* row_ptr, int* col, double* blocks) {
    std::vector<ScalarCsr> comps;
    const std::string msg = cell_jacobian(c->mesh, c->geom, c->ph.kbar, c->ph.transient != 0, c->ph.rho, c->ph.dt, comps);
    if (!msg.empty()) return const_cast<sfv_ctx*>(c)->fail(SFV_ERR_INVALID_ARGUMENT, -1, msg);
    const ScalarCsr& a0 = comps[0];
    if (a0.n == 3 * c->nc && c->nc > 0) {  // coupled components: the expanded matrix back to 3 x 3 blocks
        const int nnzb = a0.rp[a0.n] / 9;
        if (!col || !blocks) return nnzb;
        row_ptr[0] = 0;
        for (int i = 0; i < c->nc; ++i) {
            const int nb = (a0.rp[3 * i + 1] - a0.rp[3 * i]) / 3;
            row_ptr[i + 1] = row_ptr[i] + nb;
            for (int k = 0; k < nb; ++k) {
                col[row_ptr[i] + k] = a0.col[a0.rp[3 * i] + 3 * k] / 3;
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b)
                        blocks[9 * static_cast<size_t>(row_ptr[i] + k) + 3 * a + b] = a0.val[a0.rp[3 * i + a] + 3 * k + b];
            }
        }
        return nnzb;
    }
    const int nnz = a0.rp[a0.n];
    if (!col || !blocks) return nnz;  // size query
    for (int i = 0; i <= a0.n; ++i) row_ptr[i] = a0.rp[i];
    for (int k = 0; k < nnz; ++k) {
        col[k] = a0.col[k];
        double* b = blocks + 9 * static_cast<size_t>(k);
        for (int q = 0; q < 9; ++q) b[q] = 0.0;
        for (int a = 0; a < 3; ++a) b[4 * a] = comps[comps.size() == 1 ? 0 : a].val[k];
    }
    return nnz;
}

int sfv_precond_apply(sfv_ctx* c, const double* r, double* z) {
    if (int e = precond_apply_async(c, r, z)) return e;
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) return c->cuda_check("precond_apply");
    return c->cuda_check("precond_apply");
}

int sfv_precond_info(const sfv_ctx* c, int info[5]) {
    info[0] = c->pc_kind;
    info[1] = c->L[0].n_levels;
    info[2] = c->U[0].n_levels;
    info[3] = static_cast<int>(c->L[0].nnz);
    info[4] = static_cast<int>(c->U[0].nnz);
    return SFV_OK;
}

int sfv_precond_sweep(const sfv_ctx* c) {
    const bool ilu = c->pc_kind == SFV_PRECOND_ILU0 || c->pc_kind == SFV_PRECOND_ILU1 || c->pc_kind == SFV_PRECOND_ILU2;
    return ilu ? c->tri_cluster : -1;
}

int sfv_gmres_jv(sfv_ctx* c, const double* u, const double* r_u, const double* b, double* x, int restart,
                 double rel_reduction, int max_iters, int right_preconditioned, int* iters, int* status,
                 double* rel_residual) {
    if (c->singular_cell >= 0) return gradient_failure(c);
    // x is the initial guess; a nonzero guess costs one extra J.v as in the reference
    return gmres(c, u, r_u, b, x, false, restart, rel_reduction, max_iters, iters, status, rel_residual,
                 right_preconditioned != 0);
}

int sfv_jfnk_solve(sfv_ctx* c, double* u, const sfv_solver_cfg* cfg, sfv_solve_report* rep) {
    return jfnk(c, u, cfg, rep);
}

int sfv_segregated_solve(sfv_ctx* c, double* u, const sfv_solver_cfg* cfg, sfv_solve_report* rep) {
    return segregated(c, u, cfg, rep);
}

// run_steps (nonlinear.cpp:382-446)
int sfv_run_steps(sfv_ctx* c, double* field, const sfv_solver_cfg* cfg, int n_steps, sfv_solve_report* reports,
                  int cap, int* n_reports, double* wall_seconds) {
    const auto t0 = std::chrono::steady_clock::now();
    if (n_steps < 1) return c->fail(SFV_ERR_INVALID_ARGUMENT, -1, "run_steps: need at least one step");
    const int n = c->n;
    *n_reports = 0;
    const bool seg = cfg->algorithm == SFV_ALG_SEGREGATED;
    if (seg) {  // scalar_component_matrices instead of a preconditioner (nonlinear.cpp:397-400)
        if (int e = seg_create(c)) return e;
    } else if (int e = precond_create(c, cfg->preconditioner)) {
        return e;
    }
    if (!ensure_krylov(c, std::max(cfg->restart, 1))) return c->fail(SFV_ERR_CUDA, -1, "out of device memory");
    double* fu = field;
    double* fuo = field + n;
    double* fuoo = field + 2 * static_cast<size_t>(n);
    double* fvo = field + 3 * static_cast<size_t>(n);
    double* fvoo = field + 4 * static_cast<size_t>(n);
    double* fao = field + 5 * static_cast<size_t>(n);
    double* u = c->uscratch.p;
    const bool transient = c->ph.transient != 0;
    const double dt = c->ph.dt;
    for (int step = 1; step <= n_steps; ++step) {
        sfv_set_time(c, transient ? step * dt : static_cast<double>(step) / n_steps);
        if (transient) {
            sfv_set_history(c, fuo, fuoo, fvo, fvoo);
            launch_predict(u, fuo, fvo, fao, dt, n, c->stream);
            ++c->launches;
        } else {
            cudaMemcpyAsync(u, fu, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream);
        }
        sfv_solve_report rep{};
        if (*n_reports < cap) {  // the caller's unbounded-history buffer for this step
            rep.all_records = reports[*n_reports].all_records;
            rep.all_capacity = reports[*n_reports].all_capacity;
        }
        const int e = seg ? segregated(c, u, cfg, &rep) : jfnk(c, u, cfg, &rep);
        if (e) {
            clear_report(&rep);
            rep.status = SFV_DIVERGED;
            std::snprintf(rep.detail, SFV_DETAIL_LEN, "%s", c->last.msg.c_str());
        }
        rep.step = step;
        for (int i = 0; i < std::min(rep.n_records, 64); ++i) rep.records[i].step = step;
        if (rep.all_records)
            for (int i = 0; i < std::min(rep.n_records, rep.all_capacity); ++i) rep.all_records[i].step = step;
        if (*n_reports < cap) reports[*n_reports] = rep;
        ++*n_reports;
        if (rep.status != SFV_CONVERGED) break;
        if (int ec = sfv_commit(c, u)) return ec;  // eval.commit(u) (nonlinear.cpp:426)
        if (transient) {
            launch_bdf2_rotate(fuo, fuoo, fvo, fvoo, fao, u, dt, n, c->stream);
            ++c->launches;
        } else {
            cudaMemcpyAsync(fuo, u, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream);
        }
        cudaMemcpyAsync(fu, u, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->stream);
        if (c->step_fn) {  // on_step(step, field) (nonlinear.cpp:442)
            c->step_field.resize(6 * static_cast<size_t>(n));
            cudaMemcpyAsync(c->step_field.data(), field, sizeof(double) * 6 * n, cudaMemcpyDeviceToHost, c->stream);
            if (cudaStreamSynchronize(c->stream) != cudaSuccess) return c->cuda_check("run_steps");
            c->step_fn(c->step_user, step, c->step_field.data());
        }
    }
    if (*n_reports > cap) *n_reports = cap;
    if (transient) sfv_set_history(c, c->dzero.p, c->dzero.p, c->dzero.p, c->dzero.p);
    cudaStreamSynchronize(c->stream);
    *wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return c->cuda_check("run_steps");
}

int sfv_run_steps_host(sfv_ctx* c, double* field, const sfv_solver_cfg* cfg, int n_steps, sfv_solve_report* reports,
                       int cap, int* n_reports, double* wall_seconds) {
    const size_t bytes = sizeof(double) * 6 * c->n;
    double* d = nullptr;
    if (cudaMalloc(&d, bytes) != cudaSuccess) return c->fail(SFV_ERR_CUDA, -1, "out of device memory");
    cudaMemcpyAsync(d, field, bytes, cudaMemcpyHostToDevice, c->stream);
    const int e = sfv_run_steps(c, d, cfg, n_steps, reports, cap, n_reports, wall_seconds);
    cudaMemcpyAsync(field, d, bytes, cudaMemcpyDeviceToHost, c->stream);
    cudaStreamSynchronize(c->stream);
    cudaFree(d);
    return e;
}

}  // extern "C"
