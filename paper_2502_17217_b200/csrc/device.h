// device.h — device-resident layout of the JFNK hot path (B200 / sm_100a).
//
// HBM layout:
//   * cell vectors u, v, R(u), J.v are the reference's interleaved [3c + k] doubles
//     (fields.cpp:20-25) — a cell's three components are one 24-byte record, and a
//     warp of 32 consecutive cells reads 768 contiguous bytes;
//   * per-cell face slots in ELL (slot-major) form: slot s of cell c at s*nc + c, in
//     ascending face index (Mesh::cell_faces order, mesh.cpp:55-59), so slot loads
//     are fully coalesced; each slot carries the face index (bit 31 = this cell is
//     the face's neighbour), the other cell (or -(2+patch) on a boundary face) and
//     the cell's least-squares vector for that face (mesh.cpp:493-507);
//   * per-face geometry SoA: Gamma (area vector), Delta (over-relaxed orthogonal
//     vector), |d|, w — |Gamma| and |Delta| are recomputed exactly as the reference
//     does (norm(), mesh.cpp:386 / discretisation.cpp:35);
//   * per-patch BC values (already multiplied by t when ramped) are kernel arguments.
#pragma once

#include <cmath>
#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include <vector>

namespace sfv {

constexpr int kMaxPatches = 16;
constexpr int kMaxSlots = 8;

struct PatchTable {
    int n;
    int kind[kMaxPatches];
    double value[kMaxPatches][3];
    // per boundary face values (face nint + i at 3 i), sampled from BoundaryCondition::value at
    // the face centroids and the current time (ResidualEvaluator::bc_value,
    // discretisation.cpp:82-85); null: the patch values above
    const double* face_value = nullptr;
};
// prescribed value of boundary face f (patch `patch`)
__host__ __device__ inline void bc_of(const PatchTable& pt, int patch, int f, int nint, double v[3]) {
    if (pt.face_value) {
        const double* q = pt.face_value + 3 * static_cast<size_t>(f - nint);
        v[0] = q[0];
        v[1] = q[1];
        v[2] = q[2];
    } else {
        v[0] = pt.value[patch][0];
        v[1] = pt.value[patch][1];
        v[2] = pt.value[patch][2];
    }
}

struct DevMesh {
    int nc = 0, nf = 0, nint = 0, slots = 0;
    const int* slot_face = nullptr;   // [slots*nc]; -1 = padding
    const int* slot_other = nullptr;  // [slots*nc]
    const double* slot_ls = nullptr;  // [3*slots*nc], (3*s + k)*nc + c
    const double* gam = nullptr;      // [3*nf], k*nf + f
    const double* del = nullptr;      // [3*nf]
    const double* dmag = nullptr;     // [nf]
    const double* w = nullptr;        // [nf]
    const double* volume = nullptr;   // [nc]
    // Default path (jv_pair.cu): tiled ("AoSoA") tables, 32 cells or faces per tile, so that
    // entry q of cell c sits at (c >> 5) * (nq * 32) + q * 32 + (c & 31).  A warp of 32
    // consecutive cells still loads 32 consecutive values per instruction, and a gather of
    // one cell's record needs one base address: the nq field offsets are immediates.
    int spad = 0;                  // slot stride of the tiled slot tables (4, 6 or 8)
    const int* tslot = nullptr;    // [(c>>5)][2 * spad][32]: face code (slot s), then other cell (spad + s)
    const double* tls = nullptr;   // [(c>>5)][3 * spad][32]: least-squares vector of slot s, row 3 s + k
    const double* tf9 = nullptr;   // [(f>>5)][9][32]: Gamma xyz, Delta xyz, |Delta|/|d|, |Gamma|, w
};

// hypot as the reference's C library computes it (glibc's non-FMA x86-64 path: one sqrt, then
// Borges' correction step — "An Improved Algorithm for hypot(a, b)", 2019), so the Givens
// rotations of gmres_solve (linalg.cpp:481) get the reference's bits on the host loop and in
// the device cycle alike.  Checked against the host libm on 1e6 random pairs (see
// tests/test_known_answers.py).  Power-of-two scaling keeps the squares finite.
__host__ __device__ inline double sfv_hypot(double x, double y) {
    double ax = x < 0.0 ? -x : x, ay = y < 0.0 ? -y : y;
    if (ax < ay) {
        const double t = ax;
        ax = ay;
        ay = t;
    }
    if (!(ax <= 1.79769313486231570815e308)) return ax == ax ? ax : (ay == ay ? ax : ay);  // inf / nan
    if (ay == 0.0) return ax;
    double scale = 1.0;
    if (ax > 0x1p+511) {
        ax *= 0x1p-600;
        ay *= 0x1p-600;
        scale = 0x1p+600;
    } else if (ay < 0x1p-511) {
        ax *= 0x1p+600;
        ay *= 0x1p+600;
        scale = 0x1p-600;
    }
    double h = sqrt(ax * ax + ay * ay);
    double t1, t2;
    if (h <= 2.0 * ay) {
        const double delta = h - ay;
        t1 = ax * (2.0 * delta - ax);
        t2 = (delta - 2.0 * (ax - ay)) * delta;
    } else {
        const double delta = h - ax;
        t1 = 2.0 * delta * (ax - 2.0 * ay);
        t2 = (4.0 * delta - ay) * ay + delta * delta;
    }
    h -= (t1 + t2) / (2.0 * h);
    return h * scale;
}

constexpr int kTileShift = 5;  // 32 cells (faces) per tile of the tiled tables
__host__ __device__ __forceinline__ size_t tiled(int c, int nq) {
    return static_cast<size_t>(c >> kTileShift) * (static_cast<size_t>(nq) << kTileShift) + (c & 31);
}
constexpr int kWG = 12;   // rows of the tiled [w | G] record: w xyz, then G row-major
constexpr int kSig = 9;   // rows of the tiled cell-stress record (row-major, nothing mirrored)

struct Physics {
    int law;  // SFV_LAW_*
    int tl;
    int transient;
    double mu, lam, alpha, kbar;
    double rho, dt;
    int stab_only;  // ResidualEvaluator::stabilisation (discretisation.cpp:210-214)
    double gc[8];   // Guccione: C, c_f, c_t, c_fs, kappa, f0 xyz (GuccioneParams, laws.hpp:38-43)
    // J2 plasticity (J2PlasticLaw, laws.hpp:139-155): mu, kappa = mu, lam; HardeningCurve
    // (laws.hpp:52-64): saturation a, b, c, d, or a table of jn (eps_p, sigma_y) pairs
    double ja, jb, jc, jd;
    int jn;
    double jt[2 * 16];
    int commit;  // gradient pass of ResidualEvaluator::commit: write the trial state as committed
};
constexpr int kMaxHardening = 16;
constexpr int kJ2 = 19;  // rows of the tiled J2 state record: b_bar (9), eps_p, F (9)  (PlasticCell)

// Error words written by kernels (atomicMin of the first offending index; INT_MAX = none).
struct ErrWords {
    int inverted_cell;  // law stress: det F <= 0 (laws.cpp:14)
    int inverted_face;  // transform_area: det F_f <= 0 (discretisation.cpp:102)
    int nan_cell;       // residual: non-finite entry (discretisation.cpp:171-172)
    int nan_jv;         // J.v: non-finite difference quotient (nonlinear.cpp:135)
    int overflow_cell;  // law stress: Guccione exponent overflow (laws.cpp:69-70)
    int retmap_cell;    // law stress: J2 hardening Newton did not converge (laws.cpp:145-146)
};

// History for the BDF2 inertia term (interleaved [3c+k]).
struct History {
    const double* u_old = nullptr;
    const double* u_old_old = nullptr;
    const double* v_old = nullptr;
    const double* v_old_old = nullptr;
    // volume_c * body_force(centroid_c), interleaved (discretisation.cpp:160-161); null: none
    const double* body = nullptr;
};

// ---- residual.cu
// R(u) (jv_eps == nullptr) or the fused J.v epilogue (R(u + eps v) - r_u) / eps with
// eps read from *jv_eps (a zero eps means v == 0: out is zero, nonlinear.cpp:110).
void launch_residual(const DevMesh& m, const Physics& ph, const PatchTable& pt, const History& hist,
                     const double* u, const double* v, const double* jv_eps, const double* r_u,
                     double* out, double* grad_scratch, ErrWords* err, cudaStream_t s);
// ---- jv_pair.cu: same contract as launch_residual; perturb + gradient + boundary-face +
// per-(cell, face slot) flux kernels
struct PairScratch {
    double* wg = nullptr;           // tiled [w | G] (kWG rows): perturbed state u + eps v, cell gradients
    double* sig = nullptr;          // tiled cell stress (9 entries, row-major), non-Hooke / TL only
    double* lawst = nullptr;        // tiled committed J2 state (kJ2 rows), J2 only
    const int* bnd_cs = nullptr;    // [nf-nint] cell * 8 + slot of boundary face nint+fb
    double* bres = nullptr;       // [6*(nf-nint)] boundary-face flux + stabilisation
    cudaEvent_t* marks = nullptr;  // optional: recorded after the perturb, gradient, boundary passes
    // J.v: eps computed in the perturb pass from launch_norm_partials' block partials
    // (nullptr: eps given in *jv_eps)
    // boundary pass on a side stream, beside the gradient pass (null: in line)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_w = nullptr, ev_b = nullptr;
    // optional: r_u arrives on another stream (host-buffer J.v); the face pass waits for it
    cudaEvent_t ru_ready = nullptr;
    // optional (host-buffer J.v): the face pass runs in nchunk launches over consecutive tile
    // ranges; launch k waits for ru_chunk[k] (its share of r_u) and records out_chunk[k]
    int nchunk = 0;
    const cudaEvent_t* ru_chunk = nullptr;
    cudaEvent_t* out_chunk = nullptr;
    const double* partials = nullptr;  // block partials (or, with bar, the fused pass's scratch)
    int npart = 0;
    // set: eps_perturb_kernel reduces the norms itself (grid barrier on this counter) and
    // partials is only its scratch (>= 2 * eps_perturb grid doubles)
    unsigned long long* bar = nullptr;
    bool sym = false;  // the mesh has a symmetry patch (boundary faces then need boundary_kernel)
    double* u_norm = nullptr;
    bool u_norm_cached = false;
    // v = v + (*vsel_j) * vsel_stride, read on the device (the fused ε pass only): the GMRES
    // cycle graph passes the basis V and its step index
    const int* vsel_j = nullptr;
    size_t vsel_stride = 0;
    bool* vsel_failed = nullptr;  // set when the fused ε pass could not run (the other passes do not select)
    // L2 persisting window over [w | G]: both are gathered by the next pass,
    // and G is rewritten in place by the next J.v, so resident lines never reach HBM
    void* win_base = nullptr;
    size_t win_bytes = 0;
    float win_hit = 0.f;
};
void launch_residual_pair(const DevMesh& m, const Physics& ph, const PatchTable& pt, const History& hist,
                          const double* u, const double* v, const double* jv_eps, const double* r_u, double* out,
                          const PairScratch& ps, ErrWords* err, cudaStream_t s);
// cell_gradients only (discretisation.cpp:10-31), SoA [k*nc + c], k = 3i + j, through the
// default path's kernels (scratch in ps)
void launch_gradients_pair(const DevMesh& m, const PatchTable& pt, const Physics& ph, const double* u, double* G,
                           const PairScratch& ps, ErrWords* err, cudaStream_t s);
// grid of the fused ε + perturb pass for nc cells, 0 when it cannot run (not co-resident)
int eps_perturb_grid_for(int nc);
// the same through residual.cu (alternative paths)
void launch_gradients(const DevMesh& m, const PatchTable& pt, const double* u, double* G, cudaStream_t s);
// Block partials of |u|^2 and |v|^2 (2 per block, fixed order) for the jv_pair.cu path;
// returns the number of blocks.
int launch_norm_partials(const double* u, const double* v, int n, double* partial, bool u_norm_cached, cudaStream_t s);
// eps = sqrt(DBL_EPSILON) sqrt(1 + |u|) / |v| into *eps (nonlinear.cpp:109-115), with
// |u| taken from *u_norm when u_norm_cached is set.
void launch_jv_eps(const double* u, const double* v, int n, double* scratch, unsigned* counter,
                   double* eps_out, double* u_norm_inout, bool u_norm_cached, cudaStream_t s);

// ---- jv_fused.cu: one persistent kernel per residual / J.v (see the file header)
constexpr int kTile = 256;
struct FusedLayout {
    int ntiles = 0, lag = 0, ring_tiles = 0, ring_cells = 0, nfl = 0;
    const int* tile_face_ptr = nullptr;  // [ntiles+1] faces computed by each tile (lower cell in tile)
    const int* f_owner = nullptr;        // [nfl] reference owner
    const int* f_other = nullptr;        // [nfl] neighbour, or -(2+patch) on a boundary face
    const int* f_slots = nullptr;        // [nfl] slot in owner list | slot in neighbour list << 8
    const int* f_index = nullptr;        // [nfl] reference face index
    const double* f_geo = nullptr;       // [8*nfl] Gamma xyz, Delta xyz, |d|, w in processing order
    double* gring = nullptr;             // [9*ring_cells]
    double* fring = nullptr;             // [6*slots*ring_cells]
};
struct FusedArgs {
    DevMesh m;
    FusedLayout L;
    Physics ph;
    PatchTable pt;
    History hist;
    const double* u;
    const double* v;
    const double* eps;  // nullptr: plain residual
    const double* r_u;
    double* out;
    ErrWords* err;
    int* ticket;
    int* a_done;
    int* b1_done;
    int* b2_done;
    int epoch;
};
int fused_resident_ctas(bool general);  // resident CTAs of the persistent grid
void launch_fused(const FusedArgs& a, int grid, cudaStream_t s);

// ---- segregated.cu: the segregated solver's device kernels (nonlinear.cpp:268-351)
struct SegCsr {  // one component of A = -J~ (ScalarCsrMatrix)
    int n = 0;
    const int* rp = nullptr;
    const int* col = nullptr;
    const double* val = nullptr;
};
struct SegSweep {  // one IC(0) sweep in dependency-level order (TriSchedule on the device)
    int n_pos = 0;
    const int* order = nullptr;
    const int* rp = nullptr;
    const int* col = nullptr;  // row indices
    const double* val = nullptr;
    const double* diag = nullptr;
};
// z = (L L^T)^{-1} r with y as the forward-sweep scratch (vectors of n)
void seg_ic0_apply(const SegSweep& f, const SegSweep& b, const double* r, double* y, double* z, int n, int grid,
                   cudaStream_t s);
void seg_spmv(const SegCsr& a, const double* x, double* y, cudaStream_t s);
void seg_component(int n, const double* u, int c, double* out, cudaStream_t s);      // out = u[:, c]
void seg_set_component(int n, const double* x, int c, double* u, cudaStream_t s);    // u[:, c] = x
void seg_add_component(int n, const double* r, int c, double* b, cudaStream_t s);    // b += r[:, c]
void seg_rsub(int n, const double* b, double* r, cudaStream_t s);                    // r = b - r
void seg_xpby(int n, const double* z, double beta, double* p, cudaStream_t s);       // p = z + beta p
void seg_jacobi(int n, const double* inv, const double* r, double* z, cudaStream_t s);
void seg_relax(int n3, const double* un, double relax, double* u, double* du, cudaStream_t s);
int seg_sweep_grid();

// ---- krylov.cu (deterministic fixed-order reductions)
int reduce_blocks(int n);
void launch_dot(const double* a, const double* b, int n, double* out, double* scratch, unsigned* counter,
                cudaStream_t s);
// w -= (*h) * vi ; then *out = dot(w, vnext) (vnext == nullptr: *out = dot(w, w))
void launch_axpy_dot(double* w, const double* vi, const double* h, const double* vnext, int n, double* out,
                     double* scratch, unsigned* counter, cudaStream_t s);
// Reference-order sums (opt-in "sequential_reductions"): the left-to-right chain of
// std::inner_product, one CTA, ~13 ms per 3M terms.  seq_axpy_dot: w -= (*h) vi, then the
// chain of w.vnext (or w.w).  seq_eps: sums[0] = v.v, sums[1] = u.u (unless cached), then
// eps_out = the reference's ε and u_norm = |u|.
void launch_seq_dot(const double* a, const double* b, int n, double* out, cudaStream_t s);
void launch_seq_axpy_dot(double* w, const double* vi, const double* h, const double* vnext, int n, double* out,
                         cudaStream_t s);
void launch_seq_eps(const double* u, const double* v, int n, double* sums, double* eps_out, double* u_norm,
                    bool cached, cudaStream_t s);
// Fused Arnoldi step (cooperative, w held in shared memory): h[0..j] = MGS projections of
// w on V[0..j], h[j+1] = w.w after them, vnext (if not null) = w / sqrt(h[j+1]).  partial:
// 2 * SMs doubles.  Returns false (nothing launched) when w does not fit on chip.
bool launch_arnoldi_fused(const double* w, const double* V, int n, int j, double* h, double* partial, double* vnext,
                          cudaStream_t s);
// The same with the step index read on the device (*jdev) and v_{j+1} written to V[j + 1]
// when j + 1 < vcap (device-resident GMRES cycle).
int arnoldi_fused_grid(int n, int* chunk_out);  // 0: w does not fit on chip
bool launch_arnoldi_fused_dev(const double* w, const double* V, int n, const int* jdev, int vcap, double* h,
                              double* partial, cudaStream_t s);
// device-resident GMRES(m) cycle state: header + rotations, residual estimates, Hessenberg
// columns (column j at H + j * (m + 1))
struct GmresHdr {
    int j, total, restart, max_iters, happy, pad;
    double target;
};
struct GmresDev {
    GmresHdr* hdr = nullptr;
    double* cs = nullptr;
    double* sn = nullptr;
    double* g = nullptr;
    double* H = nullptr;
};
// one thread: the host half of an Arnoldi step (rotations, tests), then the cycle's WHILE condition
void launch_givens(const GmresDev& st, const double* h, const ErrWords* err, cudaGraphConditionalHandle cond,
                   cudaStream_t s);
void launch_scale_div(const double* in, const double* divisor, double* out, int n, cudaStream_t s);
void launch_scale_div_host(const double* in, double divisor, double* out, int n, cudaStream_t s);
void launch_update(double* x, const double* V, const double* y, int j, int n, cudaStream_t s);
void launch_basis_combination(double* dx, const double* V, const double* y, int j, int n, cudaStream_t s);
void launch_sub_from(const double* b, double* r, int n, cudaStream_t s);  // r = b - r
void launch_negate(const double* a, double* out, int n, cudaStream_t s);
void launch_axpy_host(double* y, double alpha, const double* x, int n, cudaStream_t s);  // y += alpha x
void launch_lincomb(double* out, const double* u, double s, const double* du, int n,
                    cudaStream_t st);  // out = u + s*du
void launch_bdf2_rotate(double* uo, double* uoo, double* vo, double* voo, double* ao, const double* u, double dt,
                        int n, cudaStream_t s);
void launch_predict(double* u, const double* uo, const double* vo, const double* ao, double dt, int n,
                    cudaStream_t s);

// ---- precond.cu
struct DevTri {  // one triangular factor in level (processing) order
    int n = 0;       // positions (rows + per-level padding)
    int n_rows = 0;  // matrix rows
    int n_levels = 0;
    const int* order = nullptr;   // [n] row processed at position p
    const int* level_ptr = nullptr;  // [n_levels+1] first position of each level
    const int* rp = nullptr;      // [n+1] entries of the row at position p
    const int* col = nullptr;     // [nnz]
    const double* val = nullptr;  // [nnz]
    const double* diag = nullptr; // [n] (upper only; per position)
    int maxd = 0;                     // widest row
    const int* ell_col = nullptr;     // [maxd*n] k-th entry of the row at position p, -1 = none
    const int* ell_pcol = nullptr;    // [maxd*n] the same entries as positions (position-space sweeps)
    const int* u2l = nullptr;         // [n] (upper only) lower-sweep position of the row at position p
    const double* ell_val = nullptr;  // [maxd*n]
};
// ILU apply on the cell graph, 3 interleaved right-hand sides (finding 4):
// forward unit-lower then backward upper, row arithmetic in the reference's order.
struct TriSet {
    DevTri t[3];
};
// y is the forward-sweep scratch vector (3n); z receives M^{-1} r.  ncomp = 1: one
// factor for all three components; ncomp = 3: factor t[k] for component k; ncomp = -1: t[0]
// is one factor over all 3n unknowns (coupled components: a symmetry plane that is not
// axis-aligned), applied by the sync-free sweep (cluster == 0).
// cluster > 0: level-synchronous sweep by one cluster of that many CTAs per component;
// cluster == 0: sync-free sentinel polling on a persistent grid of `grid` CTAs.
// pa, pb: position-space scratch vectors of 3 * max positions (cluster > 0 path).
// cluster == kDsRingMode selects the DSMEM-ring sweep (needs ring_window() >= largest
// dependency distance + 2 x widest level, checked at setup).
constexpr int kDsRingMode = 100;
int ilu_ring_window();

// ---- precond_stream.cu: streamed sweep (default; records built by build_stream_records)
constexpr int kStreamMode = 200;
#ifndef SFV_STREAM_CLUSTER
#define SFV_STREAM_CLUSTER 16
#endif
#ifndef SFV_STREAM_MAX_ROWS
#define SFV_STREAM_MAX_ROWS 256
#endif
constexpr int kStreamCluster = SFV_STREAM_CLUSTER;
constexpr int kStreamRing = 3072;    // 32-byte value slots per CTA
constexpr int kStreamMaxRows = SFV_STREAM_MAX_ROWS;  // positions per CTA per level
struct DevStream {
    int n_levels = 0;
    const int* level_ptr = nullptr;  // position-space level boundaries (same as DevTri)
    const void* rec = nullptr;       // [n_pos] 112-byte records
};
struct StreamSet {
    DevStream t[3];
    int ring = 0;      // value slots per CTA
    int max_rows = 0;  // positions per CTA per level (multiple of 32)
    int stages = 3;    // cp.async pipeline depth (levels in flight + 1)
};
// Streamed-sweep records, per chunk of 32 positions (field-major, bank-conflict-free reads):
// val[8][32] doubles, diag[32], dep[8][32] u32, own[32] u16, out[32] i32, zero tail.  A dep word
// is the dependency's shared::cluster window offset from the ring base: owner rank << 24 |
// slot * 8 (the layout mapa.shared::cluster produces on sm_100, scripts/probes/mapa_probe.cu),
// so the sweep forms each load address with one add; an absent dependency is the reading
// CTA's +0.0 slot (slot = ring size).
constexpr int kStreamChunk = 3584, kStreamRec = 112;
constexpr int kStreamOffDiag = 2048, kStreamOffDep = 2304, kStreamOffOwn = 3328, kStreamOffOut = 3392,
              kStreamOffEnd = 3520;
__host__ __device__ inline uint32_t stream_dep(int rank, int slot) {
    return (static_cast<uint32_t>(rank) << 24) | (static_cast<uint32_t>(slot) * 8u);
}
// value ring(s) incl. the +0.0 slot (3 right-hand sides of ring + 1 doubles), 128-byte rounded
__host__ __device__ inline int stream_ring_bytes(int ring) { return ((ring + 1) * 24 + 127) & ~127; }
int stream_smem_bytes(int ring, int max_rows, int stages);
cudaError_t launch_tri_stream(const StreamSet& set, bool upper, int ncomp, const double* src, double* dst,
                              cudaStream_t s);
// ---- precond_pipe.cu: block-pipelined sweep (default when build_pipe accepts the factor)
constexpr int kPipeMode = 300;
constexpr int kPipeCluster = 16;
constexpr int kPipeThreads = 512;  // consumer threads per CTA (+ producer and publisher warps)
constexpr int kPipeChunk = 3328;   // bytes per 32 records (precond_host.h: kPipeChunkBytes)
struct DevPipe {
    const int* step_off = nullptr;  // [blocks + 1]
    const int* step_ptr = nullptr;  // [total steps + blocks]
    const int* need = nullptr;      // [total steps]
    const int* guard = nullptr;     // [total steps]
    const unsigned char* rec = nullptr;
    const int* order = nullptr;     // position -> row (-1 padding)
    const int* to_lower = nullptr;  // upper sweep only: position -> lower-sweep position
    int n_pos = 0;
};
struct PipeSet {
    DevPipe t[3];  // per component (the same factor three times when shared)
    int ring = 0;
};
int pipe_smem_bytes(int ring);
cudaError_t launch_tri_pipe(const PipeSet& set, bool upper, const double* src, double* dst, cudaStream_t s);

void launch_ilu_apply(const TriSet& L, const TriSet& U, int ncomp, const double* r, double* y, double* z, int grid,
                      int sleep_ns, int cluster, double* pa, double* pb, const struct StreamSet* SL,
                      const struct StreamSet* SU, cudaStream_t s, const PipeSet* PL = nullptr,
                      const PipeSet* PU = nullptr);
// Exact dense apply z = A^{-1} r for the small-system LU path (3 interleaved RHS).
void launch_dense_apply(const double* inv, int n, const double* r, double* z, cudaStream_t s);
// Small-system exact preconditioner: W = (L L^T)^{-1} from a band Cholesky of -K, and
// z = K^{-1} r = -P W P^T r applied to 3 interleaved components.
// The band of -A (permuted, BandChol layout) factored by cuSOLVER dense Cholesky (potrf): with
// W null the band becomes that of the factor (in place); with W the explicit inverse (potri)
// is written to W (row-major n x n).  "" or the reference-style error text.
std::string device_band_cholesky(double* band, int n, int bw, cudaStream_t s, double* W = nullptr);
// ILU(<=1) numeric phase on the device (precond.cu; the IluNumericFn of precond_host.h)
struct ScalarCsr;
bool device_ilu_numeric(ScalarCsr& out, const std::vector<int>& diag, const std::vector<int>& rows,
                        cudaStream_t stream);
void launch_band_inverse(const double* l, int n, int bw, double* W, cudaStream_t s);
// comp < 0: all three components with one W; comp = k: component k only;
// comp = kDenseCoupled: W spans all 3n unknowns (n = 3 x cells, coupled components)
constexpr int kDenseCoupled = -2;
void launch_dense_apply_perm(const double* W, int n, const int* perm, const double* r, double* z, int comp,
                             cudaStream_t s);

}  // namespace sfv
