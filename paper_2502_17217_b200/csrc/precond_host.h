// precond_host.h — host setup of the reference's preconditioners on the cell graph.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "host_mesh.h"

namespace sfv {

// Allocator that leaves resized elements uninitialised: the large setup arrays below are
// written completely by parallel passes, which then also do the first touch of the pages.
template <class T>
struct NoInit : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = NoInit<U>;
    };
    NoInit() = default;
    template <class U>
    NoInit(const NoInit<U>&) noexcept {}
    template <class U>
    void construct(U* p) noexcept {
        ::new (static_cast<void*>(p)) U;
    }
    template <class U, class... A>
    void construct(U* p, A&&... a) {
        ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    }
};
template <class T>
using rawvec = std::vector<T, NoInit<T>>;

struct ScalarCsr {
    int n = 0;
    std::vector<int> rp;
    rawvec<int> col;  // columns ascending per row
    rawvec<double> val;
};

// Per-component scalar matrices of assemble_approximate_jacobian
// (/root/reference/proj/src/discretisation.cpp:216-262), accumulated entry by entry in
// the reference's face order.  ncomp = 1 when every block is c*I (no symmetry faces),
// 3 when blocks are diagonal (axis-aligned symmetry faces).  A symmetry face whose normal is not
// axis-aligned couples the components (-coeff n (x) n on the diagonal block): then comps holds ONE
// matrix with n = 3 * cells, the reference's expand_scalar() (linalg.cpp:135-158) — rows 3 i + a,
// all nine entries of every block in the pattern.  Returns "" or an error.
std::string cell_jacobian(const HostMesh& m, const HostGeometry& g, double kbar, bool transient, double rho,
                          double dt, std::vector<ScalarCsr>& comps);

// IlukPrecond ctor (linalg.cpp:251-300) on a scalar matrix: returns "" or the
// IluBreakdown message.  The factor is the combined LU in one CSR pattern.
// Numeric phase of the ILU(<=1) factorisation on another engine (the device): out holds the
// final pattern with A at its positions (fill entries 0), diag the diagonal positions and
// rows the rows in dependency-level order; factors out.val in place with the reference's
// per-entry operations, false on a breakdown (the caller reruns the sequential code).
using IluNumericFn = std::function<bool(ScalarCsr& out, const std::vector<int>& diag, const std::vector<int>& rows)>;
std::string iluk_factor(const ScalarCsr& a, int level, ScalarCsr& lu, const IluNumericFn& numeric = nullptr);



// One triangular sweep in dependency-level order, levels padded to whole warps.
struct TriSchedule {
    int n_pos = 0, n_levels = 0;
    std::vector<int> order, rp, level_ptr;
    rawvec<int> col;
    rawvec<double> val;
    std::vector<double> diag;
    int maxd = 0;
    rawvec<int> ell_col;   // [maxd * n_pos], entry k of position p at k * n_pos + p
    rawvec<int> ell_pcol;  // the same columns as positions of this schedule
    rawvec<double> ell_val;
    std::vector<int> pos;  // row -> position
};
void schedule_lower(const ScalarCsr& lu, TriSchedule& t);
void schedule_upper(const ScalarCsr& lu, TriSchedule& t);

// Ic0Precond (linalg.cpp:174-221): L on the lower pattern of A with the reference's
// row-oriented arithmetic; false on a breakdown (missing diagonal / non-positive pivot).
bool ic0_factor(const ScalarCsr& a, ScalarCsr& L);
// Its two sweeps (Ic0Precond::solve, linalg.cpp:208-218) as schedules: forward, rows of L in
// ascending column order then / L_ii; backward, the saxpy loop restated per row of L^T —
// z_i loses L_ji z_j for j descending, then / L_ii — both in dependency-level order.
void schedule_ic0(const ScalarCsr& L, TriSchedule& fwd, TriSchedule& bwd);

// Streamed-sweep records (precond.cu, tri_stream_kernel): one 112-byte record per position,
// position order.  Level l's positions are split into `cs` contiguous chunk-aligned slices
// (CTA r of the cluster owns slice r); each CTA stores its positions' values in a ring of
// `ring` slots in its shared memory, and every dependency is recorded as its DSMEM address
// (owner << 12 | slot).  Returns false when a ring slot would be overwritten before its
// last reader (then the caller keeps another sweep), or a slice exceeds max_rows.
struct StreamRecord {  // (the logical record; stored field-major per chunk, device.h kStream*)
    uint32_t dep[8];  // owner << 24 | slot * 8; absent: the reader's +0.0 slot (slot = ring size)
    uint16_t own;     // this position's slot in its owner's ring
    uint16_t pad;
    int32_t out;      // where the sweep stores the value (-1: level padding)
    double val[8];
    double diag;
};
static_assert(sizeof(StreamRecord) == 112, "record layout");
// Built directly in the device chunk layout below (every byte written by the parallel pass).
bool build_stream_records(const TriSchedule& t, int cs, int ring, int max_rows, rawvec<unsigned char>& packed,
                          const std::vector<int>* out_pos = nullptr);
// Device layout of the records: per chunk of 32 positions (levels are padded to 32), the
// fields as arrays over the 32 positions — val[8][32], diag[32], dep[8][32] (u32), own[32],
// out[32], 3584 bytes (device.h kStream*) — so that a warp reading one field of 32 consecutive rows from shared
// memory is bank-conflict free (the 96-byte AoS record was read at a 96-byte lane stride).
// out[32] (int32): where the sweep stores the position's value: the forward
// sweep writes in the backward sweep's position order, the backward sweep writes rows, so no
// permute or scatter pass runs between or after them (-1: level padding, nothing stored).
constexpr int kChunkBytes = 3584;  // = kStreamChunk (device.h)


// Block-pipelined sweep (precond_pipe.cu): the rows, in sweep order, are cut into `blocks`
// contiguous blocks, one CTA each; CTA b walks only the dependency levels present in its
// block ("steps"), in order.  Every dependency of a block-b row lies in block b or b-1
// (checked; false otherwise).  Positions are block-major, step-major, each (block, step)
// padded to 32.  Values live in a ring of `ring` doubles in each CTA's shared memory; a
// dependency is its ring slot, bit 31 set when it is in block b-1's ring (read over DSMEM).
//   need[b][s]:  steps block b-1 must have completed before block b runs step s (data);
//   guard[b][s]: steps block b+1 must have completed before block b runs step s (its ring
//                slots about to be rewritten have been read by all their remote readers).
// Both are non-decreasing in s.  Records are chunk-SoA per 32 positions: val[8][32],
// diag[32], dep[8][32] (u32); 3328 bytes.
constexpr int kPipeChunkBytes = 3328;
struct PipeSchedule {
    int blocks = 0, ring = 0, n_pos = 0, max_rows = 0;
    std::vector<int> order;       // position -> row (-1 padding)
    std::vector<int> pos;         // row -> position
    std::vector<int> step_off;    // [blocks + 1] first step of block b in the flat step tables
    std::vector<int> step_ptr;    // [total steps + blocks] positions: step s of block b spans
                                  // [step_ptr[step_off[b] + b + s], step_ptr[step_off[b] + b + s + 1])
    std::vector<int> need, guard;  // [total steps]
    std::vector<unsigned char> rec;  // n_pos / 32 chunks of kPipeChunkBytes
};
bool build_pipe(const ScalarCsr& lu, bool upper, int blocks, int ring, PipeSchedule& out, std::string* why);

// Banded Cholesky of -A after reverse Cuthill-McKee (A symmetric negative definite);
// returns "" or "lu: factorisation failed".  Band row i holds L(i, i-bw .. i).
struct BandChol {
    int n = 0, bw = 0;
    std::vector<int> perm;  // band index -> original row
    std::vector<double> l;  // n * (bw + 1), l[i*(bw+1) + (j - i + bw)]
};
// factor = false: only the ordering (perm, bw) and the band of -A in l (not factored)
std::string band_cholesky_neg(const ScalarCsr& a, BandChol& out, bool factor = true);

}  // namespace sfv
