// precond_dev.h — ILU(k <= 1) preconditioner setup on the device (precond_dev.cu).
#pragma once

#include <chrono>
#include <string>

#include <cuda_runtime.h>

namespace sfv {

// the device-resident topology and geometry fields the J~ assembly reads (geometry.cu)
struct DevTopoView {
    int nc = 0, nf = 0, nint = 0;
    const int* owner = nullptr;
    const int* neigh = nullptr;
    const int* cf_off = nullptr;     // [nc + 1]
    const int* cf = nullptr;         // faces of each cell, ascending
    const int* face_kind = nullptr;  // SFV_PATCH_* of a boundary face, -1 internal
    const double* amag = nullptr;    // |Gamma|
    const double* dmag = nullptr;    // |d|
    const double* delmag = nullptr;  // |Delta|
    const double* vol = nullptr;
};

// one triangular sweep of the streamed apply: position map, level pointers, records (and for
// the backward sweep the backward -> forward position map); device memory owned by the caller
struct DevSweep {
    int n_pos = 0, n_levels = 0;
    int* order = nullptr;          // [n_pos] position -> row (-1 padding)
    int* level_ptr = nullptr;      // [n_levels + 1]
    unsigned char* rec = nullptr;  // [n_pos / 32] chunks of 3072 bytes (precond_host.h layout)
    int* u2l = nullptr;            // backward sweep only
    void release();
};
struct DevIluSetup {
    DevSweep L, U;
    int ring = 0, max_rows = 0;
    long long nnz_L = 0, nnz_U = 0;  // strictly lower / upper entries of the factor
    void release() {
        L.release();
        U.release();
    }
};

// J~ (c I blocks), its ILU(level) factor and both sweeps' schedules and records, on stream s.
// "" on success (out owns the buffers), else why the host setup must run instead.  timing
// (optional, 5 doubles): ms of J~, pattern, schedules, numeric phase, records.
std::string device_ilu_setup(const DevTopoView& t, double kbar, bool transient, double rho, double dt, int level,
                             cudaStream_t s, DevIluSetup& out, double* timing = nullptr);

// the IKJ numeric phase over device CSR arrays, rows in dependency-level order (precond.cu);
// false on a zero / non-finite pivot or a refused cooperative launch
bool launch_ilu_numeric(int n, const int* rows, const int* rp, const int* col, const int* diag, double* val,
                        cudaStream_t s);

}  // namespace sfv
