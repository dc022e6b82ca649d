// Host-only timing of the context and preconditioner setup phases on a BASELINE box mesh
// (no GPU needed); build: g++ -O2 -ffp-contract=off -std=c++17 -pthread -I include
//   -I paper_2502_17217_b200/csrc scripts/probes/setup_bench.cpp paper_2502_17217_b200/csrc/host_mesh.cpp paper_2502_17217_b200/csrc/precond_host.cpp
#include <chrono>
#include <cstdio>
#include <vector>

#include "host_mesh.h"
#include "precond_host.h"
#include "sfv_case.h"

using namespace sfv;

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 100;
    auto t = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        const auto now = std::chrono::steady_clock::now();
        std::printf("%-22s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    };
    const double ext[3] = {1, 1, 1};
    const int div[3] = {n, n, n};
    const int kinds[6] = {SFV_PATCH_DISPLACEMENT, SFV_PATCH_TRACTION, SFV_PATCH_TRACTION,
                          SFV_PATCH_TRACTION, SFV_PATCH_TRACTION, SFV_PATCH_TRACTION};
    HostMesh m = box_hex(ext, div, kinds);
    distort(m, 0.15, 42);
    m.finalise();
    mark("mesh");
    HostGeometry g;
    compute_geometry(m, g);
    mark("compute_geometry");
    std::vector<ScalarCsr> comps;
    cell_jacobian(m, g, 2.0e11, false, 0.0, 1.0, comps);
    mark("cell_jacobian");
    ScalarCsr lu;
    iluk_factor(comps[0], 1, lu);
    mark("iluk_factor");
    TriSchedule tl, tu;
    schedule_lower(lu, tl);
    mark("schedule_lower");
    schedule_upper(lu, tu);
    mark("schedule_upper");
    int max_rows = 32;
    for (int l = 0; l < tl.n_levels; ++l)
        max_rows = std::max(max_rows, ((tl.level_ptr[l + 1] - tl.level_ptr[l]) / 32 + 15) / 16 * 32);
    rawvec<unsigned char> packed;
    const bool ok = build_stream_records(tl, 16, 3072, max_rows, packed);
    mark(ok ? "stream records (L)" : "stream records FAILED");
    return 0;
}
