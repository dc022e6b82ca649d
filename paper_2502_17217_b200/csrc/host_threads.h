// host_threads.h — worker count of the multi-threaded host setup passes (geometry, layout,
// J~ assembly, ILU factorisation, schedules).  Every pass partitions independent entries
// (or runs level-synchronously), so the results do not depend on the count.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>

namespace sfv {

// SFV_THREADS overrides; default: all hardware threads, at most 64
inline int host_threads() {
    static const int n = [] {
        if (const char* e = std::getenv("SFV_THREADS"); e && std::atoi(e) > 0) return std::atoi(e);
        return std::max(1, std::min(64, static_cast<int>(std::thread::hardware_concurrency())));
    }();
    return n;
}

// SFV_TIMING=1: a phase's wall time on stderr (setup profiling)
struct StageClock {
    bool on = std::getenv("SFV_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto n = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[sfv]   %-26s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};

}  // namespace sfv
