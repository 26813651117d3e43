// Tracing mode of the library (pmg_set_tracing; the
// reference has only wall time around the iteration loop and communication
// counters).  Host-side only:
//  * NVTX ranges -- solve, cycle, level and halo exchange -- pushed while
//    tracing is on (NVTX 3 is header-only: without a tool attached a push is
//    a function-pointer check).  Inside a captured cycle graph the level
//    ranges mark the capture, the cycle ranges every replay.
//  * CycleClock: a CUDA event pair around every cycle's graph replay on the
//    solve stream, read after the per-cycle host sync the drivers already do,
//    so the device time of each cycle costs no extra synchronisation.
#pragma once

#include <atomic>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

namespace pmg {

extern std::atomic<int> g_trace;

inline bool tracing() { return g_trace.load(std::memory_order_relaxed) != 0; }

struct Trace {
    bool on;
    explicit Trace(const char *name) : on(tracing()) {
        if (on) nvtxRangePushA(name);
    }
    Trace(const char *fmt, int a) : on(tracing()) {
        if (on) {
            char buf[64];
            std::snprintf(buf, sizeof buf, fmt, a);
            nvtxRangePushA(buf);
        }
    }
    ~Trace() {
        if (on) nvtxRangePop();
    }
    Trace(const Trace &) = delete;
    Trace &operator=(const Trace &) = delete;
};

// device time of each cycle of the last traced solve
struct CycleClock {
    cudaEvent_t a = nullptr, b = nullptr;
    std::vector<double> ms;
    bool armed = false;

    void reset() {
        ms.clear();
        armed = false;
    }
    cudaError_t start(cudaStream_t st) {
        armed = false;
        if (!tracing()) return cudaSuccess;
        cudaError_t e = cudaSuccess;
        if (!a) e = cudaEventCreate(&a);
        if (e == cudaSuccess && !b) e = cudaEventCreate(&b);
        if (e == cudaSuccess) e = cudaEventRecord(a, st);
        armed = e == cudaSuccess;
        return e;
    }
    cudaError_t stop(cudaStream_t st) {
        if (!armed) return cudaSuccess;
        cudaError_t e = cudaEventRecord(b, st);
        if (e == cudaSuccess) e = cudaEventSynchronize(b);
        float t = 0.f;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&t, a, b);
        if (e == cudaSuccess) ms.push_back(t);
        armed = false;
        return e;
    }
    int copy_out(double *out, int cap) const {
        const int n = (int)ms.size();
        for (int i = 0; i < n && i < cap; ++i) out[i] = ms[i];
        return n;
    }
    ~CycleClock() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
};

}  // namespace pmg
