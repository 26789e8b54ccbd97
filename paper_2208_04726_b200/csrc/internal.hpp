// internal.hpp — host-side internals shared by capi.cu and graph.cpp.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/pvo_capi.h"

namespace pvo_host {

// Error carrying a pvo_status across the C++ host code; converted to a
// status + thread-local message at the extern "C" boundary.
struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};
[[noreturn]] inline void fail(int status, const std::string& msg) { throw Error(status, msg); }
void set_last_error(const std::string& msg);

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return PVO_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.status;
    } catch (const std::bad_alloc&) {
        set_last_error("out of host memory");
        return PVO_CUDA_ERROR;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return PVO_INVALID_ARGUMENT;
    }
}

// NVTX range in the "pvo" domain (nvtx3 is header-only; without a profiler
// attached a push/pop is a null-pointer check).  Every C-ABI entry point
// opens one named after itself; the launch helpers nest "corr" / "ba" /
// "measure" / ... inside it, so an nsys / ncu --nvtx timeline shows the
// reference-facing call and the kernels it issued.
inline nvtxDomainHandle_t nvtx_domain() {
    static const nvtxDomainHandle_t d = nvtxDomainCreateA("pvo");
    return d;
}
struct NvtxRange {
    explicit NvtxRange(const char* name) {
        nvtxEventAttributes_t ev{};
        ev.version = NVTX_VERSION;
        ev.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
        ev.messageType = NVTX_MESSAGE_TYPE_ASCII;
        ev.message.ascii = name;
        nvtxDomainRangePushEx(nvtx_domain(), &ev);
    }
    ~NvtxRange() { nvtxDomainRangePop(nvtx_domain()); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

template <typename F>
int guarded(const char* entry, F&& f) {
    NvtxRange range(entry);
    return guarded(std::forward<F>(f));
}

inline void cuda_check(cudaError_t err, const char* what) {
    if (err == cudaErrorNotSupported) fail(PVO_UNSUPPORTED, std::string(what) + ": shape not supported by the kernel");
    if (err != cudaSuccess) fail(PVO_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(err));
}

// Growable device allocation.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes == 0) bytes = 16;
        if (bytes > cap) {
            // a regrown buffer gets 1.5x headroom (at most +256 MiB): buffers that track a
            // growing graph (one more frame of patches / edges per call) would otherwise be
            // freed and reallocated on every call — cudaFree synchronises the device, and
            // the driver's (un)mapping made the per-frame pipeline's host time spiky
            if (cap) bytes = std::max(bytes, std::min(cap + cap / 2, bytes + (size_t(256) << 20)));
            const auto t0 = std::chrono::steady_clock::now();
            if (p) cudaFree(p);
            p = nullptr;
            cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
            if (trace_alloc())
                std::fprintf(stderr, "[pvo alloc] %zu -> %zu bytes, %.3f ms\n", cap, bytes,
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
            cap = bytes;
        }
        return p;
    }
    static bool trace_alloc() {  // PVO_TRACE_ALLOC=1: log every (re)allocation to stderr
        static const bool on = std::getenv("PVO_TRACE_ALLOC") != nullptr;
        return on;
    }
    template <typename T>
    T* as(size_t count) {
        return static_cast<T*>(get(count * sizeof(T)));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

// Flat BA problem as passed through the C-ABI (host arrays).
struct HostProblem {
    int n_poses = 0;
    const double* poses = nullptr;
    const uint8_t* fixed = nullptr;
    int n_patches = 0, p = 3;
    const int* src = nullptr;
    const double* px = nullptr;
    const double* py = nullptr;
    const double* depth = nullptr;
    const uint8_t* depth_free = nullptr;
    int n_edges = 0;
    const int* e_patch = nullptr;
    const int* e_pose = nullptr;
    const double* e_in = nullptr;  // targets or deltas
    const double* e_w = nullptr;
    double K[4] = {0, 0, 0, 0};
    int image_w = 0, image_h = 0;
    double damping = 1e-4;
};

// Run the device BA on a flattened problem.  Mode flags mirror BAParams.
struct BARun {
    int freeze_targets = 0;
    int iterations = 0;
    int structure_only = 0;
    int gn_step_mode = 0;
    double* out_poses = nullptr;     // host [n_poses][7]
    double* out_depth = nullptr;     // host [n_patches]
    double* residual_norms = nullptr;
    int* n_norms = nullptr;
    double* debug_h = nullptr;
    double* debug_b = nullptr;
    int* n_free_poses = nullptr;
    int* n_free_depths = nullptr;
};

void run_ba(pvo_ctx* ctx, const HostProblem& pr, const BARun& run);

// se3 log (se3.cpp:52-80) on the host; throws Error(PVO_DOMAIN_ERROR).
void se3_log_host(const double* pose7, double* xi6);

}  // namespace pvo_host
