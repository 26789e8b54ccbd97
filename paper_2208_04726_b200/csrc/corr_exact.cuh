// corr_exact.cuh — the reference's correlate_at, evaluated directly (FP64).
//
// The correlation kernels form each output from per-cell dots and per-frame
// Gram terms in FP32 (corr_tma.cu) or FP32-stored terms recombined in FP64
// (corr.cu).  That regrouping is exact in real arithmetic, but when the four
// bilinear taps cancel (anti-correlated neighbour cells) the sampled
// descriptor's norm ||f(x)||^2 = sum_t sum_t' w_t w_t' <f_t, f_t'> is a small
// difference of large terms and loses its relative accuracy.  The kernels
// detect that case — n2 below half of its diagonal part
// sum_t w_t^2 |f_t|^2, i.e. the cross terms <f_t, f_t'> cancel most of it
// (orthogonal taps give n2 = diagonal, positively correlated ones more, a
// sample over the zero padding keeps only diagonal terms), or n2 within 2 %
// of the 1e-12 threshold — and recompute the output here exactly as
// correlation.cpp:8-23 does: every channel sampled by the zero-padded
// bilinear sampler (features.cpp:9-21) in FP64, dot and squared norm
// accumulated in FP64.  (sum_t w_t |f_t|)^2 <= 4 * diagonal, so every output
// whose norm is below 1/8 of the aligned-taps norm is re-evaluated.
#pragma once

#include <cuda_runtime.h>

namespace pvo_dev {

// n2 below this fraction of its diagonal part: recompute directly
constexpr float kCancelRatio = 0.5f;

__device__ __forceinline__ bool corr_needs_exact(float n2, float diag) {
#ifdef PVO_CORR_NO_EXACT  // A/B knob (tools/build_variant.sh): the Gram form alone
    return false;
#else
    return n2 < kCancelRatio * diag || (n2 > 0.98e-12f && n2 < 1.02e-12f);
#endif
}

// Partial sums over channels c = c0, c0 + cstep, ... < C of
//   v_c = sample_zero_padded(x, y, c), dot += g_c v_c, n2 += v_c^2
// with the reference's expression order (features.cpp:10-20, correlation.cpp:16-21).
__device__ inline void corr_exact_partial(const float* g, const float* grid, int W, int H, int C, double x, double y,
                                          int c0, int cstep, double& dot, double& n2) {
    dot = 0.0;
    n2 = 0.0;
    const double xf = floor(x), yf = floor(y);
    if (xf < -1.0 || yf < -1.0 || xf > (double)W || yf > (double)H) return;  // every tap is padding
    const int x0 = (int)xf, y0 = (int)yf;
    const double ax = x - x0, ay = y - y0;
    const bool in00 = x0 >= 0 && y0 >= 0 && x0 < W && y0 < H;
    const bool in10 = x0 + 1 >= 0 && y0 >= 0 && x0 + 1 < W && y0 < H;
    const bool in01 = x0 >= 0 && y0 + 1 >= 0 && x0 < W && y0 + 1 < H;
    const bool in11 = x0 + 1 >= 0 && y0 + 1 >= 0 && x0 + 1 < W && y0 + 1 < H;
    const float* p00 = in00 ? grid + ((size_t)y0 * W + x0) * C : nullptr;
    const float* p10 = in10 ? grid + ((size_t)y0 * W + x0 + 1) * C : nullptr;
    const float* p01 = in01 ? grid + ((size_t)(y0 + 1) * W + x0) * C : nullptr;
    const float* p11 = in11 ? grid + ((size_t)(y0 + 1) * W + x0 + 1) * C : nullptr;
    for (int c = c0; c < C; c += cstep) {
        const double v00 = p00 ? (double)p00[c] : 0.0, v10 = p10 ? (double)p10[c] : 0.0;
        const double v01 = p01 ? (double)p01[c] : 0.0, v11 = p11 ? (double)p11[c] : 0.0;
        const double v = (1 - ax) * (1 - ay) * v00 + ax * (1 - ay) * v10 + (1 - ax) * ay * v01 + ax * ay * v11;
        dot += (double)g[c] * v;
        n2 += v * v;
    }
}

__device__ __forceinline__ float corr_exact_finish(double dot, double n2) {
#ifdef PVO_CORR_EXACT_SENTINEL  // debug knob: mark re-evaluated outputs
    return __int_as_float(0x7fc00001);
#endif
    return n2 > 1e-12 ? (float)(dot / sqrt(n2)) : 0.f;  // correlation.cpp:22
}

// One thread evaluates one output.
__device__ inline float corr_exact_thread(const float* g, const float* grid, int W, int H, int C, double x, double y) {
    double dot, n2;
    corr_exact_partial(g, grid, W, H, C, x, y, 0, 1, dot, n2);
    return corr_exact_finish(dot, n2);
}

// A whole (converged) warp evaluates one output: lanes split the channels,
// fixed-order shuffle tree.
__device__ inline float corr_exact_warp(const float* g, const float* grid, int W, int H, int C, double x, double y) {
    const int lane = threadIdx.x & 31;
    double dot, n2;
    corr_exact_partial(g, grid, W, H, C, x, y, lane, 32, dot, n2);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        dot += __shfl_xor_sync(0xffffffffu, dot, off);
        n2 += __shfl_xor_sync(0xffffffffu, n2, off);
    }
    return corr_exact_finish(dot, n2);
}

}  // namespace pvo_dev
