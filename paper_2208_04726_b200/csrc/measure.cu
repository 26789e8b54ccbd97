// measure.cu — the correlation flow provider's per-edge measurement (§8f row 1),
// sm_100a, FP64 like the reference.
//
// Reference: CorrelationFlowProvider::measure / subpixel_peak / parabola_refine
// (flow_provider.cpp:150-287) and propose's per-edge part (:297-312), over
// correlate_at / correlate_at_cubic (correlation.cpp:8-35) and the
// zero-padded bilinear / Catmull-Rom samplers (features.cpp:9-52).
//
// Two warps per edge (one per pyramid level, joined by a named barrier), lanes
// over channels (C <= 128: four channels per lane, the centre pixel's
// descriptor held in registers).  Every
// correlation sample is the reference's per-channel FP64 formula with the
// reference's operation order (this file is compiled with --fmad=false, so
// every product and sum rounds like the x86-64 reference build); only the
// channel sum is a warp tree instead of a sequential loop (a difference of a
// few ulp).  Work per edge: the 7x7 level-0 slice (shared by the flatness /
// sharpness scores and the level-0 subpixel peak, which the reference
// evaluates twice with identical arguments), the 7x7 level-1 slice, then two
// hill climbs of at most 1 + 6 x 2 x 3 Catmull-Rom samples each (the centre
// value f1 of every parabola step IS the current value: reused).
#include <cuda_runtime.h>

#include <math_constants.h>

#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <cstdint>

#include "ba_common.cuh"
#include "corr_exact.cuh"
#include "kernels.cuh"

namespace pvo_dev {

namespace {

constexpr int kR = 3, kS = 7;  // kCorrRadius, kCorrSize (correlation.hpp:11-12)
constexpr double kStride = 4.0;  // kFeatureStride (features.hpp:46)
constexpr int kCh = 4;           // channels per lane (C <= 128)

struct Level {
    const float* f;  // [H][W][C] of this edge's target frame
    int W, H;
};

// The lane's 4 channels c = lane + 32 k of the centre pixel's descriptor.
struct G4 {
    float v[kCh];
};

// Channel-sum epilogue of correlate_at / correlate_at_cubic (correlation.cpp:16-22)
__device__ __forceinline__ double finish(double dot, double nrm) {
    dot = warp_sum(dot);
    nrm = warp_sum(nrm);
    return nrm > 1e-12 ? dot / sqrt(nrm) : 0.0;
}

// The same epilogue bit for bit as the reference: the per-channel products
// g_c v_c and v_c^2 (each rounded once, as `dot += feature[c] * v` rounds them)
// are staged in the warp's scratch xs[2][128] and summed in channel order
// c = 0, 1, ... by lanes 0 (dot) and 1 (norm) — the sequential loop of
// correlation.cpp:18-21.  Used by the exact replay of near-tie edges.
__device__ __noinline__ double finish_seq(const G4& g, const double* v, int C, double* xs) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < kCh; ++k) {
        const int c = lane + 32 * k;
        if (c < C) {
            xs[c] = (double)g.v[k] * v[k];
            xs[128 + c] = v[k] * v[k];
        }
    }
    __syncwarp();
    double s = 0;
    if (lane < 2) {
        const double* p = xs + 128 * lane;
        int c = 0;
        for (; c + 16 <= C; c += 16) {  // loads batched ahead of the dependent adds
            double t[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) t[k] = p[c + k];
#pragma unroll
            for (int k = 0; k < 16; ++k) s += t[k];
        }
        for (; c < C; ++c) s += p[c];
    }
    const double dot = __shfl_sync(0xffffffffu, s, 0), nrm = __shfl_sync(0xffffffffu, s, 1);
    __syncwarp();  // xs is rewritten by the next sample
    return nrm > 1e-12 ? dot / sqrt(nrm) : 0.0;
}

// correlate_at (correlation.cpp:8-23) with sample_zero_padded (features.cpp:9-21).
// Not inlined: one copy of the sampler keeps the kernel inside the instruction cache.
// xs: null -> warp-tree channel sum; else the reference's sequential sum (finish_seq)
__device__ __noinline__ double corr_bilinear(const float* f, int W, int H, int C, G4 g, double x, double y,
                                             double* xs = nullptr) {
    const int lane = threadIdx.x & 31;
    const int x0 = (int)floor(x), y0 = (int)floor(y);
    const double ax = x - x0, ay = y - y0;
    const double w[4] = {(1 - ax) * (1 - ay), ax * (1 - ay), (1 - ax) * ay, ax * ay};
    double v[kCh] = {0, 0, 0, 0};
#pragma unroll
    for (int t = 0; t < 4; ++t) {  // taps in the reference's order: (x0,y0) (x0+1,y0) (x0,y0+1) (x0+1,y0+1)
        const int xi = x0 + (t & 1), yi = y0 + (t >> 1);
        const bool in = xi >= 0 && yi >= 0 && xi < W && yi < H;
        const float* p = f + ((size_t)(in ? yi : 0) * W + (in ? xi : 0)) * C + lane;
#pragma unroll
        for (int k = 0; k < kCh; ++k) {
            const double val = (in && lane + 32 * k < C) ? (double)__ldg(p + 32 * k) : 0.0;
            v[k] = t == 0 ? w[0] * val : v[k] + w[t] * val;
        }
    }
    if (xs) return finish_seq(g, v, C, xs);
    double dot = 0, nrm = 0;
#pragma unroll
    for (int k = 0; k < kCh; ++k) {
        dot += (double)g.v[k] * v[k];
        nrm += v[k] * v[k];
    }
    return finish(dot, nrm);
}

__device__ __forceinline__ void cubic_weights(double t, double w[4]) {  // features.cpp:29-34
    w[0] = ((-0.5 * t + 1.0) * t - 0.5) * t;
    w[1] = (1.5 * t - 2.5) * t * t + 1.0;
    w[2] = ((-1.5 * t + 2.0) * t + 0.5) * t;
    w[3] = (0.5 * t - 0.5) * t * t;
}

// A square window of n x n cells of one level staged in the warp's shared
// memory for the exact replay ([cell][C + 1] floats: an odd stride, so lanes on
// distinct cells or on consecutive channels hit distinct banks); cells outside
// the grid hold 0, the reference's zero padding (features.cpp:15-17).
struct SmemWin {
    float* s = nullptr;
    int x0 = 0, y0 = 0, n = 0, stride = 0;
    __device__ bool holds(int x, int y, int span) const {  // cells x .. x + span - 1 (same in y)
        return s && x >= x0 && y >= y0 && x + span <= x0 + n && y + span <= y0 + n;
    }
    __device__ const float* cell(int x, int y) const { return s + ((y - y0) * n + (x - x0)) * stride; }
};

__device__ void stage_window(SmemWin& w, const Level& L, int C, int x0, int y0, int n) {
    const int lane = threadIdx.x & 31;
    __syncwarp();  // the previous window's readers are done
    w.x0 = x0;
    w.y0 = y0;
    w.n = n;
    w.stride = C + 1;
    const int cells = n * n;
    constexpr int kBatch = 16;  // cells whose loads are all in flight before any store
    for (int q0 = 0; q0 < cells; q0 += kBatch) {
        float r[kBatch][kCh];
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            const int q = q0 + j, x = x0 + q % n, y = y0 + q / n;
            const bool in = q < cells && x >= 0 && y >= 0 && x < L.W && y < L.H;
            const float* src = L.f + (in ? (size_t)y * L.W + x : 0) * C;
#pragma unroll
            for (int k = 0; k < kCh; ++k) r[j][k] = (in && lane + 32 * k < C) ? __ldg(src + lane + 32 * k) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < kBatch; ++j)
#pragma unroll
            for (int k = 0; k < kCh; ++k)
                if (q0 + j < cells && lane + 32 * k < C) w.s[(q0 + j) * w.stride + lane + 32 * k] = r[j][k];
    }
    __syncwarp();
}

// correlate_at_cubic (correlation.cpp:25-35) with sample_cubic (features.cpp:23-52).
// kPreload (the exact replay, which has the registers): all 16 taps' channel
// loads are issued first — from the staged window when it holds the footprint —
// then the reference's per-channel operation order; out-of-grid taps read as 0,
// and adding their zero term where the reference skips it (features.cpp:40-47)
// leaves every sum bit-identical (x + 0 == x; +0 + -0 == +0).  Otherwise taps
// outer with one address per tap (few registers: the Gram-form kernel's rare
// direct re-evaluations must not make its hill climb spill).
template <bool kPreload>
__device__ __noinline__ double corr_cubic_t(const float* f, int W, int H, int C, G4 g, double x, double y,
                                            double* xs, const SmemWin* win) {
    const int lane = threadIdx.x & 31;
    const int x0 = (int)floor(x), y0 = (int)floor(y);
    double wx[4], wy[4];
    cubic_weights(x - x0, wx);
    cubic_weights(y - y0, wy);
    double v[kCh] = {0, 0, 0, 0};
    if constexpr (kPreload) {
        float val[16][kCh];
        if (win && win->holds(x0 - 1, y0 - 1, 4)) {  // the 4 x 4 footprint is staged (zeros outside the grid)
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                const float* p = win->cell(x0 - 1 + (t & 3), y0 - 1 + (t >> 2)) + lane;
#pragma unroll
                for (int k = 0; k < kCh; ++k) val[t][k] = lane + 32 * k < C ? p[32 * k] : 0.f;
            }
        } else {
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                const int xi = x0 - 1 + (t & 3), yi = y0 - 1 + (t >> 2);
                const bool in = xi >= 0 && xi < W && yi >= 0 && yi < H;
                const float* p = f + (in ? (size_t)yi * W + xi : 0) * C + lane;
#pragma unroll
                for (int k = 0; k < kCh; ++k) val[t][k] = (in && lane + 32 * k < C) ? __ldg(p + 32 * k) : 0.f;
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            double row[kCh] = {0, 0, 0, 0};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int k = 0; k < kCh; ++k) row[k] += wx[i] * (double)val[4 * j + i][k];
#pragma unroll
            for (int k = 0; k < kCh; ++k) v[k] += wy[j] * row[k];
        }
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int yi = y0 - 1 + j;
            if (yi < 0 || yi >= H) continue;
            double row[kCh] = {0, 0, 0, 0};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int xi = x0 - 1 + i;
                if (xi < 0 || xi >= W) continue;
                const float* p = f + ((size_t)yi * W + xi) * C + lane;
#pragma unroll
                for (int k = 0; k < kCh; ++k)
                    if (lane + 32 * k < C) row[k] += wx[i] * (double)__ldg(p + 32 * k);
            }
#pragma unroll
            for (int k = 0; k < kCh; ++k) v[k] += wy[j] * row[k];
        }
    }
    if (xs) return finish_seq(g, v, C, xs);
    double dot = 0, nrm = 0;
#pragma unroll
    for (int k = 0; k < kCh; ++k) {
        dot += (double)g.v[k] * v[k];
        nrm += v[k] * v[k];
    }
    return finish(dot, nrm);
}
__device__ __forceinline__ double corr_cubic(const float* f, int W, int H, int C, G4 g, double x, double y,
                                            double* xs = nullptr) {
    return corr_cubic_t<false>(f, W, H, C, g, x, y, xs, nullptr);
}
__device__ __forceinline__ double corr_cubic_exact(const float* f, int W, int H, int C, G4 g, double x, double y,
                                                  double* xs, const SmemWin* win) {
    return win ? corr_cubic_t<true>(f, W, H, C, g, x, y, xs, win) : corr_cubic_t<false>(f, W, H, C, g, x, y, xs, win);
}

// subpixel_peak (flow_provider.cpp:167-205) from the 7x7 slice `vals` (already
// evaluated at base + (beta - 3, alpha - 3)); returns the offset in cells
__device__ void subpixel_peak(const Level& L, int C, G4 g, double bx, double by,
                              const double* vals, double* ox, double* oy, bool* on_border, double* xs,
                              SmemWin* win) {
    int best_a = kR, best_b = kR;
    double best = -CUDART_INF;
    for (int alpha = 0; alpha < kS; ++alpha)
        for (int beta = 0; beta < kS; ++beta) {
            const double v = vals[alpha * kS + beta];
            if (v > best) {
                best = v;
                best_a = alpha;
                best_b = beta;
            }
        }
    *on_border = best_a == 0 || best_a == kS - 1 || best_b == 0 || best_b == kS - 1;
    double dx = best_b - kR, dy = best_a - kR;
    // every climb sample lies within 1 cell of the discrete peak (sum of steps < 1): its
    // Catmull-Rom footprint is inside the 6 x 6 window at floor(peak) - 2
    if (win && fabs(bx) < 1e8 && fabs(by) < 1e8)
        stage_window(*win, L, C, (int)floor(bx + dx) - 2, (int)floor(by + dy) - 2, 6);
    double current = corr_cubic_exact(L.f, L.W, L.H, C, g, bx + dx, by + dy, xs, win);
    double h = 0.5;
    for (int hs = 0; hs < 6; ++hs, h *= 0.5) {
        for (int ax = 0; ax < 2; ++ax) {
            const bool along_x = ax == 0;
            // parabola_refine (flow_provider.cpp:152-162); f1 = the current value
            const double x = bx + dx, y = by + dy;
            const double f0 =
                corr_cubic_exact(L.f, L.W, L.H, C, g, x - (along_x ? h : 0), y - (along_x ? 0 : h), xs, win);
            const double f1 = current;
            const double f2 =
                corr_cubic_exact(L.f, L.W, L.H, C, g, x + (along_x ? h : 0), y + (along_x ? 0 : h), xs, win);
            const double denom = f0 - 2 * f1 + f2;
            double step = 0.0;
            if (!(fabs(denom) < 1e-12 || denom > 0)) step = fmin(fmax(0.5 * h * (f0 - f2) / denom, -h), h);
            if (step == 0.0) continue;
            const double nx = dx + (along_x ? step : 0);
            const double ny = dy + (along_x ? 0 : step);
            const double value = corr_cubic_exact(L.f, L.W, L.H, C, g, bx + nx, by + ny, xs, win);
            if (value >= current) {  // hill climb only
                dx = nx;
                dy = ny;
                current = value;
            }
        }
    }
    *ox = dx;
    *oy = dy;
}

// The direct measurement of edge e by a warp pair (warp `level` of the pair):
// every sample through the per-channel samplers above.  xs: null -> warp-tree
// channel sums (the PVO_MEASURE_DIRECT A/B kernel); else the warp's [2][128]
// scratch -> the reference's sequential channel sums, so every sample, and
// with it every decision, is bit-identical to the reference (the exact replay
// of near-tie edges, measure_exact_kernel).  vals: the warp's 7x7 slice;
// peak1 / border1: the pair's level-1 result; bar: the pair's named barrier.
__device__ __forceinline__ void measure_direct_edge(const MeasureParams& a, int e, int level, double* vals,
                                                    double* peak1, int* border1, int bar, double* xs,
                                                    float* win_buf) {
    const int lane = threadIdx.x & 31;
    double cx, cy;
    bool behind;
    if (a.centers) {
        cx = a.centers[2 * e];
        cy = a.centers[2 * e + 1];
        behind = a.behind && a.behind[e];
    } else {  // window mode: reproject_patch of the current state (camera.cpp:47-71)
        const int k = a.e_patch[e];
        const SE3 pi = se3_load(a.poses + 7 * a.patch_src[k]);
        const SE3 pj = se3_load(a.poses + 7 * a.e_pose[e]);
        const Cam K{a.K[0], a.K[1], a.K[2], a.K[3]};
        reproject_center(pi, pj, K, a.patch_x + 9 * (size_t)k, a.patch_y + 9 * (size_t)k, a.depth[k], &cx, &cy,
                         &behind);
    }
    double dxo = 0, dyo = 0, wgt = 0.01;
    int flags = 0;
    const bool valid = !behind && isfinite(cx) && isfinite(cy);
    if (behind) {
        flags = 4;  // flow_provider.cpp:301-302
    } else if (!valid) {
        flags = 8;
        if (lane == 0 && level == 0) atomicOr(a.status, 1 << kDevBadCoords);
    }
    // level-0 results carried across the pair's barrier
    bool flat = true, border0 = false;
    double confidence = 0.01, p0x = 0, p0y = 0;
    if (valid) {
        const int slot = a.e_slot ? a.e_slot[e] : a.pose_slot[a.e_pose[e]];
        const float* gp = a.patch_feats + (size_t)a.e_patch[e] * 2 * 9 * a.channels;
        const Level L = level ? Level{a.feat1 + (size_t)slot * a.h1 * a.w1 * a.channels, a.w1, a.h1}
                              : Level{a.feat0 + (size_t)slot * a.h0 * a.w0 * a.channels, a.w0, a.h0};
        G4 g;
#pragma unroll
        for (int k = 0; k < kCh; ++k) {
            const int c = lane + 32 * k;
            g.v[k] = c < a.channels ? gp[(9 * level + 4) * a.channels + c] : 0.f;  // centre pixel of the level
        }
        double* v = vals;
        const double sc = level ? kStride * kStride : kStride;
        const double bx = cx / sc, by = cy / sc;
        SmemWin win;
        win.s = win_buf;
        if (xs) {  // exact: a lane per slice sample, the reference's sequential channel loop
            const float* gc = gp + (9 * level + 4) * a.channels;
            const bool span = fabs(bx) < 1e8 && fabs(by) < 1e8;
            if (span && win.s)  // the 8 x 8 cells the 7 x 7 bilinear samples touch
                stage_window(win, L, a.channels, (int)floor(bx) - kR, (int)floor(by) - kR, 8);
            for (int i = lane; i < kS * kS; i += 32) {
                const int alpha = i / kS, beta = i % kS;
                const double x = bx + beta - kR, y = by + alpha - kR;
                double dot = 0, n2 = 0;
                const int x0 = span ? (int)floor(x) : 0, y0 = span ? (int)floor(y) : 0;
                if (span && win.s && win.holds(x0, y0, 2)) {
                    // features.cpp:9-21 per channel (window zeros = out-of-grid taps), sums in order
                    const double ax = x - x0, ay = y - y0;
                    const float *p00 = win.cell(x0, y0), *p10 = win.cell(x0 + 1, y0);
                    const float *p01 = win.cell(x0, y0 + 1), *p11 = win.cell(x0 + 1, y0 + 1);
#pragma unroll 8
                    for (int c = 0; c < a.channels; ++c) {
                        const double vv = (1 - ax) * (1 - ay) * (double)p00[c] + ax * (1 - ay) * (double)p10[c] +
                                          (1 - ax) * ay * (double)p01[c] + ax * ay * (double)p11[c];
                        dot += (double)__ldg(gc + c) * vv;
                        n2 += vv * vv;
                    }
                } else {
                    corr_exact_partial(gc, L.f, L.W, L.H, a.channels, x, y, 0, 1, dot, n2);
                }
                v[i] = n2 > 1e-12 ? dot / sqrt(n2) : 0.0;  // correlation.cpp:22
            }
        } else {
            for (int i = 0; i < kS * kS; ++i) {
                const int alpha = i / kS, beta = i % kS;
                const double va = corr_bilinear(L.f, L.W, L.H, a.channels, g, bx + beta - kR, by + alpha - kR);
                if (lane == 0) v[i] = va;
            }
        }
        __syncwarp();
        if (level == 1) {
            // level-1 subpixel peak (flow_provider.cpp:264-265), needed unless level 0 is flat
            double px, py;
            bool border;
            subpixel_peak(L, a.channels, g, bx, by, v, &px, &py, &border, xs, win.s ? &win : nullptr);
            if (lane == 0) {
                peak1[0] = px;
                peak1[1] = py;
                *border1 = border;
            }
        } else {
            // level 0: flatness / sharpness scores on the slice (flow_provider.cpp:217-250)
            double peak = -CUDART_INF, minimum = CUDART_INF, mean = 0;
            int peak_a = 0, peak_b = 0;
            for (int i = 0; i < kS * kS; ++i) {
                const double val = v[i];
                mean += val;
                minimum = fmin(minimum, val);
                if (val > peak) {
                    peak = val;
                    peak_a = i / kS;
                    peak_b = i % kS;
                }
            }
            mean /= kS * kS;
            const double peak_to_mean = (peak - minimum) / (mean - minimum + 1e-9);
            flat = !(peak_to_mean >= 1.05);
            if (!flat) {
                double second = -CUDART_INF;
                for (int i = 0; i < kS * kS; ++i) {
                    const int alpha = i / kS, beta = i % kS;
                    if (max(abs(alpha - peak_a), abs(beta - peak_b)) <= 1) continue;
                    second = fmax(second, v[i]);
                }
                const double score = 2.0 * (peak - 0.75) + (peak - second - 0.08);
                confidence = fmin(fmax(1.0 / (1.0 + exp(-12.0 * score)), 0.01), 0.99);
                subpixel_peak(L, a.channels, g, bx, by, v, &p0x, &p0y, &border0, xs, win.s ? &win : nullptr);
            }
        }
    }
    // the pair meets on its named barrier at one program point, unconditionally (also
    // for behind / non-finite edges), each warp converged: bar.sync counts threads
    __syncwarp();
    asm volatile("bar.sync %0, 64;" ::"r"(bar) : "memory");
    if (valid && level == 0) {
        if (flat) {
            flags = 1;  // flat: delta 0, weight 0.01
        } else {
            const bool b1 = *border1;
            const double p1x = peak1[0], p1y = peak1[1];
            const double e0x = kStride * p0x, e0y = kStride * p0y;
            const double e1x = kStride * kStride * p1x, e1y = kStride * kStride * p1y;
            if (border0 && b1) {
                flags = 2;  // out of range: delta 0, weight 0.01
            } else {
                if (border0) {
                    dxo = e1x;
                    dyo = e1y;
                    confidence = fmin(confidence, 0.25);
                } else {
                    dxo = e0x;
                    dyo = e0y;
                    const double ddx = e1x - e0x, ddy = e1y - e0y;
                    if (!b1 && sqrt(ddx * ddx + ddy * ddy) > 2.0 * kStride * kStride)
                        confidence = fmin(confidence, 0.25);
                }
                wgt = confidence;
            }
        }
    }
    if (level == 1) return;
    if (lane == 0) {
        a.delta[2 * e] = dxo;
        a.delta[2 * e + 1] = dyo;
        a.weight[2 * e] = wgt;
        a.weight[2 * e + 1] = wgt;
        if (a.flags) a.flags[e] = (uint8_t)flags;
    }
}

#ifndef PVO_MEASURE_MINB
#define PVO_MEASURE_MINB 1
#endif
// The direct kernel (PVO_MEASURE_DIRECT=1; A/B): four edges per block.
__global__ void __launch_bounds__(256, PVO_MEASURE_MINB) measure_kernel(MeasureParams a) {
    __shared__ double s_vals[8][kS * kS];
    __shared__ double s_peak1[4][2];
    __shared__ int s_border1[4];
    const int warp = threadIdx.x >> 5;
    const int pair = warp >> 1, level = warp & 1;
    const int e = blockIdx.x * 4 + pair;
    if (e >= a.n_edges) return;  // both warps of the pair
    measure_direct_edge(a, e, level, s_vals[warp], s_peak1[pair], &s_border1[pair], 1 + pair, nullptr, nullptr);
}

// Exact replay: the edges the Gram-form kernel found within a rounding margin of
// one of the reference's discrete decisions (a tied argmax, a hill-climb
// comparison, a parabola denominator or the flatness / level-consistency
// thresholds; measure_gram_kernel) are measured again, a warp pair per edge,
// with every sample bit-identical to the reference.  The list is
// replay[0] = count, replay[1 ..] = edges; it is left zeroed for the next call.
constexpr int kExactBlocks = 296;
constexpr int kExactWinFloats = 64 * 129;  // an 8 x 8 window at C <= 128
constexpr int kExactSmem = 2 * kExactWinFloats * (int)sizeof(float);
__global__ void __launch_bounds__(64) measure_exact_kernel(MeasureParams a) {
    __shared__ double s_vals[2][kS * kS];
    __shared__ double s_xs[2][2 * 128];
    __shared__ double s_peak1[2];
    __shared__ int s_border1;
    extern __shared__ float s_win[];  // [2][kExactWinFloats]
    const int warp = threadIdx.x >> 5;
    const int n = min(__ldcg(a.replay), a.n_edges);
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        measure_direct_edge(a, __ldcg(a.replay + 1 + i), warp, s_vals[warp], s_peak1, &s_border1, 1, s_xs[warp],
                            s_win + warp * kExactWinFloats);
        __syncthreads();  // s_peak1 / s_border1 are rewritten by the next edge
    }
    // the last block to finish leaves the count zero for the next launch
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(a.replay_done, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        if (a.replay_stat) *a.replay_stat = a.replay[0];
        a.replay[0] = 0;
        *a.replay_done = 0;
    }
}

// ============================================================================
// Gram-form measurement (the default when the frame store's FP64 neighbour-Gram
// maps exist).  By linearity every sample the provider takes is a weighted sum
// of integer cells, f(x) = sum_t w_t f_t, so
//   dot   = <g, f(x)>  = sum_t w_t <g, f_t>               (cell dots, FP64)
//   |f|^2 = sum_t sum_t' w_t w_t' <f_t, f_t'>              (frame Gram maps, FP64)
// with the reference's own weights (bilinear: features.cpp:10-20; Catmull-Rom:
// features.cpp:23-52, this file is compiled with --fmad=false so they round
// as the x86-64 reference build does).  Per edge and level the warp computes
// the <g, f_t> of the 8x8 slice window and of the 6x6 window around the
// discrete peak (lane per cell, channels in order, FP64 sums of exact
// products) and stages their Gram terms in shared memory; a sample is then a
// few dozen FP64 operations instead of a pass over all channels, and the hill
// climb's samples need no channel reduction (16 lanes, one per tap).  Products
// of FP32 features are exact in FP64, so the regrouping changes only the
// summation order (~1e-16 relative) — except where the taps cancel: a sample
// whose |f|^2 falls below half its diagonal part (or near the 1e-12 threshold,
// correlation.cpp:22) is re-evaluated by the direct samplers above, as are the
// (rounding-edge) samples whose taps leave the staged windows.
// ============================================================================
__host__ __device__ constexpr int g25_index(int dx, int dy) { return dy == 0 ? dx : 4 + (dy - 1) * 7 + dx + 3; }

constexpr int kG25TileW = 8, kG25TileH = 4;                   // cells per block
constexpr int kG25SW = kG25TileW + 6, kG25SH = kG25TileH + 3;  // staged: cols x-3 .. x+10, rows y .. y+6

__global__ void __launch_bounds__(256) gram25_kernel(const float* feat, int W, int H, int C, double* g25) {
    extern __shared__ float s_f[];  // [kG25SH * kG25SW][C + 1] (odd stride: conflict-free per cell)
    const int tx0 = blockIdx.x * kG25TileW, ty0 = blockIdx.y * kG25TileH;
    const int stride = C + 1;
    // staged in batches: every thread's loads of a batch are in flight before its stores
    constexpr int kStageBatch = 8;
    const int total = kG25SW * kG25SH * C;
    for (int t0 = threadIdx.x; t0 < total; t0 += kStageBatch * blockDim.x) {
        float r[kStageBatch];
#pragma unroll
        for (int b = 0; b < kStageBatch; ++b) {
            const int t = t0 + b * blockDim.x;
            const int cell = t / C, c = t - cell * C;
            const int x = tx0 - 3 + cell % kG25SW, y = ty0 + cell / kG25SW;
            r[b] = (t < total && x >= 0 && y >= 0 && x < W && y < H) ? __ldg(feat + ((size_t)y * W + x) * C + c) : 0.f;
        }
#pragma unroll
        for (int b = 0; b < kStageBatch; ++b) {
            const int t = t0 + b * blockDim.x;
            const int cell = t / C, c = t - cell * C;
            if (t < total) s_f[cell * stride + c] = r[b];
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < kG25TileW * kG25TileH * kGram25; t += blockDim.x) {
        const int cl = t / kGram25, m = t - cl * kGram25;
        const int lx = cl % kG25TileW, ly = cl / kG25TileW;
        const int x = tx0 + lx, y = ty0 + ly;
        if (x >= W || y >= H) continue;
        const int dy = m < 4 ? 0 : 1 + (m - 4) / 7, dx = m < 4 ? m : (m - 4) % 7 - 3;
        const float* fa = s_f + (ly * kG25SW + lx + 3) * stride;
        const float* fb = s_f + ((ly + dy) * kG25SW + lx + 3 + dx) * stride;  // zero outside the grid
        // FP64 sums of exact products (an FP32 x FP32 product is exact in FP64, so the
        // FMA rounds like the separate add), four interleaved chains
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        int c = 0;
        for (; c + 4 <= C; c += 4) {
            s0 = __fma_rn((double)fa[c], (double)fb[c], s0);
            s1 = __fma_rn((double)fa[c + 1], (double)fb[c + 1], s1);
            s2 = __fma_rn((double)fa[c + 2], (double)fb[c + 2], s2);
            s3 = __fma_rn((double)fa[c + 3], (double)fb[c + 3], s3);
        }
        for (; c < C; ++c) s0 = __fma_rn((double)fa[c], (double)fb[c], s0);
        g25[((size_t)y * W + x) * kGram25 + m] = (s0 + s1) + (s2 + s3);
    }
}

#ifndef PVO_MEASURE_WARPS
#define PVO_MEASURE_WARPS 8
#endif
constexpr int kMeasWarps = PVO_MEASURE_WARPS;  // kMeasWarps / 2 edges per block, a warp per (edge, level)

struct alignas(16) MeasWarpSmem {
    float g[128];         // the level's centre-pixel descriptor
    double v[kS * kS];    // the 7x7 slice
    double sd[64];        // <g, f> of the 8x8 slice window (kept: the climb window reuses them)
    double xs[256];       // finish_seq scratch (exact re-evaluation of near-tie comparisons)
    union {
        double sgr[64][5];  // Gram (0,0) (1,0) (0,1) (1,1) (-1,1) of the slice window
        struct {
            double d[36];             // <g, f> of the 6x6 window around the discrete peak
            double gr[36][kGram25];   // its Gram maps
        } climb;
    } u;
};
constexpr int kMeasSmem = kMeasWarps * (int)sizeof(MeasWarpSmem);

#ifndef PVO_CELL_DOT_UNROLL
#define PVO_CELL_DOT_UNROLL 4
#endif
constexpr int kCellDotUnroll = PVO_CELL_DOT_UNROLL;  // channel quads per batch of loads in flight (A/B knob)
// <g, f_cell> (g in shared memory): FP64 sums of exact products (explicit FMAs:
// the product of two FP32 values is exact in FP64, so an FMA rounds like the
// separate add), four interleaved partial sums (short dependent chains)
__device__ __noinline__ double cell_dot(const float* gs, const float* fc, int C) {
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    if ((C & 3) == 0) {
        const float4* f4 = reinterpret_cast<const float4*>(fc);
        const float4* g4 = reinterpret_cast<const float4*>(gs);
#pragma unroll(kCellDotUnroll)
        for (int q = 0; q < (C >> 2); ++q) {
            const float4 fv = __ldg(f4 + q), gv = g4[q];
            s0 = __fma_rn((double)gv.x, (double)fv.x, s0);
            s1 = __fma_rn((double)gv.y, (double)fv.y, s1);
            s2 = __fma_rn((double)gv.z, (double)fv.z, s2);
            s3 = __fma_rn((double)gv.w, (double)fv.w, s3);
        }
    } else {
        for (int c = 0; c < C; ++c) s0 = __fma_rn((double)gs[c], (double)__ldg(fc + c), s0);
    }
    return (s0 + s1) + (s2 + s3);
}

// Two cells at once (independent load streams in flight together).
__device__ __noinline__ void cell_dot2(const float* gs, const float* fa, const float* fb, int C, double* da,
                                       double* db) {
    double a0 = 0, a1 = 0, b0 = 0, b1 = 0;
    if ((C & 3) == 0) {
        const float4* fa4 = reinterpret_cast<const float4*>(fa);
        const float4* fb4 = reinterpret_cast<const float4*>(fb);
        const float4* g4 = reinterpret_cast<const float4*>(gs);
#pragma unroll(kCellDotUnroll)
        for (int q = 0; q < (C >> 2); ++q) {
            const float4 va = __ldg(fa4 + q), vb = __ldg(fb4 + q), gv = g4[q];
            a0 = __fma_rn((double)gv.x, (double)va.x, a0);
            b0 = __fma_rn((double)gv.x, (double)vb.x, b0);
            a1 = __fma_rn((double)gv.y, (double)va.y, a1);
            b1 = __fma_rn((double)gv.y, (double)vb.y, b1);
            a0 = __fma_rn((double)gv.z, (double)va.z, a0);
            b0 = __fma_rn((double)gv.z, (double)vb.z, b0);
            a1 = __fma_rn((double)gv.w, (double)va.w, a1);
            b1 = __fma_rn((double)gv.w, (double)vb.w, b1);
        }
    } else {
        for (int c = 0; c < C; ++c) {
            a0 = __fma_rn((double)gs[c], (double)__ldg(fa + c), a0);
            b0 = __fma_rn((double)gs[c], (double)__ldg(fb + c), b0);
        }
    }
    *da = a0 + a1;
    *db = b0 + b1;
}

// Per-lane shared-memory offsets (in doubles, relative to the lane's tap cell's
// Gram record) of the 16 Gram terms <f_p, f_q> of a 4x4 tap footprint in the
// 6x6 climb window: the record of p at offset q - p when that offset lies in
// the stored half plane, else the record of q at offset p - q.
__device__ __forceinline__ void cubic_gram_offsets(int p, int off[16]) {
    const int pi = p & 3, pj = p >> 2;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int ddx = (q & 3) - pi, ddy = (q >> 2) - pj;
        const bool fwd = ddy > 0 || (ddy == 0 && ddx >= 0);
        off[q] = fwd ? g25_index(ddx, ddy) : (ddy * 6 + ddx) * kGram25 + g25_index(-ddx, -ddy);
    }
}

// One Catmull-Rom correlation sample on a half warp (lane & 15 = tap j * 4 + i)
// from the staged 6x6 window at (qx, qy); both halves call it together (each
// with its own position).  *redo: the sample must be evaluated directly.
__device__ __noinline__ double cubic_gram(const MeasWarpSmem& S, const int* off, int qx, int qy, double x, double y,
                             bool* redo) {
    const int p = threadIdx.x & 15;
    const int x0 = (int)floor(x), y0 = (int)floor(y);
    double wx[4], wy[4];
    cubic_weights(x - x0, wx);
    cubic_weights(y - y0, wy);
    const int bxl = x0 - 1 - qx, byl = y0 - 1 - qy;  // window index of tap (0, 0)
    const bool inwin = bxl >= 0 && byl >= 0 && bxl <= 2 && byl <= 2;
    double dot = 0, n2 = 0, diag = 0;
    if (inwin) {
        const int pi = p & 3, pj = p >> 2;
        const int cp = (byl + pj) * 6 + bxl + pi;
        const double* gp = &S.u.climb.gr[cp][0];
        double r0 = 0, r1 = 0;
#pragma unroll
        for (int q = 0; q < 16; q += 2) {
            r0 = __fma_rn(wy[q >> 2] * wx[q & 3], gp[off[q]], r0);
            r1 = __fma_rn(wy[(q + 1) >> 2] * wx[(q + 1) & 3], gp[off[q + 1]], r1);
        }
        const double wp = wy[pj] * wx[pi];
        dot = wp * S.u.climb.d[cp];
        n2 = wp * (r0 + r1);
        diag = wp * wp * gp[0];
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
        dot += __shfl_xor_sync(0xffffffffu, dot, o);
        n2 += __shfl_xor_sync(0xffffffffu, n2, o);
        diag += __shfl_xor_sync(0xffffffffu, diag, o);
    }
    *redo = !inwin || n2 < 0.5 * diag || (n2 > 0.98e-12 && n2 < 1.02e-12);
    return n2 > 1e-12 ? dot / sqrt(n2) : 0.0;
}

// Rounding margin of the Gram-form samples for the discrete decisions: a sample
// is a cosine against g (|value| <= |g|) whose regrouped FP64 sums differ from
// the reference's sequential ones by ~1e-16 |g|; any decision closer than
// kTieRel |g| to flipping sends the edge to the exact replay.
constexpr double kTieRel = 1e-12;
constexpr double kTieExactRel = 1e-14;  // residual margin after an exact re-evaluation of both sides
// near-tie reasons (bit mask)
constexpr int kTieArgmax = 1, kTieFlat = 2, kTieDenom = 4, kTieStep = 8, kTieClimb = 16, kTieDist = 32;

// Two Catmull-Rom samples with the reference's exact arithmetic (kept out of
// line: the Gram-form climb's registers stay free of the direct sampler's).
__device__ __noinline__ void resolve_exact(const Level& L, int C, const G4& g4, double xa, double ya, double xb,
                                           double yb, double* xs, double* va, double* vb) {
    *va = corr_cubic(L.f, L.W, L.H, C, g4, xa, ya, xs);
    *vb = corr_cubic(L.f, L.W, L.H, C, g4, xb, yb, xs);
}

// Every tap of the Catmull-Rom sample at (x, y) lies outside the grid (the
// sample is an exact zero in the reference and here).
__device__ __forceinline__ bool cubic_pad(double x, double y, int W, int H) {
    const double xf = floor(x), yf = floor(y);
    return xf + 2 < 0 || xf - 1 >= W || yf + 2 < 0 || yf - 1 >= H;
}

// First-occurrence argmax of the slice (the reference's `v > best` scan order)
// as a warp reduction: lanes hold samples lane and lane + 32.  *tie: another
// sample lies within eps of the maximum (the reference's choice depends on
// rounding there).
__device__ __forceinline__ int slice_argmax(const double* v, double eps = -1.0, int* tie = nullptr,
                                            const unsigned* pad = nullptr) {
    const int lane = threadIdx.x & 31;
    double b = -CUDART_INF;
    int bi = kR * kS + kR;  // no sample above -inf: the reference keeps (3, 3)
    for (int i = lane; i < kS * kS; i += 32)
        if (v[i] > b) {
            b = v[i];
            bi = i;
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, b, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > b || (ob == b && oi < bi && ob > -CUDART_INF)) {
            b = ob;
            bi = oi;
        }
    }
    if (tie) {
        // exact zeros of padding-only samples are exact in the reference too: two
        // of them never tie by rounding (pad: bit n of lane l = sample l + 32 n)
        const bool bpad = pad && ((__shfl_sync(0xffffffffu, pad[0], bi & 31) >> (bi >> 5)) & 1);
        bool near = false;
        for (int i = lane, n = 0; i < kS * kS; i += 32, ++n)
            near |= i != bi && v[i] >= b - eps && !(bpad && ((pad[0] >> n) & 1));
        if (__any_sync(0xffffffffu, near)) *tie |= kTieArgmax;
    }
    return bi;
}

// subpixel_peak (flow_provider.cpp:167-205) on the Gram form: the discrete
// argmax of the slice S.v, the 6x6 window around it staged, then the hill climb
// with f0 / f2 of each parabola step on the two half warps.
__device__ __noinline__ void subpixel_peak_gram(MeasWarpSmem& S, const Level& L, int C, const double* gm, const G4& g4,
                                   double bx, double by, int ox, int oy, int bi, double* px, double* py, double eps,
                                   int* tie) {
    const int lane = threadIdx.x & 31;
    const int best_a = bi / kS, best_b = bi % kS;  // the slice argmax (measure_task)
    double dx = best_b - kR, dy = best_a - kR;
    if (!(fabs(bx) < 1e8 && fabs(by) < 1e8)) {  // every sample is zero padding: no parabola step moves
        *px = dx;
        *py = dy;
        return;
    }
    const int qx = (int)floor(bx + dx) - 2, qy = (int)floor(by + dy) - 2;
    __syncwarp();  // the slice Gram buffer is reused for the climb window
    {  // cells lane and lane + 32 (lanes 0-3); dots outside the slice window computed
       // here, a lane's two fresh cells together (one load stream pair in flight)
        int cx[2], cy[2], kind[2];  // kind: 0 zero padding, 1 slice dot, 2 fresh dot
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int q = lane + 32 * h;
            cx[h] = qx + q % 6;
            cy[h] = qy + q / 6;
            const int sx = cx[h] - ox, sy = cy[h] - oy;
            const bool in = q < 36 && cx[h] >= 0 && cy[h] >= 0 && cx[h] < L.W && cy[h] < L.H;
            kind[h] = !in ? 0 : (sx >= 0 && sx < 8 && sy >= 0 && sy < 8) ? 1 : 2;
        }
        double dv[2];
#pragma unroll
        for (int h = 0; h < 2; ++h)
            dv[h] = kind[h] == 1 ? S.sd[(cy[h] - oy) * 8 + cx[h] - ox] : 0.0;
        const float* f0 = L.f + ((size_t)cy[0] * L.W + cx[0]) * C;
        const float* f1 = L.f + ((size_t)cy[1] * L.W + cx[1]) * C;
        if (kind[0] == 2 && kind[1] == 2)
            cell_dot2(S.g, f0, f1, C, &dv[0], &dv[1]);
        else if (kind[0] == 2)
            dv[0] = cell_dot(S.g, f0, C);
        else if (kind[1] == 2)
            dv[1] = cell_dot(S.g, f1, C);
        S.u.climb.d[lane] = dv[0];
        if (lane < 4) S.u.climb.d[lane + 32] = dv[1];
    }
    // the window's Gram records: each window row is 6 x 25 contiguous doubles of
    // the map, 5 coalesced loads per lane; three rows (15 loads) in flight per batch
    // (a load-store loop kept one L2 round trip per element in flight)
    constexpr int kRowG = 6 * kGram25, kPerRow = (kRowG + 31) / 32;
#pragma unroll 1
    for (int r0 = 0; r0 < 6; r0 += 3) {
        double tv[3][kPerRow];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const int y = qy + r0 + r;
#pragma unroll
            for (int i = 0; i < kPerRow; ++i) {
                const int j = lane + 32 * i, x = qx + j / kGram25;
                const bool in = j < kRowG && x >= 0 && y >= 0 && x < L.W && y < L.H;
                tv[r][i] = in ? __ldg(gm + ((size_t)y * L.W + qx) * kGram25 + j) : 0.0;
            }
        }
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int i = 0; i < kPerRow; ++i) {
                const int j = lane + 32 * i;
                if (j < kRowG) (&S.u.climb.gr[(r0 + r) * 6][0])[j] = tv[r][i];
            }
    }
    __syncwarp();
    int off[16];
    cubic_gram_offsets(lane & 15, off);
    bool redo;
    double current = cubic_gram(S, off, qx, qy, bx + dx, by + dy, &redo);
    if (redo) current = corr_cubic(L.f, L.W, L.H, C, g4, bx + dx, by + dy);
    double h = 0.5;
    const bool upper = lane >= 16;
#pragma unroll 1
    for (int hs = 0; hs < 6; ++hs, h *= 0.5) {
#pragma unroll 1
        for (int ax = 0; ax < 2; ++ax) {
            const bool along_x = ax == 0;
            // parabola_refine (flow_provider.cpp:152-162): f0 on lanes 0-15, f2 on 16-31; f1 = current
            const double x = bx + dx, y = by + dy;
            const double sx = upper ? x + (along_x ? h : 0) : x - (along_x ? h : 0);
            const double sy = upper ? y + (along_x ? 0 : h) : y - (along_x ? 0 : h);
            const double fv = cubic_gram(S, off, qx, qy, sx, sy, &redo);
            double f0 = __shfl_sync(0xffffffffu, fv, 0), f2 = __shfl_sync(0xffffffffu, fv, 16);
            const unsigned rb = __ballot_sync(0xffffffffu, redo);
            if (rb & 1u) f0 = corr_cubic(L.f, L.W, L.H, C, g4, x - (along_x ? h : 0), y - (along_x ? 0 : h));
            if (rb & 0x10000u) f2 = corr_cubic(L.f, L.W, L.H, C, g4, x + (along_x ? h : 0), y + (along_x ? 0 : h));
            const double f1 = current;
            const double denom = f0 - 2 * f1 + f2;
            // near-flips of parabola_refine's tests (denominator sign / 1e-12 floor, step == 0)
            // (padding-only samples are exact zeros in the reference too: no rounding ties)
            if ((fabs(denom) <= 4 * eps || fabs(fabs(denom) - 1e-12) <= 4 * eps) &&
                !(cubic_pad(x - (along_x ? h : 0), y - (along_x ? 0 : h), L.W, L.H) &&
                  cubic_pad(x + (along_x ? h : 0), y + (along_x ? 0 : h), L.W, L.H) && cubic_pad(x, y, L.W, L.H)))
                *tie |= kTieDenom;
            double step = 0.0;
            if (!(fabs(denom) < 1e-12 || denom > 0)) {
                step = fmin(fmax(0.5 * h * (f0 - f2) / denom, -h), h);
                if (fabs(f0 - f2) <= 2 * eps && !(cubic_pad(x - (along_x ? h : 0), y - (along_x ? 0 : h), L.W, L.H) &&
                                                   cubic_pad(x + (along_x ? h : 0), y + (along_x ? 0 : h), L.W, L.H)))
                    *tie |= kTieStep;
            }
            if (step == 0.0) continue;
            const double nx = dx + (along_x ? step : 0);
            const double ny = dy + (along_x ? 0 : step);
            double value = cubic_gram(S, off, qx, qy, bx + nx, by + ny, &redo);
            if (redo) value = corr_cubic(L.f, L.W, L.H, C, g4, bx + nx, by + ny);
            if (fabs(value - current) <= 2 * eps &&
                !(cubic_pad(bx + nx, by + ny, L.W, L.H) && cubic_pad(bx + dx, by + dy, L.W, L.H))) {
                // the comparison is within the Gram form's rounding margin: evaluate both
                // samples with the reference's exact arithmetic (per-channel samplers,
                // sequential channel sums) at these positions, which differ from the
                // reference's by the ~1e-16 rounding of earlier steps; only a remaining
                // gap below kTieExactRel |g| (a true tie) needs the full exact replay
                resolve_exact(L, C, g4, bx + nx, by + ny, bx + dx, by + dy, S.xs, &value, &current);
                if (fabs(value - current) <= kTieExactRel / kTieRel * eps) *tie |= kTieClimb;
            }
            if (value >= current) {  // hill climb only
                dx = nx;
                dy = ny;
                current = value;
            }
        }
    }
    *px = dx;
    *py = dy;
}

// One (edge, level) measurement task of a warp: the slice, then (level 0) the
// flatness / sharpness scores and, unless flat, the subpixel peak, or (level 1)
// the subpixel peak.  Result record: {px, py, confidence, border | flat << 1 |
// tie << 2 (a decision within the rounding margin: replay exactly)};
// *valid_out / *behind_out: the edge's centre state (identical for both levels).
struct MeasRecord {
    double px, py, conf;
    int bits;  // border | flat << 1 | tie reasons << 2
};
// Two phases around the pair's mid barrier (id `bar_mid`, both warps reach it
// unconditionally): (A) slice, argmax and border flag, and on level 0 the
// flatness / sharpness scores; the pair exchanges {border, flat} through `xchg`
// ([2] ints); (B) the hill climbs — skipped when their results are discarded:
// a flat slice (flow_provider.cpp:236-240 returns before any subpixel peak) or
// both argmaxes on the border (out of range, :266-270), as in the reference's
// outputs (it evaluates and drops the out-of-range climbs).
__device__ __forceinline__ MeasRecord measure_task(const MeasureParams& a, MeasWarpSmem& S, int e, int level,
                                                   bool* valid_out, bool* behind_out, int* xchg, int bar_mid) {
    const int lane = threadIdx.x & 31;
    const int C = a.channels;
    double cx, cy;
    bool behind;
    if (a.centers) {
        cx = a.centers[2 * e];
        cy = a.centers[2 * e + 1];
        behind = a.behind && a.behind[e];
    } else {  // window mode: reproject_patch of the current state (camera.cpp:47-71)
        const int k = a.e_patch[e];
        const SE3 pi = se3_load(a.poses + 7 * a.patch_src[k]);
        const SE3 pj = se3_load(a.poses + 7 * a.e_pose[e]);
        const Cam K{a.K[0], a.K[1], a.K[2], a.K[3]};
        reproject_center(pi, pj, K, a.patch_x + 9 * (size_t)k, a.patch_y + 9 * (size_t)k, a.depth[k], &cx,
                         &cy, &behind);
    }
    const bool valid = !behind && isfinite(cx) && isfinite(cy);
    // this task's record: level 0 {flat, confidence, p0x, p0y, border0}, level 1 {p1x, p1y, border1}
    double r_conf = 0.01, r_px = 0, r_py = 0;
    int r_flat = 1, r_border = 0;
    // phase-A results the climb needs (defined for valid edges)
    Level L{nullptr, 0, 0};
    const double* gm = nullptr;
    G4 g;
    double eps = 0.0, bx = 0.0, by = 0.0;
    int ox = 0, oy = 0, bi = kR * kS + kR, tie = 0;
    unsigned pad = 0;
    bool span = false, border = false;
    if (valid) {
        const int slot = a.e_slot ? a.e_slot[e] : a.pose_slot[a.e_pose[e]];
        L = level ? Level{a.feat1 + (size_t)slot * a.h1 * a.w1 * C, a.w1, a.h1}
                  : Level{a.feat0 + (size_t)slot * a.h0 * a.w0 * C, a.w0, a.h0};
        gm = level ? a.g25_1 + (size_t)slot * a.h1 * a.w1 * kGram25 : a.g25_0 + (size_t)slot * a.h0 * a.w0 * kGram25;
        const float* gp = a.patch_feats + ((size_t)a.e_patch[e] * 2 * 9 + 9 * level + 4) * C;  // centre pixel
        __syncwarp();  // the previous task is done with S
#pragma unroll
        for (int k = 0; k < kCh; ++k) {
            const int c = lane + 32 * k;
            g.v[k] = c < C ? gp[c] : 0.f;
            if (c < C) S.g[c] = g.v[k];
        }
        double gn2 = 0;
#pragma unroll
        for (int k = 0; k < kCh; ++k) gn2 += (double)g.v[k] * g.v[k];
        eps = kTieRel * sqrt(warp_sum(gn2));
        const double sc = level ? kStride * kStride : kStride;
        bx = cx / sc;
        by = cy / sc;
        span = fabs(bx) < 1e8 && fabs(by) < 1e8;  // else every tap is zero padding
        ox = span ? (int)floor(bx) - kR : 0;
        oy = span ? (int)floor(by) - kR : 0;
        __syncwarp();
        if (span) {
            {  // slice window dots: cells lane and lane + 32, interleaved
                const int x0 = ox + (lane & 7), y0 = oy + (lane >> 3), y1 = y0 + 4;
                const bool in0 = x0 >= 0 && y0 >= 0 && x0 < L.W && y0 < L.H;
                const bool in1 = x0 >= 0 && y1 >= 0 && x0 < L.W && y1 < L.H;
                double d0, d1;
                cell_dot2(S.g, L.f + (in0 ? (size_t)y0 * L.W + x0 : 0) * C,
                          L.f + (in1 ? (size_t)y1 * L.W + x0 : 0) * C, C, &d0, &d1);
                S.sd[lane] = in0 ? d0 : 0.0;
                S.sd[lane + 32] = in1 ? d1 : 0.0;
            }
            {  // the slice window's Gram terms, both cells' ten loads in flight together
                constexpr int kG5[5] = {g25_index(0, 0), g25_index(1, 0), g25_index(0, 1), g25_index(1, 1),
                                        g25_index(-1, 1)};
                double tv[2][5];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int q = lane + 32 * h, x = ox + (q & 7), y = oy + (q >> 3);
                    const bool in = x >= 0 && y >= 0 && x < L.W && y < L.H;
                    const double* gc = gm + (in ? (size_t)y * L.W + x : 0) * kGram25;
#pragma unroll
                    for (int m = 0; m < 5; ++m) tv[h][m] = in ? __ldg(gc + kG5[m]) : 0.0;
                }
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int m = 0; m < 5; ++m) S.u.sgr[lane + 32 * h][m] = tv[h][m];
            }
            __syncwarp();
        }
        // the 7x7 slice (correlate_at at base + (beta - 3, alpha - 3)), lane per sample
        unsigned redo = 0;  // pad: padding-only samples (exact zeros, as in the reference)
        for (int n = 0; n < 2; ++n) {
            const int i = lane + 32 * n;
            if (i >= kS * kS) break;
            const int alpha = i / kS, beta = i % kS;
            double val = 0.0;
            if (span) {
                const double x = bx + beta - kR, y = by + alpha - kR;  // flow_provider.cpp:226-227
                const int x0 = (int)floor(x), y0 = (int)floor(y);
                if (x0 + 1 < 0 || x0 >= L.W || y0 + 1 < 0 || y0 >= L.H) pad |= 1u << n;
                const double ax = x - x0, ay = y - y0;
                const int lx = x0 - ox, ly = y0 - oy;
                if (lx >= 0 && lx <= 6 && ly >= 0 && ly <= 6) {
                    const double w0 = (1 - ax) * (1 - ay), w1 = ax * (1 - ay), w2 = (1 - ax) * ay, w3 = ax * ay;
                    const int c0 = ly * 8 + lx;
                    const double* d = S.sd;
                    const double(*G)[5] = S.u.sgr;
                    const double dot = w0 * d[c0] + w1 * d[c0 + 1] + w2 * d[c0 + 8] + w3 * d[c0 + 9];
                    const double diag = w0 * w0 * G[c0][0] + w1 * w1 * G[c0 + 1][0] + w2 * w2 * G[c0 + 8][0] +
                                        w3 * w3 * G[c0 + 9][0];
                    const double cross = w0 * w1 * G[c0][1] + w0 * w2 * G[c0][2] + w0 * w3 * G[c0][3] +
                                         w1 * w2 * G[c0 + 1][4] + w1 * w3 * G[c0 + 1][2] + w2 * w3 * G[c0 + 8][1];
                    const double n2 = diag + 2.0 * cross;
                    if (n2 < 0.5 * diag || (n2 > 0.98e-12 && n2 < 1.02e-12)) redo |= 1u << n;
                    val = n2 > 1e-12 ? dot / sqrt(n2) : 0.0;
                } else {
                    redo |= 1u << n;
                }
            }
            S.v[i] = val;
        }
        __syncwarp();  // the owners' writes of S.v are ordered before lane 0 rewrites flagged samples
        unsigned todo = __ballot_sync(0xffffffffu, redo != 0);
        while (todo) {  // direct evaluation of the flagged samples, a warp each
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            unsigned m = __shfl_sync(0xffffffffu, redo, src);
            while (m) {
                const int n = __ffs(m) - 1;
                m &= m - 1;
                const int i = src + 32 * n, alpha = i / kS, beta = i % kS;
                const double r = corr_bilinear(L.f, L.W, L.H, C, g, bx + beta - kR, by + alpha - kR);
                if (lane == 0) S.v[i] = r;
            }
        }
        __syncwarp();
        // argmax (the reference's first maximum) and border flag; a near-tied argmax
        // matters for level 1 (its peak and border) and, unless flat, for level 0
        int targ = 0;
        bi = slice_argmax(S.v, eps, &targ, &pad);
        const int best_a = bi / kS, best_b = bi % kS;
        border = best_a == 0 || best_a == kS - 1 || best_b == 0 || best_b == kS - 1;
        if (level == 1) {
            r_flat = 0;
            tie = targ;
        } else {
            // level 0: flatness / sharpness scores on the slice (flow_provider.cpp:217-250),
            // as warp reductions (the mean as a fixed-order tree)
            const double peak = S.v[bi];
            double minimum = CUDART_INF, mean = 0, second = -CUDART_INF;
            for (int i = lane; i < kS * kS; i += 32) {
                const double val = S.v[i];
                mean += val;
                minimum = fmin(minimum, val);
                if (max(abs(i / kS - best_a), abs(i % kS - best_b)) > 1) second = fmax(second, val);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                mean += __shfl_xor_sync(0xffffffffu, mean, o);
                minimum = fmin(minimum, __shfl_xor_sync(0xffffffffu, minimum, o));
                second = fmax(second, __shfl_xor_sync(0xffffffffu, second, o));
            }
            mean /= kS * kS;
            const double peak_to_mean = (peak - minimum) / (mean - minimum + 1e-9);
            r_flat = !(peak_to_mean >= 1.05);
            // the flatness threshold within the propagated rounding margin of peak, min, mean
            if (fabs(peak_to_mean - 1.05) <= 8 * eps * (1 + fabs(peak_to_mean)) / (mean - minimum + 1e-9))
                tie |= kTieFlat;
            if (!r_flat) {
                tie |= targ;
                const double score = 2.0 * (peak - 0.75) + (peak - second - 0.08);
                r_conf = fmin(fmax(1.0 / (1.0 + exp(-12.0 * score)), 0.01), 0.99);
            }
        }
    }
    // ---- the pair exchanges {border, flat}; the climbs run only where they are used ----
    if (lane == 0) xchg[level] = valid ? (int)border | (level == 0 ? r_flat << 1 : 0) : 3;
    __syncwarp();
    asm volatile("bar.sync %0, 64;" ::"r"(bar_mid) : "memory");
    const int x0 = xchg[0], x1 = xchg[1];
    const bool climb = valid && span && !((x0 >> 1) & 1) && !((x0 & 1) && (x1 & 1));
    if (climb) subpixel_peak_gram(S, L, C, gm, g, bx, by, ox, oy, bi, &r_px, &r_py, eps, &tie);
    else if (valid) {  // no climb: the discrete peak (the reference's starting point)
        r_px = bi % kS - kR;
        r_py = bi / kS - kR;
    }
    if (valid) r_border = border | (span ? tie << 2 : 0);
    *valid_out = valid;
    *behind_out = behind;
    return MeasRecord{r_px, r_py, r_conf, r_border | (r_flat << 1)};
}

// The measurement of an edge from its two level records (flow_provider.cpp:252-287).
__device__ __forceinline__ void measure_combine(const MeasureParams& a, int e, bool valid, bool behind,
                                                const MeasRecord& r0, const MeasRecord& r1) {
    const double p0x = r0.px, p0y = r0.py, p1x = r1.px, p1y = r1.py;
    double confidence = r0.conf;
    const int b0 = r0.bits, b1 = r1.bits;
    const bool flat = (b0 >> 1) & 1, border0 = b0 & 1, border1 = b1 & 1;
    // near-tie decisions: level 0's always count, level 1's only when its peak is used
    int tie = valid ? (b0 >> 2) | (flat ? 0 : b1 >> 2) : 0;
    double dxo = 0, dyo = 0, wgt = 0.01;
    int flags = 0;
    if (behind) {
        flags = 4;  // flow_provider.cpp:301-302
    } else if (!valid) {
        flags = 8;
        atomicOr(a.status, 1 << kDevBadCoords);
    } else if (flat) {
        flags = 1;  // flat: delta 0, weight 0.01
    } else {
        const double e0x = kStride * p0x, e0y = kStride * p0y;
        const double e1x = kStride * kStride * p1x, e1y = kStride * kStride * p1y;
        if (border0 && border1) {
            flags = 2;  // out of range: delta 0, weight 0.01
        } else {
            if (border0) {
                dxo = e1x;
                dyo = e1y;
                confidence = fmin(confidence, 0.25);
            } else {
                dxo = e0x;
                dyo = e0y;
                const double ddx = e1x - e0x, ddy = e1y - e0y;
                const double dist = sqrt(ddx * ddx + ddy * ddy);
                if (!border1 && dist > 2.0 * kStride * kStride) confidence = fmin(confidence, 0.25);
                if (!border1 && fabs(dist - 2.0 * kStride * kStride) <= 1e-9) tie |= kTieDist;
            }
            wgt = confidence;
        }
    }
    if (tie) a.replay[1 + atomicAdd(a.replay, 1)] = e;  // measure_exact_kernel rewrites this edge
#ifdef PVO_MEASURE_TIE_STATS  // debug variant (tools/measure_ties.py): flags = 128 | reasons, no replay
    if (tie) flags = 128 | tie;
#endif
    a.delta[2 * e] = dxo;
    a.delta[2 * e + 1] = dyo;
    a.weight[2 * e] = wgt;
    a.weight[2 * e + 1] = wgt;
    if (a.flags) a.flags[e] = (uint8_t)flags;
}

// Paired warps (default): a block runs kMeasWarps / 2 edges, warp 2m level 0 and
// warp 2m + 1 level 1 of edge m; they meet on a named barrier.
#ifndef PVO_MEASURE_GRAM_MINB
#define PVO_MEASURE_GRAM_MINB 2
#endif
// A block runs kMeasWarps / 2 edges: warp 2m level 0 and warp 2m + 1 level 1 of edge
// m, meeting on a named barrier.  (A persistent grid of warp pairs taking edges from a
// queue ran 15 % slower: profiles/r2/measure_ab.txt.)
__global__ void __launch_bounds__(32 * kMeasWarps, PVO_MEASURE_GRAM_MINB) measure_gram_kernel(MeasureParams a) {
    extern __shared__ __align__(16) unsigned char s_meas[];
    __shared__ MeasRecord s_rec1[kMeasWarps / 2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pair = warp >> 1, level = warp & 1;
    const int e = blockIdx.x * (kMeasWarps / 2) + pair;
    if (e >= a.n_edges) return;  // both warps of the pair
    MeasWarpSmem& S = reinterpret_cast<MeasWarpSmem*>(s_meas)[warp];
    __shared__ int s_x[kMeasWarps / 2][2];
    bool valid, behind;
    const MeasRecord r = measure_task(a, S, e, level, &valid, &behind, s_x[pair], 1 + kMeasWarps / 2 + pair);
    if (level == 1 && lane == 0) s_rec1[pair] = r;
    __syncwarp();
    asm volatile("bar.sync %0, 64;" ::"r"(1 + pair) : "memory");
    if (level == 0 && lane == 0) measure_combine(a, e, valid, behind, r, s_rec1[pair]);
}

// ---- OracleFlowProvider::propose (flow_provider.cpp:34-93), simulator revisions ----
// pass 0: ground-truth reprojection of each edge's patch centre (a 1x1 probe at
// the centre with the scene inverse depth, between the scene poses) and the
// current-state centre; behind flag of either.  pass 1: noise, clamp, weights.
__global__ void oracle_propose_kernel(OracleParams a, int pass) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= a.n_edges) return;
    if (pass == 0) {
        const int k = a.e_patch[e], i = a.patch_src[k], j = a.e_pose[e];
        const Cam K{a.K[0], a.K[1], a.K[2], a.K[3]};
        const double cxp = a.patch_x[9 * (size_t)k + 4], cyp = a.patch_y[9 * (size_t)k + 4];
        const SE3 gi = se3_load(a.gt_poses + 7 * i), gj = se3_load(a.gt_poses + 7 * j);
        double gu, gv;
        bool gb;
        reproject_center_probe(gi, gj, K, cxp, cyp, a.gt_depth[k], &gu, &gv, &gb);
        double cu, cv;
        bool cb;
        reproject_center(se3_load(a.poses + 7 * i), se3_load(a.poses + 7 * j), K, a.patch_x + 9 * (size_t)k,
                         a.patch_y + 9 * (size_t)k, a.depth[k], &cu, &cv, &cb);
        a.behind[e] = gb || cb;
        a.delta[2 * e] = gu - cu;
        a.delta[2 * e + 1] = gv - cv;
        return;
    }
    double dx = 0, dy = 0, w = 0.01;
    if (!a.behind[e]) {
        dx = a.delta[2 * e];
        dy = a.delta[2 * e + 1];
        if (a.flow_sigma > 0) {
            dx += a.noise[2 * e];
            dy += a.noise[2 * e + 1];
        }
        const bool in_range = fabs(dx) <= 64.0 && fabs(dy) <= 64.0;  // kMaxRevisionPx (flow_provider.hpp:47)
        dx = fmin(fmax(dx, -64.0), 64.0);
        dy = fmin(fmax(dy, -64.0), 64.0);
        w = in_range ? a.weight_in_range : 0.01;
    }
    if (a.outlier && a.outlier[e]) {
        dx = a.outlier_delta[2 * e];
        dy = a.outlier_delta[2 * e + 1];
        w = 0.01;
    }
    a.delta[2 * e] = dx;
    a.delta[2 * e + 1] = dy;
    a.weight[2 * e] = w;
    a.weight[2 * e + 1] = w;
}


// ---- correlate_at / correlate_at_cubic at free points (correlation.cpp:8-35) ----
// One warp per query point, lanes over channels c = lane, lane + 32, ... (any C);
// each channel's sample is the reference's per-channel expression
// (features.cpp:9-52; this file is compiled with --fmad=false), the channel
// sums a fixed warp tree.  Non-finite or out-of-int-range positions sample only
// padding (the reference's int conversion of such a floor lands outside the
// grid): the result is 0.
__global__ void points_kernel(PointsParams a) {
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= a.n) return;
    const double x = a.xy[2 * (size_t)i], y = a.xy[2 * (size_t)i + 1];
    const float* g = a.features + (size_t)i * a.channels;
    double dot = 0, nrm = 0;
    const bool ok = fabs(x) < 1e9 && fabs(y) < 1e9;  // false for NaN / inf too
    if (ok) {
        const int x0 = (int)floor(x), y0 = (int)floor(y);
        if (!a.cubic) {
            const double ax = x - x0, ay = y - y0;
            for (int c = lane; c < a.channels; c += 32) {
                double v[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int xi = x0 + (t & 1), yi = y0 + (t >> 1);
                    v[t] = (xi < 0 || yi < 0 || xi >= a.W || yi >= a.H)
                               ? 0.0
                               : (double)a.grid[((size_t)yi * a.W + xi) * a.channels + c];
                }
                const double s = (1 - ax) * (1 - ay) * v[0] + ax * (1 - ay) * v[1] + (1 - ax) * ay * v[2] +
                                 ax * ay * v[3];
                dot += g[c] * s;
                nrm += s * s;
            }
        } else {
            double wx[4], wy[4];
            cubic_weights(x - x0, wx);
            cubic_weights(y - y0, wy);
            for (int c = lane; c < a.channels; c += 32) {
                double s = 0;
                for (int j = 0; j < 4; ++j) {
                    const int yi = y0 - 1 + j;
                    if (yi < 0 || yi >= a.H) continue;
                    double row = 0;
                    for (int k = 0; k < 4; ++k) {
                        const int xi = x0 - 1 + k;
                        if (xi < 0 || xi >= a.W) continue;
                        row += wx[k] * (double)a.grid[((size_t)yi * a.W + xi) * a.channels + c];
                    }
                    s += wy[j] * row;
                }
                dot += g[c] * s;
                nrm += s * s;
            }
        }
    }
    const double r = finish(dot, nrm);
    if (lane == 0) a.out[i] = r;
}
}  // namespace

cudaError_t launch_oracle_propose(const OracleParams& p, int pass, cudaStream_t stream) {
    if (p.n_edges <= 0) return cudaSuccess;
    oracle_propose_kernel<<<(p.n_edges + 127) / 128, 128, 0, stream>>>(p, pass);
    return cudaGetLastError();
}

cudaError_t launch_points(const PointsParams& p, cudaStream_t stream) {
    if (p.n <= 0) return cudaSuccess;
    points_kernel<<<(p.n + 7) / 8, 256, 0, stream>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_measure(const MeasureParams& p, cudaStream_t stream) {
    if (p.n_edges <= 0) return cudaSuccess;
    if (p.channels > 32 * kCh) return cudaErrorNotSupported;
    if (p.g25_0 && p.g25_1) {
        cudaError_t err =
            cudaFuncSetAttribute(measure_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMeasSmem);
        if (err != cudaSuccess) return err;
        if (!p.replay || !p.replay_done) return cudaErrorInvalidValue;
        measure_gram_kernel<<<(p.n_edges + kMeasWarps / 2 - 1) / (kMeasWarps / 2), 32 * kMeasWarps, kMeasSmem,
                              stream>>>(p);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
#ifndef PVO_MEASURE_TIE_STATS
        err = cudaFuncSetAttribute(measure_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kExactSmem);
        if (err != cudaSuccess) return err;
        measure_exact_kernel<<<kExactBlocks, 64, kExactSmem, stream>>>(p);
#endif
        return cudaGetLastError();
    }
    measure_kernel<<<(p.n_edges + 3) / 4, 256, 0, stream>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_gram25(const float* feat, int W, int H, int C, double* g25, cudaStream_t stream) {
    if (W <= 0 || H <= 0) return cudaSuccess;
    const int smem = kG25SW * kG25SH * (C + 1) * (int)sizeof(float);
    cudaError_t err = cudaFuncSetAttribute(gram25_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    const dim3 grid((W + kG25TileW - 1) / kG25TileW, (H + kG25TileH - 1) / kG25TileH);
    gram25_kernel<<<grid, 256, smem, stream>>>(feat, W, H, C, g25);
    return cudaGetLastError();
}

}  // namespace pvo_dev
