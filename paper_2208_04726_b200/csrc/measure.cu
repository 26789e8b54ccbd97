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

#include <cfloat>
#include <cstdint>

#include "ba_common.cuh"
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

// correlate_at (correlation.cpp:8-23) with sample_zero_padded (features.cpp:9-21).
// Not inlined: one copy of the sampler keeps the kernel inside the instruction cache.
__device__ __noinline__ double corr_bilinear(const float* f, int W, int H, int C, G4 g, double x, double y) {
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

// correlate_at_cubic (correlation.cpp:25-35) with sample_cubic (features.cpp:23-52):
// taps outer (one address per tap, four channel loads at immediate offsets),
// the per-channel operation order unchanged.
__device__ __noinline__ double corr_cubic(const float* f, int W, int H, int C, G4 g, double x, double y) {
    const int lane = threadIdx.x & 31;
    const int x0 = (int)floor(x), y0 = (int)floor(y);
    double wx[4], wy[4];
    cubic_weights(x - x0, wx);
    cubic_weights(y - y0, wy);
    double v[kCh] = {0, 0, 0, 0};
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
    double dot = 0, nrm = 0;
#pragma unroll
    for (int k = 0; k < kCh; ++k) {
        dot += (double)g.v[k] * v[k];
        nrm += v[k] * v[k];
    }
    return finish(dot, nrm);
}

// subpixel_peak (flow_provider.cpp:167-205) from the 7x7 slice `vals` (already
// evaluated at base + (beta - 3, alpha - 3)); returns the offset in cells
__device__ void subpixel_peak(const Level& L, int C, G4 g, double bx, double by,
                              const double* vals, double* ox, double* oy, bool* on_border) {
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
    double current = corr_cubic(L.f, L.W, L.H, C, g, bx + dx, by + dy);
    double h = 0.5;
    for (int hs = 0; hs < 6; ++hs, h *= 0.5) {
        for (int ax = 0; ax < 2; ++ax) {
            const bool along_x = ax == 0;
            // parabola_refine (flow_provider.cpp:152-162); f1 = the current value
            const double x = bx + dx, y = by + dy;
            const double f0 = corr_cubic(L.f, L.W, L.H, C, g, x - (along_x ? h : 0), y - (along_x ? 0 : h));
            const double f1 = current;
            const double f2 = corr_cubic(L.f, L.W, L.H, C, g, x + (along_x ? h : 0), y + (along_x ? 0 : h));
            const double denom = f0 - 2 * f1 + f2;
            double step = 0.0;
            if (!(fabs(denom) < 1e-12 || denom > 0)) step = fmin(fmax(0.5 * h * (f0 - f2) / denom, -h), h);
            if (step == 0.0) continue;
            const double nx = dx + (along_x ? step : 0);
            const double ny = dy + (along_x ? 0 : step);
            const double value = corr_cubic(L.f, L.W, L.H, C, g, bx + nx, by + ny);
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

#ifndef PVO_MEASURE_MINB
#define PVO_MEASURE_MINB 1
#endif
__global__ void __launch_bounds__(256, PVO_MEASURE_MINB) measure_kernel(MeasureParams a) {
    // two warps per edge: warp 2m runs level 0 (slice, scores, subpixel peak), warp
    // 2m+1 level 1 (slice, subpixel peak) concurrently; they meet on a named barrier
    __shared__ double s_vals[8][kS * kS];
    __shared__ double s_peak1[4][2];
    __shared__ int s_border1[4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pair = warp >> 1, level = warp & 1;
    const int e = blockIdx.x * 4 + pair;
    if (e >= a.n_edges) return;  // both warps of the pair
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
        double* v = s_vals[warp];
        const double sc = level ? kStride * kStride : kStride;
        const double bx = cx / sc, by = cy / sc;
        for (int i = 0; i < kS * kS; ++i) {
            const int alpha = i / kS, beta = i % kS;
            const double va = corr_bilinear(L.f, L.W, L.H, a.channels, g, bx + beta - kR, by + alpha - kR);
            if (lane == 0) v[i] = va;
        }
        __syncwarp();
        if (level == 1) {
            // level-1 subpixel peak (flow_provider.cpp:264-265), needed unless level 0 is flat
            double px, py;
            bool border;
            subpixel_peak(L, a.channels, g, bx, by, v, &px, &py, &border);
            if (lane == 0) {
                s_peak1[pair][0] = px;
                s_peak1[pair][1] = py;
                s_border1[pair] = border;
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
                subpixel_peak(L, a.channels, g, bx, by, v, &p0x, &p0y, &border0);
            }
        }
    }
    // the pair meets on its named barrier at one program point, unconditionally (also
    // for behind / non-finite edges), each warp converged: bar.sync counts threads
    __syncwarp();
    asm volatile("bar.sync %0, 64;" ::"r"(1 + pair) : "memory");
    if (valid && level == 0) {
        if (flat) {
            flags = 1;  // flat: delta 0, weight 0.01
        } else {
            const bool border1 = s_border1[pair];
            const double p1x = s_peak1[pair][0], p1y = s_peak1[pair][1];
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
                    if (!border1 && sqrt(ddx * ddx + ddy * ddy) > 2.0 * kStride * kStride)
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
    measure_kernel<<<(p.n_edges + 3) / 4, 256, 0, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace pvo_dev
