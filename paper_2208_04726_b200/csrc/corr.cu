// corr.cu — normalised patch-to-frame correlation (K2) and per-frame Gram
// terms, sm_100a.
//
// Reference semantics (correlation.cpp:8-71, features.cpp:9-21): for each
// edge, level l in {0,1}, patch pixel (u,v) and offset (alpha,beta) in 7x7,
//     C = <g, f(x)> / ||f(x)||   (0 when ||f(x)||^2 <= 1e-12)
// where f(x) is the zero-padded bilinear sample of the target frame's level-l
// grid at x = reproj/(4 or 16) + (beta-3, alpha-3), and g the patch pixel's
// level-l descriptor.
//
// B200 formulation.  Offsets are whole cells, so every bilinear tap of a
// patch pixel lands on the integer cells of an 8x8 window, and the 9 pixels
// of a patch share one union tile (<= 10x10 cells).  Per (edge, level) the
// CTA therefore
//   1. stages the union tile (cells x D fp32) in shared memory with 128-bit
//      coalesced loads (a tile row is contiguous in the HWC layout),
//   2. computes the 9 x tile dot products <g_p, f_cell> once (register-
//      blocked: each lane owns up to 4 cells x 9 pixels, each warp a quarter
//      of the channel chunks; fixed-order cross-warp sum),
//   3. forms every output from 4 dots and the per-frame Gram terms
//      (||f||^2, <f,f_right>, <f,f_down>, <f,f_diag>, <f_right,f_down>) in
//      FP64: dot = sum w_t d_t, ||f(x)||^2 = sum_t sum_t' w_t w_t' <f_t,f_t'>.
// This is the reference's arithmetic regrouped by linearity: 9*T*D MACs per
// edge-level instead of 9*49*4*D.  Out-of-bounds cells are zero in the tile
// and zero in the Gram maps, which reproduces the zero padding exactly.
#include <cuda_runtime.h>

#include <cstdint>

#include "corr_exact.cuh"
#include "geometry.cuh"
#include "kernels.cuh"

namespace pvo_dev {

namespace {

constexpr int kThreads = 128;
constexpr int kMaxCells = 100;  // union tile capacity: 10 x 10 cells
constexpr int kPix = 9;         // 3x3 patch

struct SmemLayout {
    int tile, g, gram, part, total_bytes;
};

__host__ __device__ inline int padded_stride(int D) {
    int dp = (D + 3) & ~3;
    if ((dp & 7) == 0) dp += 4;  // odd multiple of 4 floats: conflict-free 128-bit lanes-over-cells
    return dp;
}

__host__ __device__ inline SmemLayout corr_layout(int D) {
    const int dp = padded_stride(D);
    SmemLayout L;
    L.tile = 0;
    L.g = L.tile + kMaxCells * dp;
    L.gram = L.g + kPix * dp;
    L.part = L.gram + kMaxCells * 5;
    const int floats = L.part + 4 * kPix * kMaxCells;
    L.total_bytes = floats * 4;
    return L;
}

// Reprojected coordinates of the 9 patch pixels of edge e (reproject_patch,
// camera.cpp:47-71, including the bitwise-equal-pose shortcut).
__device__ inline void edge_coords(const CorrParams& a, int e, int pix, double* xy) {
    const int k = a.e_patch[e];
    if (a.coords) {
        xy[0] = a.coords[(size_t)e * 18 + 2 * pix];
        xy[1] = a.coords[(size_t)e * 18 + 2 * pix + 1];
        return;
    }
    const int src = a.patch_src[k];
    const int tgt = a.e_pose[e];
    const SE3 pi = se3_load(a.poses + 7 * src);
    const SE3 pj = se3_load(a.poses + 7 * tgt);
    const double px = a.patch_x[(size_t)k * 9 + pix];
    const double py = a.patch_y[(size_t)k * 9 + pix];
    if (se3_equal(pi, pj)) {
        xy[0] = px;
        xy[1] = py;
        return;
    }
    const Relative rel = relative_pose(pi, pj);
    const Cam K{a.K[0], a.K[1], a.K[2], a.K[3]};
    reproject_point(rel, K, a.depth[k], px, py, &xy[0], &xy[1]);
}

__global__ void __launch_bounds__(kThreads) corr_kernel(CorrParams a) {
    extern __shared__ __align__(16) float smem[];
    __shared__ double s_bx[kPix], s_by[kPix];
    __shared__ int s_fx[kPix], s_fy[kPix];
    __shared__ double s_xy[2 * kPix];
    __shared__ int s_bad;

    // one edge (both levels) per CTA
    for (int item = blockIdx.x; item < a.n_edges; item += gridDim.x) {
    const int e = item;
    const int lv_begin = 0, lv_end = 2;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int D = a.channels;
    const int dp = padded_stride(D);
    const int nch4 = dp >> 2;
    const SmemLayout L = corr_layout(D);
    float* s_tile = smem + L.tile;
    float* s_g = smem + L.g;
    float* s_gram = smem + L.gram;
    float* s_part = smem + L.part;

    if (tid == 0) s_bad = 0;
    __syncthreads();
    if (tid < kPix) {
        double xy[2];
        edge_coords(a, e, tid, xy);
        s_xy[2 * tid] = xy[0];
        s_xy[2 * tid + 1] = xy[1];
        if (!isfinite(xy[0]) || !isfinite(xy[1])) s_bad = 1;
    }
    __syncthreads();
    if (s_bad) {
        if (tid == 0) atomicOr(a.status, 1 << kDevBadCoords);  // correlation.cpp:43-45
        __syncthreads();
        continue;
    }

    const int k = a.e_patch[e];
    const int slot = a.e_slot ? a.e_slot[e] : a.pose_slot[a.e_pose[e]];

    for (int level = lv_begin; level < lv_end; ++level) {
        const int W = level ? a.w1 : a.w0;
        const int H = level ? a.h1 : a.h0;
        const float* fbase = (level ? a.feat1 : a.feat0) + (size_t)slot * W * H * D;
        const int Wg = gram_stride(W);
        const float* gbase = (level ? a.gram1 : a.gram0) + (size_t)slot * Wg * H * 8;
        const float* pfeat = a.patch_feats + ((size_t)k * 2 + level) * kPix * D;
        const double scale = level ? 16.0 : 4.0;  // kFeatureStride (features.hpp:46)

        if (tid < kPix) {
            const double bx = s_xy[2 * tid] / scale;
            const double by = s_xy[2 * tid + 1] / scale;
            s_bx[tid] = bx;
            s_by[tid] = by;
            // Clamp far-away pixels: every tap is out of bounds there anyway.
            const double lo = -16.0;
            s_fx[tid] = (int)floor(fmin(fmax(bx, lo), (double)W + 16.0));
            s_fy[tid] = (int)floor(fmin(fmax(by, lo), (double)H + 16.0));
        }
        __syncthreads();

        int xmin = s_fx[0], xmax = s_fx[0], ymin = s_fy[0], ymax = s_fy[0];
#pragma unroll
        for (int p = 1; p < kPix; ++p) {
            xmin = min(xmin, s_fx[p]);
            xmax = max(xmax, s_fx[p]);
            ymin = min(ymin, s_fy[p]);
            ymax = max(ymax, s_fy[p]);
        }
        const bool unified = (xmax - xmin + 8) * (ymax - ymin + 8) <= kMaxCells;
        const int ngroups = unified ? 1 : kPix;

        for (int grp = 0; grp < ngroups; ++grp) {
            const int p0 = unified ? 0 : grp;
            const int npx = unified ? kPix : 1;
            const int X0 = (unified ? xmin : s_fx[p0]) - 3;
            const int Y0 = (unified ? ymin : s_fy[p0]) - 3;
            const int TW = (unified ? xmax - xmin : 0) + 8;
            const int TH = (unified ? ymax - ymin : 0) + 8;
            const int NC = TW * TH;

            // ---- 1. stage tile, Gram terms and descriptors ----
            if ((D & 3) == 0) {
                const int D4 = D >> 2;
                const int total = NC * D4;
                for (int i = tid; i < total; i += kThreads) {
                    const int cell = i / D4;
                    const int c4 = i - cell * D4;
                    const int cy = Y0 + cell / TW;
                    const int cx = X0 + cell % TW;
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (cx >= 0 && cy >= 0 && cx < W && cy < H) {
                        v = __ldg(reinterpret_cast<const float4*>(fbase + ((size_t)cy * W + cx) * D) + c4);
                    }
                    *reinterpret_cast<float4*>(s_tile + cell * dp + 4 * c4) = v;
                }
            } else {
                const int total = NC * D;
                for (int i = tid; i < total; i += kThreads) {
                    const int cell = i / D;
                    const int c = i - cell * D;
                    const int cy = Y0 + cell / TW;
                    const int cx = X0 + cell % TW;
                    float v = 0.f;
                    if (cx >= 0 && cy >= 0 && cx < W && cy < H) v = __ldg(fbase + ((size_t)cy * W + cx) * D + c);
                    s_tile[cell * dp + c] = v;
                }
            }
            if (dp > D) {
                const int padw = dp - D;
                for (int i = tid; i < NC * padw; i += kThreads) {
                    s_tile[(i / padw) * dp + D + (i % padw)] = 0.f;
                }
            }
            for (int i = tid; i < NC * 5; i += kThreads) {
                const int cell = i / 5, t = i - 5 * (i / 5);
                const int cy = Y0 + cell / TW;
                const int cx = X0 + cell % TW;
                float v = 0.f;
                if (cx >= 0 && cy >= 0 && cx < W && cy < H) v = __ldg(gbase + (size_t)t * Wg * H + (size_t)cy * Wg + cx);
                s_gram[i] = v;
            }
            for (int i = tid; i < npx * dp; i += kThreads) {
                const int pi = i / dp, c = i - pi * dp;
                s_g[i] = c < D ? __ldg(pfeat + (size_t)(p0 + pi) * D + c) : 0.f;
            }
            __syncthreads();

            // ---- 2. dot products <g_p, f_cell> ----
            float acc[4][kPix];
#pragma unroll
            for (int ci = 0; ci < 4; ++ci)
#pragma unroll
                for (int p = 0; p < kPix; ++p) acc[ci][p] = 0.f;

            for (int ch = warp; ch < nch4; ch += 4) {
                float4 gv[kPix];
#pragma unroll
                for (int p = 0; p < kPix; ++p) gv[p] = *reinterpret_cast<const float4*>(s_g + p * dp + 4 * ch);
#pragma unroll
                for (int ci = 0; ci < 4; ++ci) {
                    const int cell = lane + 32 * ci;
                    if (cell < NC) {
                        const float4 t = *reinterpret_cast<const float4*>(s_tile + cell * dp + 4 * ch);
#pragma unroll
                        for (int p = 0; p < kPix; ++p) {
                            float s = acc[ci][p];
                            s = fmaf(t.x, gv[p].x, s);
                            s = fmaf(t.y, gv[p].y, s);
                            s = fmaf(t.z, gv[p].z, s);
                            s = fmaf(t.w, gv[p].w, s);
                            acc[ci][p] = s;
                        }
                    }
                }
            }
#pragma unroll
            for (int ci = 0; ci < 4; ++ci) {
                const int cell = lane + 32 * ci;
                if (cell < NC) {
#pragma unroll
                    for (int p = 0; p < kPix; ++p) s_part[(warp * kPix + p) * kMaxCells + cell] = acc[ci][p];
                }
            }
            __syncthreads();
            for (int i = tid; i < npx * NC; i += kThreads) {
                const int p = i / NC, cell = i - p * NC;
                float s = s_part[(0 * kPix + p) * kMaxCells + cell];
                s += s_part[(1 * kPix + p) * kMaxCells + cell];
                s += s_part[(2 * kPix + p) * kMaxCells + cell];
                s += s_part[(3 * kPix + p) * kMaxCells + cell];
                s_part[p * kMaxCells + cell] = s;
            }
            __syncthreads();

            // ---- 3. bilinear recombination + normalisation (FP64) ----
            float* out = a.out + ((size_t)e * 2 + level) * kPix * 49;
            for (int o = tid; o < npx * 49; o += kThreads) {
                const int pi = o / 49;
                const int ab = o - pi * 49;
                const int alpha = ab / 7, beta = ab - 7 * (ab / 7);
                const int p = p0 + pi;
                // x = base + (beta - 3): same double expression as the reference;
                // x0e = floor(base) + beta - 3 <= x <= x0e + 1, so ax is exact
                // and the taps equal the reference's (features.cpp:10-13).
                const double xs = s_bx[p] + (double)(beta - 3);
                const double ys = s_by[p] + (double)(alpha - 3);
                const int x0 = s_fx[p] + beta - 3;
                const int y0 = s_fy[p] + alpha - 3;
                const double ax = xs - (double)x0;
                const double ay = ys - (double)y0;
                const int c00 = (y0 - Y0) * TW + (x0 - X0);
                const float* dots = s_part + pi * kMaxCells;
                const double d00 = dots[c00], d10 = dots[c00 + 1];
                const double d01 = dots[c00 + TW], d11 = dots[c00 + TW + 1];
                const double w00 = (1 - ax) * (1 - ay), w10 = ax * (1 - ay);
                const double w01 = (1 - ax) * ay, w11 = ax * ay;
                const double dot = w00 * d00 + w10 * d10 + w01 * d01 + w11 * d11;
                const float* g00 = s_gram + 5 * c00;
                const float* g10 = s_gram + 5 * (c00 + 1);
                const float* g01 = s_gram + 5 * (c00 + TW);
                const float* g11 = s_gram + 5 * (c00 + TW + 1);
                // Gram record: [0]=|f|^2 [1]=<f,f_right> [2]=<f,f_down> [3]=<f,f_diag> [4]=<f_right,f_down>
                const double diag = w00 * w00 * (double)g00[0] + w10 * w10 * (double)g10[0] +
                                    w01 * w01 * (double)g01[0] + w11 * w11 * (double)g11[0];
                double n2 = diag;
                n2 += 2.0 * (w00 * w10 * (double)g00[1] + w01 * w11 * (double)g01[1] + w00 * w01 * (double)g00[2] +
                             w10 * w11 * (double)g10[2] + w00 * w11 * (double)g00[3] + w10 * w01 * (double)g00[4]);
                float c;
                if (corr_needs_exact((float)n2, (float)diag))  // cancelling taps: the reference's way
                    c = corr_exact_thread(pfeat + (size_t)p * D, fbase, W, H, D, xs, ys);
                else
                    c = n2 > 1e-12 ? (float)(dot / sqrt(n2)) : 0.f;  // correlation.cpp:22
                out[(size_t)p * 49 + ab] = c;
            }
            __syncthreads();
        }
    }
    }  // item loop
}

// Gram terms of both pyramid levels of one frame in one launch (cells of level
// 0, then of level 1).  One warp per cell.
struct GramLevel {
    const float* feat;
    float* gram;
    int W, H;
};
__global__ void gram_kernel(GramLevel l0, GramLevel l1, int D) {
    const int warps_per_block = blockDim.x >> 5;
    const int lane = threadIdx.x & 31;
    const int n0 = l0.W * l0.H, ncell = n0 + l1.W * l1.H;
    for (int all = blockIdx.x * warps_per_block + (threadIdx.x >> 5); all < ncell;
         all += gridDim.x * warps_per_block) {
        const bool lv1 = all >= n0;
        const GramLevel& L = lv1 ? l1 : l0;
        const int cell = lv1 ? all - n0 : all;
        const int W = L.W, H = L.H, Wp = gram_stride(W);
        const float* feat = L.feat;
        float* gram = L.gram;
        const int y = cell / W, x = cell - (cell / W) * W;
        const float* f = feat + (size_t)cell * D;
        const bool hr = x + 1 < W, hd = y + 1 < H;
        const float* fr = hr ? f + D : nullptr;
        const float* fd = hd ? f + (size_t)W * D : nullptr;
        const float* fdr = (hr && hd) ? f + (size_t)(W + 1) * D : nullptr;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f, s4 = 0.f;
        if (D == 128) {  // one 16-byte load per lane and neighbour, all in flight together
            const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 v = reinterpret_cast<const float4*>(f)[lane];
            const float4 r = hr ? reinterpret_cast<const float4*>(fr)[lane] : zero;
            const float4 d = hd ? reinterpret_cast<const float4*>(fd)[lane] : zero;
            const float4 dr = (hr && hd) ? reinterpret_cast<const float4*>(fdr)[lane] : zero;
            s0 = fmaf(v.w, v.w, fmaf(v.z, v.z, fmaf(v.y, v.y, v.x * v.x)));
            s1 = fmaf(v.w, r.w, fmaf(v.z, r.z, fmaf(v.y, r.y, v.x * r.x)));
            s2 = fmaf(v.w, d.w, fmaf(v.z, d.z, fmaf(v.y, d.y, v.x * d.x)));
            s3 = fmaf(v.w, dr.w, fmaf(v.z, dr.z, fmaf(v.y, dr.y, v.x * dr.x)));
            s4 = fmaf(r.w, d.w, fmaf(r.z, d.z, fmaf(r.y, d.y, r.x * d.x)));
        } else
        for (int c = lane; c < D; c += 32) {
            const float v = f[c];
            const float r = hr ? fr[c] : 0.f;
            const float d = hd ? fd[c] : 0.f;
            const float dr = (hr && hd) ? fdr[c] : 0.f;
            s0 = fmaf(v, v, s0);
            s1 = fmaf(v, r, s1);
            s2 = fmaf(v, d, s2);
            s3 = fmaf(v, dr, s3);
            s4 = fmaf(r, d, s4);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, off);
            s1 += __shfl_xor_sync(0xffffffffu, s1, off);
            s2 += __shfl_xor_sync(0xffffffffu, s2, off);
            s3 += __shfl_xor_sync(0xffffffffu, s3, off);
            s4 += __shfl_xor_sync(0xffffffffu, s4, off);
        }
        if (lane == 0) {  // planar records: plane k at gram + k * H * Wp (8 planes reserved, 5 used)
            const size_t plane = (size_t)H * Wp;
            float* g = gram + (size_t)y * Wp + x;
            g[0 * plane] = s0;
            g[1 * plane] = s1;
            g[2 * plane] = s2;
            g[3 * plane] = s3;
            g[4 * plane] = s4;
        }
    }
}

// correlate() for one patch of any width (correlation.cpp:37-71): block (pixel,
// level), a warp per output over the 49 offsets, evaluated directly.
__global__ void corr_direct_kernel(int pp, int C, const float* feats, const double* coords, const float* f0, int w0,
                                   int h0, const float* f1, int w1, int h1, float* out) {
    const int pix = blockIdx.x, level = blockIdx.y;
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const float* g = feats + ((size_t)level * pp + pix) * C;
    const double scale = level == 0 ? 4.0 : 16.0;  // kFeatureStride, kFeatureStride^2 (correlation.cpp:51)
    const double bx = coords[2 * pix] / scale, by = coords[2 * pix + 1] / scale;
    for (int o = warp; o < 49; o += nw) {
        const int alpha = o / 7, beta = o - 7 * alpha;
        const float r = level == 0 ? corr_exact_warp(g, f0, w0, h0, C, bx + (beta - 3), by + (alpha - 3))
                                   : corr_exact_warp(g, f1, w1, h1, C, bx + (beta - 3), by + (alpha - 3));
        if ((threadIdx.x & 31) == 0) out[((size_t)level * pp + pix) * 49 + o] = r;
    }
}

}  // namespace

int corr_smem_bytes(int channels) { return corr_layout(channels).total_bytes; }

cudaError_t launch_corr(const CorrParams& p, cudaStream_t stream) {
    if (p.n_edges <= 0) return cudaSuccess;
    const int smem = corr_smem_bytes(p.channels);
    cudaError_t err = cudaFuncSetAttribute(corr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    corr_kernel<<<p.n_edges, kThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_corr_direct(int pp, int C, const float* feats, const double* coords, const float* f0, int w0,
                               int h0, const float* f1, int w1, int h1, float* out, cudaStream_t stream) {
    if (pp <= 0) return cudaSuccess;
    corr_direct_kernel<<<dim3(pp, 2), 256, 0, stream>>>(pp, C, feats, coords, f0, w0, h0, f1, w1, h1, out);
    return cudaGetLastError();
}

cudaError_t launch_gram(const float* feat0, float* gram0, int W0, int H0, const float* feat1, float* gram1, int W1,
                        int H1, int D, int num_sms, cudaStream_t stream) {
    const int threads = 256;
    const int cells = W0 * H0 + W1 * H1;
    if (cells <= 0) return cudaSuccess;
    int blocks = (cells + 7) / 8;
    const int cap = num_sms * 16;
    if (blocks > cap) blocks = cap;
    gram_kernel<<<blocks, threads, 0, stream>>>(GramLevel{feat0, gram0, W0, H0}, GramLevel{feat1, gram1, W1, H1}, D);
    return cudaGetLastError();
}

}  // namespace pvo_dev
