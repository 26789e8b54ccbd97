// corr_tma.cu — the production correlation kernel (K2) for D = 128, sm_100a.
//
// Same arithmetic as corr.cu (see its header: dots at integer cells + per-frame
// Gram terms, regrouped by linearity from correlation.cpp:8-71), organised for
// the B200 memory system:
//   * persistent CTAs (one per SM), each walking its share of the edges in
//     target-frame order, so the frames being read stay resident in L2;
//   * a 3-stage TMA pipeline: for every (edge, level) one elected thread issues
//       - a 4-D tensor copy of the 9x9-cell tile [9][9][132] fp32 whose channel
//         box (132) overhangs the 128 stored channels, so TMA zero-fills 4 pad
//         channels per cell — the padded, bank-conflict-free layout the FMA loop
//         wants — and zero-fills out-of-image cells, which IS the reference's
//         zero padding (features.cpp:15-17);
//       - a 4-D tensor copy of the tile's Gram records [9][9][8];
//       - a 1-D bulk copy of the patch's 9 x 128 descriptors;
//     all completing on one mbarrier (complete_tx bytes);
//   * FP32 FMA dot products, register-blocked 3 cells x 9 pixels per lane, warps
//     split the channel chunks; fixed-order cross-warp sum (deterministic);
//   * output recombination in FP32 with the bilinear weights' fractional parts
//     taken exactly in FP64 (x - floor(x)), as the reference does.
// (edge, level) tiles whose 9 pixel windows do not fit one 9x9 tile (extreme
// zoom, pixels far outside the image) are diverted to an overflow list that the
// generic kernel (corr.cu) finishes.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "geometry.cuh"
#include "kernels.cuh"

namespace pvo_dev {

namespace {

#ifndef PVO_CORR_UNROLL
#define PVO_CORR_UNROLL 2
#endif
constexpr int kCorrUnroll = PVO_CORR_UNROLL;  // channel-chunk unroll of the FMA loop
constexpr int kConsumerWarps = 8;              // two groups of 4 warps (ping-pong)
constexpr int kGroupWarps = 4;
constexpr int kGroupThreads = 32 * kGroupWarps;
constexpr int kThreads = 32 * (kConsumerWarps + 1);  // + one producer warp
constexpr int kD = 128;
constexpr int kDP = 132;  // padded cell stride (floats)
constexpr int kBox = 9;
constexpr int kCells = kBox * kBox;
constexpr int kPix = 9;
constexpr int kStages = 3;
constexpr int kTileBytes = kCells * kDP * 4;                  // 42768
constexpr int kTileRegion = (kTileBytes + 127) / 128 * 128;   // 42880
constexpr int kGramBytes = kCells * 8 * 4;                    // 2592
constexpr int kGramRegion = (kGramBytes + 127) / 128 * 128;   // 2688
constexpr int kGBytes = kPix * kD * 4;                        // 4608
constexpr int kCoordBytes = kPix * 2 * 8;                    // 144: the 9 reprojected pixels
constexpr int kInfoOff = kTileRegion + kGramRegion + kGBytes;  // tile info written by the producer
constexpr int kCoordOff = kInfoOff + 32;
constexpr int kStageBytes = (kCoordOff + 160 + 1023) / 1024 * 1024;  // 51200: TMA dst needs 128 B alignment
constexpr int kTxBytes = kTileBytes + kGramBytes + kGBytes + kCoordBytes;
struct StageInfo {
    int4 meta;  // union origin x, y, extent w, h (w <= 0: not on this path)
    int e, level;
    int seq;  // tile index the stage currently holds (written by the producer)
};
// per consumer group scratch (after the stages); dots / gram / pixel data are
// double-buffered by the group's tile parity
constexpr int kPartBytes = kGroupWarps * kPix * kCells * 4;   // [4][9][81] f32
constexpr int kDotsBytes = kPix * kCells * 4;                  // [9][81] f32
constexpr int kGramSBytes = kCells * 5 * 4;                    // [81][5] f32
constexpr int kGroupBytes = kPartBytes + 2 * (kDotsBytes + kGramSBytes) + 2 * 640;
constexpr int kScratchOff = kStages * kStageBytes;
constexpr int kSmemBytes = kScratchOff + 2 * kGroupBytes + 1024;  // + alignment slack

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_barrier(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

struct TileMeta {
    int x0, y0, tw, th;  // union origin (cells) and extent; tw <= 0: not on this path
};

// reproject_patch of pixel `pix` of edge e (camera.cpp:47-71)
__device__ inline void edge_pixel(const CorrTmaParams& a, int e, int pix, double* xy) {
    if (a.coords_in) {
        xy[0] = a.coords_in[(size_t)e * 18 + 2 * pix];
        xy[1] = a.coords_in[(size_t)e * 18 + 2 * pix + 1];
        return;
    }
    const int k = a.e_patch[e];
    const SE3 pi = se3_load(a.poses + 7 * a.patch_src[k]);
    const SE3 pj = se3_load(a.poses + 7 * a.e_pose[e]);
    const double px = a.patch_x[(size_t)k * 9 + pix], py = a.patch_y[(size_t)k * 9 + pix];
    if (se3_equal(pi, pj)) {
        xy[0] = px;
        xy[1] = py;
        return;
    }
    const Relative rel = relative_pose(pi, pj);
    const Cam K{a.K[0], a.K[1], a.K[2], a.K[3]};
    reproject_point(rel, K, a.depth[k], px, py, &xy[0], &xy[1]);
}

__device__ __forceinline__ int clamp_floor(double b, int extent) {
    return (int)floor(fmin(fmax(b, -16.0), (double)extent + 16.0));
}


// Dot products of one tile for this warp's 8 channel chunks: lane owns NCS
// union cells (lane, lane+32, ...) x 9 pixels.  Component-major FMA order
// (9 * NCS independent FMAs between dependent ones).  Writes the partials.
template <int NCS>
__device__ __forceinline__ void dot_phase(const float* tile, const float* g, float* s_part, int TW, int NC, int lane,
                                          int gw) {
    int roff[NCS];
#pragma unroll
    for (int ci = 0; ci < NCS; ++ci) {
        const int c = lane + 32 * ci;
        const int cy = TW == 8 ? c >> 3 : (c * 57) >> 9, cx = c - cy * TW;  // c / TW, TW in {8, 9}
        roff[ci] = c < NC ? (cy * kBox + cx) * kDP : 0;  // cells past NC read cell 0; never stored
    }
    float acc[NCS][kPix];
#pragma unroll
    for (int ci = 0; ci < NCS; ++ci)
#pragma unroll
        for (int p = 0; p < kPix; ++p) acc[ci][p] = 0.f;
#pragma unroll kCorrUnroll
    for (int j = 0; j < 8; ++j) {
        const int ch = gw + kGroupWarps * j;
        float4 gv[kPix], v[NCS];
#pragma unroll
        for (int p = 0; p < kPix; ++p) gv[p] = *reinterpret_cast<const float4*>(g + p * kD + 4 * ch);
#pragma unroll
        for (int ci = 0; ci < NCS; ++ci) v[ci] = *reinterpret_cast<const float4*>(tile + roff[ci] + 4 * ch);
#pragma unroll
        for (int ci = 0; ci < NCS; ++ci)
#pragma unroll
            for (int p = 0; p < kPix; ++p) acc[ci][p] = fmaf(v[ci].x, gv[p].x, acc[ci][p]);
#pragma unroll
        for (int ci = 0; ci < NCS; ++ci)
#pragma unroll
            for (int p = 0; p < kPix; ++p) acc[ci][p] = fmaf(v[ci].y, gv[p].y, acc[ci][p]);
#pragma unroll
        for (int ci = 0; ci < NCS; ++ci)
#pragma unroll
            for (int p = 0; p < kPix; ++p) acc[ci][p] = fmaf(v[ci].z, gv[p].z, acc[ci][p]);
#pragma unroll
        for (int ci = 0; ci < NCS; ++ci)
#pragma unroll
            for (int p = 0; p < kPix; ++p) acc[ci][p] = fmaf(v[ci].w, gv[p].w, acc[ci][p]);
    }
#pragma unroll
    for (int ci = 0; ci < NCS; ++ci) {
        const int c = lane + 32 * ci;
        if (c < NC) {
#pragma unroll
            for (int p = 0; p < kPix; ++p) s_part[(gw * kPix + p) * kCells + c] = acc[ci][p];
        }
    }
}

// Per-pixel data of one tile: fractional bilinear weights per offset (exact
// x - floor(x) in FP64, stored FP32) and the pixel's window origin in the
// union tile.
struct PixData {
    float ax[kPix][7];
    float ay[kPix][7];
    int cx0[kPix];
    int cy0[kPix];
};
static_assert(sizeof(PixData) <= 640, "PixData");

__global__ void __launch_bounds__(kThreads, 1)
    corr_tma_kernel(const __grid_constant__ CUtensorMap feat0, const __grid_constant__ CUtensorMap feat1,
                    const __grid_constant__ CUtensorMap gram0, const __grid_constant__ CUtensorMap gram1,
                    CorrTmaParams a) {
    extern __shared__ unsigned char smem_raw[];
    unsigned char* smem =
        reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[kStages];
    __shared__ __align__(8) uint64_t empty[kStages];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int G = gridDim.x, b = blockIdx.x;
    const int my_edges = a.n_edges > b ? (a.n_edges - 1 - b) / G + 1 : 0;
    const int n_tiles = 2 * my_edges;

    // ---- phase 0 (all warps): coordinates and tile geometry of this CTA's edges ----
    for (int i = tid; i < my_edges * kPix; i += kThreads) {
        const int e = a.order ? a.order[b + (i / kPix) * G] : b + (i / kPix) * G;
        const int pix = i % kPix;
        double xy[2];
        edge_pixel(a, e, pix, xy);
        a.coords[(size_t)e * 18 + 2 * pix] = xy[0];
        a.coords[(size_t)e * 18 + 2 * pix + 1] = xy[1];
    }
    // the producer re-reads these coordinates with bulk (async-proxy) copies
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    for (int i = tid; i < my_edges * 2; i += kThreads) {
        const int e = a.order ? a.order[b + (i >> 1) * G] : b + (i >> 1) * G;
        const int level = i & 1;
        const double scale = level ? 16.0 : 4.0;
        const int W = level ? a.w1 : a.w0, H = level ? a.h1 : a.h0;
        int xmin = 1 << 30, xmax = -(1 << 30), ymin = 1 << 30, ymax = -(1 << 30);
        bool finite = true;
        int far = 0;  // pixels whose whole 8x8 tap window lies outside the grid: all 49 outputs are 0
        for (int p = 0; p < kPix; ++p) {
            const double x = a.coords[(size_t)e * 18 + 2 * p], y = a.coords[(size_t)e * 18 + 2 * p + 1];
            finite = finite && isfinite(x) && isfinite(y);
            const int fx = clamp_floor(x / scale, W), fy = clamp_floor(y / scale, H);
            if (fx + 4 < 0 || fx - 3 >= W || fy + 4 < 0 || fy - 3 >= H) {
                far |= 1 << p;
                continue;
            }
            xmin = min(xmin, fx);
            xmax = max(xmax, fx);
            ymin = min(ymin, fy);
            ymax = max(ymax, fy);
        }
        TileMeta m{xmin - 3, ymin - 3, xmax - xmin + 8, ymax - ymin + 8};
        if (!finite) {
            atomicOr(a.status, 1 << kDevBadCoords);  // correlation.cpp:43-45
            m.tw = -1;
        } else if (far == (1 << kPix) - 1) {
            m = TileMeta{0, 0, -2, 0};  // every tap of every pixel is zero padding
        } else if (m.tw > kBox || m.th > kBox) {
            const int slot = atomicAdd(a.overflow_count, 1);
            a.overflow[slot] = 2 * e + level;
            m.tw = 0;
        }
        reinterpret_cast<int4*>(a.meta)[2 * e + level] = make_int4(m.x0, m.y0, m.tw, m.th | (far << 8));
    }
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kGroupWarps);
            reinterpret_cast<StageInfo*>(smem + s * kStageBytes + kInfoOff)->seq = -1;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto tile_edge = [&](int t) { return a.order ? a.order[b + (t >> 1) * G] : b + (t >> 1) * G; };

    if (warp == kConsumerWarps) {
        // ================= producer warp =================
        if (lane == 0) {
            for (int t = 0; t < n_tiles; ++t) {
                const int s = t % kStages;
                if (t >= kStages) mbar_wait(&empty[s], (uint32_t)(((t / kStages) - 1) & 1));
                const int e = tile_edge(t), level = t & 1;
                const int4 m = reinterpret_cast<const int4*>(a.meta)[2 * e + level];
                unsigned char* st = smem + s * kStageBytes;
                StageInfo* info = reinterpret_cast<StageInfo*>(st + kInfoOff);
                info->meta = m;
                info->e = e;
                info->level = level;
                *reinterpret_cast<volatile int*>(&info->seq) = t;
                if (m.z <= 0) {  // not on this path: complete the phase without data
                    mbar_arrive(&full[s]);
                    continue;
                }
                const int slot = a.e_slot ? a.e_slot[e] : a.pose_slot[a.e_pose[e]];
                mbar_expect_tx(&full[s], kTxBytes);
                tma_load_4d(st, level ? &feat1 : &feat0, 0, m.x, m.y, slot, &full[s]);
                tma_load_4d(st + kTileRegion, level ? &gram1 : &gram0, 0, m.x, m.y, slot, &full[s]);
                const float* g = a.patch_feats + ((size_t)a.e_patch[e] * 2 + level) * kPix * kD;
                bulk_load(st + kTileRegion + kGramRegion, g, kGBytes, &full[s]);
                bulk_load(st + kCoordOff, a.coords + (size_t)e * 18, kCoordBytes, &full[s]);
            }
        }
        return;
    }

    // ================= consumer groups =================
    const int grp = warp / kGroupWarps;           // 0 or 1
    const int gw = warp - grp * kGroupWarps;       // warp within the group
    const int gtid = tid - grp * kGroupThreads;    // thread within the group
    unsigned char* gscr = smem + kScratchOff + grp * kGroupBytes;
    float* s_part = reinterpret_cast<float*>(gscr);
    const int bar_id = 1 + grp;

    int parity = 0;  // this group's tile parity (double buffers)
    for (int t = grp; t < n_tiles; t += 2, parity ^= 1) {
        const int s = t % kStages;
        float* s_dots = reinterpret_cast<float*>(gscr + kPartBytes + parity * (kDotsBytes + kGramSBytes));
        float* s_gram = s_dots + kPix * kCells;
        PixData* pd = reinterpret_cast<PixData*>(gscr + kPartBytes + 2 * (kDotsBytes + kGramSBytes) + parity * 640);
        const unsigned char* st = smem + s * kStageBytes;
        // Stages alternate between the two groups (kStages is odd), so a group
        // can reach stage s while it still holds an older phase: the parity
        // wait alone would then pass on the stale phase.  Wait for the producer
        // to claim the stage for tile t first; from then on the parity is exact.
        while (reinterpret_cast<const volatile StageInfo*>(st + kInfoOff)->seq != t) {
        }
        mbar_wait(&full[s], (uint32_t)((t / kStages) & 1));
        const StageInfo info = *reinterpret_cast<const StageInfo*>(st + kInfoOff);
        const int e = info.e, level = info.level;
        const int4 m = info.meta;
        const double* tc = reinterpret_cast<const double*>(st + kCoordOff);
        const bool active = m.z > 0;
        const int TW = m.z, TH = m.w & 0xff, far = m.w >> 8, NC = active ? TW * TH : 0;
        if (m.z == -2) {  // all taps outside the grid: the reference's zero padding gives 0 everywhere
            float* out = a.out + ((size_t)e * 2 + level) * kPix * 49;
            for (int o = gtid; o < kPix * 49; o += kGroupThreads) out[o] = 0.f;
        }

        if (active) {
            const float* tile = reinterpret_cast<const float*>(st);
            const float* g = reinterpret_cast<const float*>(st + kTileRegion + kGramRegion);
            // ---- dot products: lane owns 2 or 3 union cells x 9 pixels; warp owns 8 chunks ----
            if (NC <= 64) {
                dot_phase<2>(tile, g, s_part, TW, NC, lane, gw);
            } else {
                dot_phase<3>(tile, g, s_part, TW, NC, lane, gw);
            }
            // Gram records of the union cells (this group's copy); TW is 8 or 9
            const float* gr = reinterpret_cast<const float*>(st + kTileRegion);
            if (gtid < NC) {
                const int c = gtid;
                const int cy = TW == 8 ? c >> 3 : (c * 57) >> 9, cx = c - cy * TW;
                const float* src = gr + (cy * kBox + cx) * 8;
#pragma unroll
                for (int r = 0; r < 5; ++r) s_gram[5 * c + r] = src[r];
            }
            // per-pixel bilinear data (features.cpp:10-13 arithmetic)
            if (gtid >= kGroupThreads - kPix) {
                const int p = gtid - (kGroupThreads - kPix);
                const double scale = level ? 16.0 : 4.0;
                const int W = level ? a.w1 : a.w0, H = level ? a.h1 : a.h0;
                const double bx = tc[2 * p] / scale;
                const double by = tc[2 * p + 1] / scale;
                const int fx = clamp_floor(bx, W), fy = clamp_floor(by, H);
#pragma unroll
                for (int o = 0; o < 7; ++o) {
                    pd->ax[p][o] = (float)((bx + (double)(o - 3)) - (double)(fx + o - 3));
                    pd->ay[p][o] = (float)((by + (double)(o - 3)) - (double)(fy + o - 3));
                }
                pd->cx0[p] = fx - 3 - m.x;
                pd->cy0[p] = fy - 3 - m.y;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
        named_barrier(bar_id, kGroupThreads);   // partials, gram copy and pixel data complete
        if (active && gtid < NC) {
            const int c = gtid;
#pragma unroll
            for (int p = 0; p < kPix; ++p) {
                float sum = s_part[(0 * kPix + p) * kCells + c];
                sum += s_part[(1 * kPix + p) * kCells + c];
                sum += s_part[(2 * kPix + p) * kCells + c];
                sum += s_part[(3 * kPix + p) * kCells + c];
                s_dots[p * kCells + c] = sum;
            }
        }
        named_barrier(bar_id, kGroupThreads);  // dots complete; s_part free for the next tile
        if (active && gtid < 2 * kPix * 7) {
            // thread -> (pixel p, row alpha, half of the 7 beta offsets)
            const int pair = gtid >> 1, half = gtid & 1;
            const int p = (pair * 37) >> 8, alpha = pair - 7 * p;  // pair / 7 for pair < 63
            const float ay = pd->ay[p][alpha];
            const int row = (pd->cy0[p] + alpha) * TW + pd->cx0[p];
            const float* d = s_dots + p * kCells;
            float* out = a.out + ((size_t)e * 2 + level) * kPix * 49 + p * 49 + alpha * 7;
            const int b0 = half ? 4 : 0, b1 = half ? 7 : 4;
            const bool far_p = (far >> p) & 1;  // window entirely outside the grid
            for (int beta = b0; beta < b1; ++beta) {
                if (far_p) {
                    out[beta] = 0.f;
                    continue;
                }
                const float ax = pd->ax[p][beta];
                const int c00 = row + beta;
                const float w00 = (1.f - ax) * (1.f - ay), w10 = ax * (1.f - ay);
                const float w01 = (1.f - ax) * ay, w11 = ax * ay;
                float dot = w00 * d[c00];
                dot = fmaf(w10, d[c00 + 1], dot);
                dot = fmaf(w01, d[c00 + TW], dot);
                dot = fmaf(w11, d[c00 + TW + 1], dot);
                const float* g00 = s_gram + 5 * c00;
                const float* g10 = g00 + 5;
                const float* g01 = g00 + 5 * TW;
                const float* g11 = g01 + 5;
                // |f(x)|^2 = sum_t sum_t' w_t w_t' <f_t, f_t'> (Gram record: |f|^2, right, down, diag, anti)
                float n2 = w00 * w00 * g00[0];
                n2 = fmaf(w10 * w10, g10[0], n2);
                n2 = fmaf(w01 * w01, g01[0], n2);
                n2 = fmaf(w11 * w11, g11[0], n2);
                float cross = w00 * w10 * g00[1];
                cross = fmaf(w01 * w11, g01[1], cross);
                cross = fmaf(w00 * w01, g00[2], cross);
                cross = fmaf(w10 * w11, g10[2], cross);
                cross = fmaf(w00 * w11, g00[3], cross);
                cross = fmaf(w10 * w01, g00[4], cross);
                n2 = fmaf(2.f, cross, n2);
                out[beta] = n2 > 1e-12f ? dot * rsqrtf(n2) : 0.f;  // correlation.cpp:22
            }
        }
    }
}

}  // namespace

int corr_tma_smem_bytes() { return kSmemBytes; }

cudaError_t launch_corr_tma(const CorrTmaParams& p, const CUtensorMap* maps, int num_sms, cudaStream_t stream) {
    if (p.n_edges <= 0) return cudaSuccess;
    cudaError_t err = cudaFuncSetAttribute(corr_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (err != cudaSuccess) return err;
    int grid = num_sms;
    if (grid > p.n_edges) grid = p.n_edges;
    corr_tma_kernel<<<grid, kThreads, kSmemBytes, stream>>>(maps[0], maps[1], maps[2], maps[3], p);
    return cudaGetLastError();
}

}  // namespace pvo_dev
