// corr_tma.cu — the production correlation kernel (K2) for D = 128, sm_100a.
//
// Same arithmetic as corr.cu (see its header: dots at integer cells + per-frame
// Gram terms, regrouped by linearity from correlation.cpp:8-71), organised for
// the B200 memory system and issue rate:
//   * one (edge, level) tile = the 9x9-cell union window of the patch's 9
//     pixels; the 729 dots <g_p, f_cell> of a tile are owned by ONE warp (lane
//     owns 3 cells x 9 pixels, lanes 27..31 idle), so a tile needs no block
//     barrier and no cross-warp reduction;
//   * persistent CTAs (one per SM, 8 warps), each walking its share of the
//     edges in target-frame order so the frames being read stay in L2; warps
//     grab tiles dynamically from a CTA counter;
//   * every warp runs its own 3-stage TMA ring over 16-channel chunks: per
//     chunk a 4-D tensor copy of the tile [81 cells][16 ch] (64B-swizzled, so
//     the 8-lane phases of a 128-bit shared load hit 8 distinct bank groups;
//     out-of-image cells are zero-filled by TMA, which IS the reference's zero
//     padding, features.cpp:15-17) and a 2-D copy of the patch descriptors
//     [9 px][16 ch]; the first chunk of a tile also brings the tile's planar
//     Gram records [5][9][12] and its 9 reprojected pixels.  The warp's elected
//     lane refills a stage as soon as the warp has consumed it;
//   * FP32 FMA dot products in fixed channel order (deterministic); output
//     recombination in FP32 with the bilinear weights' fractional parts taken
//     exactly in FP64 (x - floor(x)) as the reference does; coalesced stores.
// (edge, level) tiles whose pixel windows do not fit one 9x9 tile (extreme
// zoom) are diverted to an overflow list that the generic kernel (corr.cu)
// finishes; tiles whose every tap is zero padding are zero-filled directly.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "geometry.cuh"
#include "kernels.cuh"

namespace pvo_dev {

namespace {

constexpr int kWarps = 8;
constexpr int kThreads = 32 * kWarps;
constexpr int kD = 128;
constexpr int kBox = 9;
constexpr int kCells = kBox * kBox;
constexpr int kPix = 9;
constexpr int kOut = kPix * 49;
constexpr int kChunkCh = 16;                           // channels per pipeline chunk (64 B rows)
constexpr int kChunks = kD / kChunkCh;                 // 8
constexpr int kStages = 3;                             // per-warp ring depth
constexpr int kChunkTileBytes = kCells * kChunkCh * 4;  // 5184: [81][16] f32, 64B swizzle
constexpr int kChunkGOff = 5248;                        // 128-aligned
constexpr int kChunkGBytes = kPix * kChunkCh * 4;       // 576: [9][16] f32
constexpr int kStageBytes = 6144;                       // 1024-aligned stages
constexpr int kGramW = 12;                              // Gram box x extent (48 B rows)
constexpr int kGramPlane = kBox * kGramW;               // 108
constexpr int kGramBytes = 5 * kGramPlane * 4;          // 2160: [5][9][12]
constexpr int kCoordBytes = kPix * 2 * 8;               // 144
constexpr int kHeaderBytes = 2304;
constexpr uint32_t kChunkTx = kChunkTileBytes + kChunkGBytes;
constexpr uint32_t kHeaderTx = kGramBytes + kCoordBytes;
constexpr int kHeaderOff = kStages * kStageBytes;        // 18432, 2 tile headers
constexpr int kDotsOff = kHeaderOff + 2 * kHeaderBytes;  // 23040: [9][81] f32
constexpr int kPixOff = kDotsOff + 2944;                 // 25984: PixData
constexpr int kMetaOff = kPixOff + 640;                  // 26624: 2 tile records
constexpr int kWarpBytes = 27648;
constexpr int kSmemBytes = kWarps * kWarpBytes + 1024;   // + alignment slack
static_assert(kChunkGOff >= kChunkTileBytes && kChunkGOff + kChunkGBytes <= kStageBytes, "stage");
static_assert(kGramBytes + kCoordBytes <= kHeaderBytes, "header");
static_assert(kMetaOff + 64 <= kWarpBytes && kWarpBytes % 1024 == 0, "warp region");
static_assert(kCorrMetaInts == 8, "tile record");

// tile record kinds (TileRec.code bits 0..1); bits 8..16: far-pixel mask
constexpr int kKindTma = 0, kKindOverflow = 1, kKindZero = 2, kKindBad = 3;

struct TileRec {
    int x0, y0, code, slot;  // window origin (cells), kind | far << 8, frame-store slot
    int grow, e, level, pad;  // patch-descriptor row ((patch * 2 + level) * 9), edge, level
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ float rsqrt_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

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

__global__ void __launch_bounds__(kThreads, 1)
    corr_tma_kernel(const __grid_constant__ CUtensorMap feat0, const __grid_constant__ CUtensorMap feat1,
                    const __grid_constant__ CUtensorMap gram0, const __grid_constant__ CUtensorMap gram1,
                    const __grid_constant__ CUtensorMap patch, CorrTmaParams a) {
    extern __shared__ unsigned char smem_raw[];
    // 1024-aligned base, derived by offset so the compiler keeps the shared address space
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t full[kWarps * kStages];
    __shared__ int s_next;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int G = gridDim.x, b = blockIdx.x;
    const int my_edges = a.n_edges > b ? (a.n_edges - 1 - b) / G + 1 : 0;
    const int n_tiles = 2 * my_edges;

    // ---- prologue (all warps): coordinates and tile records of this CTA's edges ----
    for (int i = tid; i < my_edges * kPix; i += kThreads) {
        const int pos = b + (i / kPix) * G;
        const int e = a.order ? a.order[pos] : pos;
        const int pix = i % kPix;
        double xy[2];
        edge_pixel(a, e, pix, xy);
        a.coords[(size_t)e * 18 + 2 * pix] = xy[0];
        a.coords[(size_t)e * 18 + 2 * pix + 1] = xy[1];
    }
    // the tile headers re-read these coordinates with bulk (async-proxy) copies
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    for (int i = tid; i < n_tiles; i += kThreads) {
        const int pos = b + (i >> 1) * G;
        const int e = a.order ? a.order[pos] : pos;
        const int level = i & 1;
        const double scale = level ? 16.0 : 4.0;  // kFeatureStride (features.hpp:46)
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
        int kind = kKindTma;
        if (!finite) {
            atomicOr(a.status, 1 << kDevBadCoords);  // correlation.cpp:43-45
            kind = kKindBad;
        } else if (far == (1 << kPix) - 1) {
            kind = kKindZero;  // every tap of every pixel is zero padding
        } else if (xmax - xmin + 8 > kBox || ymax - ymin + 8 > kBox) {
            const int slot = atomicAdd(a.overflow_count, 1);
            a.overflow[slot] = 2 * e + level;
            kind = kKindOverflow;
        }
        const int fslot = a.e_slot ? a.e_slot[e] : a.pose_slot[a.e_pose[e]];
        int4* rec = reinterpret_cast<int4*>(a.meta) + 2 * ((size_t)2 * pos + level);
        rec[0] = make_int4(xmin - 3, ymin - 3, kind | (far << 8), fslot);
        rec[1] = make_int4((a.e_patch[e] * 2 + level) * kPix, e, level, 0);
    }
    if (tid < kWarps * kStages) mbar_init(&full[tid], 1);
    if (tid == 0) s_next = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    // ================= per-warp pipeline =================
    unsigned char* wb = smem + warp * kWarpBytes;
    const uint32_t wbu = smem_u32(wb);                    // shared-window addresses, computed once
    const uint32_t baru = smem_u32(full + warp * kStages);  // stage s barrier: baru + 8 * s

    // issue cursor (warp-uniform): pending tile + its record, current tile, chunk
    int pend = 0;
    int4 pr0 = make_int4(0, 0, 0, 0), pr1 = make_int4(0, 0, 0, 0);
    auto grab = [&]() {
        int t = 0;
        if (lane == 0) t = atomicAdd(&s_next, 1);
        pend = __shfl_sync(0xffffffffu, t, 0);
        if (pend < n_tiles) {
            const int4* src = reinterpret_cast<const int4*>(a.meta) + 2 * ((size_t)2 * (b + (pend >> 1) * G) + (pend & 1));
            pr0 = __ldcg(src);
            pr1 = __ldcg(src + 1);
        }
    };
    grab();
    int4 ir0 = make_int4(0, 0, 0, 0), ir1 = make_int4(0, 0, 0, 0);
    int ichunk = kChunks;  // chunks of the current issue tile already issued
    bool idone = false;
    int is = 0, hi = 0;    // next stage to fill, tiles issued
    auto issue_one = [&]() {
        if (idone) return;
        while (ichunk == kChunks) {  // advance to the next tile that needs the pipeline
            if (pend >= n_tiles) {
                idone = true;
                return;
            }
            const int4 r0 = pr0, r1 = pr1;
            grab();
            const int kind = r0.z & 3;
            if (kind == kKindTma) {
                ir0 = r0;
                ir1 = r1;
                ichunk = 0;
            } else if (kind == kKindZero) {
                float* out = a.out + ((size_t)r1.y * 2 + r1.z) * kOut;
                for (int o = lane; o < kOut; o += 32) out[o] = 0.f;
            }
        }
        if (lane == 0) {
            const int level = ir1.z;
            const uint32_t bar = baru + 8 * is;
            const uint32_t st = wbu + is * kStageBytes;
            if (ichunk == 0) {
                const int hb = hi & 1;
                int4* rec = reinterpret_cast<int4*>(wb + kMetaOff + 32 * hb);
                rec[0] = ir0;
                rec[1] = ir1;
                const uint32_t hd = wbu + kHeaderOff + hb * kHeaderBytes;
                mbar_expect_tx(bar, kChunkTx + kHeaderTx);
                // TMA needs a 16-byte aligned start in the innermost (x) dimension: start at
                // floor4(x0); the 12-wide box still covers x0 .. x0 + 8
                tma_load_4d(hd, level ? &gram1 : &gram0, ir0.x & ~3, ir0.y, 0, ir0.w, bar);
                bulk_load(hd + kGramBytes, a.coords + (size_t)ir1.y * 18, kCoordBytes, bar);
            } else {
                mbar_expect_tx(bar, kChunkTx);
            }
            tma_load_4d(st, level ? &feat1 : &feat0, ichunk * kChunkCh, ir0.x, ir0.y, ir0.w, bar);
            tma_load_2d(st + kChunkGOff, &patch, ichunk * kChunkCh, ir1.x, bar);
        }
        if (ichunk == 0) ++hi;
        ++ichunk;
        is = is == kStages - 1 ? 0 : is + 1;
    };
    for (int k = 0; k < kStages; ++k) issue_one();
    __syncwarp();

    // lane -> its 3 cells (rows of the 9x9 box); lanes 27..31 compute throwaway rows
    int roff[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int r = lane + 27 * k;
        roff[k] = r * 64;
    }
    float* dots = reinterpret_cast<float*>(wb + kDotsOff);
    int cs = 0;          // stage being consumed
    uint32_t cph = 0;    // its barrier phase parity
    for (int hc = 0; hc < hi; ++hc) {
        // (even, odd)-channel sums per (cell, pixel): packed FP32x2 FMAs (FFMA2)
        float2 acc[3][kPix];
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int p = 0; p < kPix; ++p) acc[k][p] = make_float2(0.f, 0.f);
        for (int c = 0; c < kChunks; ++c) {
            mbar_wait(baru + 8 * cs, cph);
            const unsigned char* st = wb + cs * kStageBytes;
            const float* g = reinterpret_cast<const float*>(st + kChunkGOff);
            // per-chunk partial sums, then one add into the tile total: short chains
            // (8 + 8 terms per component) keep the FP32 error far inside 1e-4
            float2 part[3][kPix];
#pragma unroll
            for (int u = 0; u < kChunkCh / 4; ++u) {
                float4 v[3], gv[kPix];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    // 64B swizzle: 16-byte unit u of row r lives at unit u ^ ((r >> 1) & 3)
                    const int sw = (roff[k] >> 7) & 3;
                    v[k] = *reinterpret_cast<const float4*>(st + roff[k] + ((u ^ sw) << 4));
                }
#pragma unroll
                for (int p = 0; p < kPix; ++p) gv[p] = *reinterpret_cast<const float4*>(g + p * kChunkCh + 4 * u);
#pragma unroll
                for (int k = 0; k < 3; ++k)
#pragma unroll
                    for (int p = 0; p < kPix; ++p) {
                        const float2 va = make_float2(v[k].x, v[k].y), ga = make_float2(gv[p].x, gv[p].y);
                        part[k][p] = u == 0 ? __fmul2_rn(va, ga) : __ffma2_rn(va, ga, part[k][p]);
                    }
#pragma unroll
                for (int k = 0; k < 3; ++k)
#pragma unroll
                    for (int p = 0; p < kPix; ++p)
                        part[k][p] = __ffma2_rn(make_float2(v[k].z, v[k].w), make_float2(gv[p].z, gv[p].w), part[k][p]);
            }
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int p = 0; p < kPix; ++p) acc[k][p] = __fadd2_rn(acc[k][p], part[k][p]);
            __syncwarp();  // every lane is done with this stage: refill it
            if (++cs == kStages) {
                cs = 0;
                cph ^= 1;
            }
            issue_one();
        }

        // ---- epilogue ----
        const int hb = hc & 1;
        const int4 r0 = *reinterpret_cast<const int4*>(wb + kMetaOff + 32 * hb);
        const int4 r1 = *reinterpret_cast<const int4*>(wb + kMetaOff + 32 * hb + 16);
        const unsigned char* hd = wb + kHeaderOff + hb * kHeaderBytes;
        const float* gram = reinterpret_cast<const float*>(hd) + (r0.x & 3);  // box starts at floor4(x0)
        const double* tc = reinterpret_cast<const double*>(hd + kGramBytes);
        const int e = r1.y, level = r1.z, far = r0.z >> 8;
        if (lane < 27) {
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int p = 0; p < kPix; ++p) dots[p * kCells + lane + 27 * k] = acc[k][p].x + acc[k][p].y;
        }
        __syncwarp();
        // Separable bilinear recombination (correlation.cpp:8-23 regrouped): lane owns
        // the output column (pixel p, offset beta) and walks alpha = 0..6, carrying the
        // x-interpolated row terms of row alpha + 1 into the next step:
        //   fx(y)   = (1-ax) f[y][x] + ax f[y][x+1]
        //   dot     = (1-ay) <g, fx(y)> + ay <g, fx(y+1)>
        //   |f(x)|^2 = (1-ay)^2 |fx(y)|^2 + ay^2 |fx(y+1)|^2 + 2 ay (1-ay) <fx(y), fx(y+1)>
        // with |fx|^2 and <fx(y), fx(y+1)> from the Gram records (|f|^2, right, down,
        // diag, anti).  ax / ay are the reference's per-offset fractional parts (FP64).
        const double scale = level ? 16.0 : 4.0;  // kFeatureStride (features.hpp:46)
        const int W = level ? a.w1 : a.w0, H = level ? a.h1 : a.h0;
        float* out = a.out + ((size_t)e * 2 + level) * kOut;
#pragma unroll 1
        for (int col = lane; col < kPix * 7; col += 32) {
            const int p = (col * 37) >> 8, beta = col - 7 * p;  // col / 7 for col < 63
            float* o = out + p * 49 + beta;
            if ((far >> p) & 1) {  // every tap of this pixel is zero padding
#pragma unroll
                for (int alpha = 0; alpha < 7; ++alpha) o[alpha * 7] = 0.f;
                continue;
            }
            const double bx = tc[2 * p] / scale, by = tc[2 * p + 1] / scale;
            const int fx = clamp_floor(bx, W), fy = clamp_floor(by, H);
            const float ax = (float)((bx + (double)(beta - 3)) - (double)(fx + beta - 3));
            const float bx0 = 1.f - ax;
            const int cx = fx - 3 - r0.x + beta, cy = fy - 3 - r0.y;
            const float* d = dots + p * kCells + cy * kBox + cx;
            const float* G = gram + cy * kGramW + cx;
            const float qa = bx0 * bx0, qb = ax * ax, qc = 2.f * ax * bx0, qd = ax * bx0;
            // row terms of row y: <g, fx(y)>, |fx(y)|^2
            float dA = fmaf(ax, d[1], bx0 * d[0]);
            float nA = fmaf(qc, G[kGramPlane], fmaf(qb, G[1], qa * G[0]));
#pragma unroll
            for (int alpha = 0; alpha < 7; ++alpha) {
                const float* dn = d + (alpha + 1) * kBox;
                const float* Gn = G + (alpha + 1) * kGramW;
                const float* Gc = G + alpha * kGramW;
                const float dB = fmaf(ax, dn[1], bx0 * dn[0]);
                const float nB = fmaf(qc, Gn[kGramPlane], fmaf(qb, Gn[1], qa * Gn[0]));
                // <fx(y), fx(y+1)> = (1-ax)^2 down[x] + ax^2 down[x+1] + ax(1-ax) (diag[x] + anti[x])
                const float cr = fmaf(qd, Gc[3 * kGramPlane] + Gc[4 * kGramPlane],
                                      fmaf(qb, Gc[2 * kGramPlane + 1], qa * Gc[2 * kGramPlane]));
                const float ay = (float)((by + (double)(alpha - 3)) - (double)(fy + alpha - 3));
                const float by0 = 1.f - ay;
                const float dot = fmaf(ay, dB, by0 * dA);
                const float n2 = fmaf(2.f * ay * by0, cr, fmaf(ay * ay, nB, by0 * by0 * nA));
                o[alpha * 7] = n2 > 1e-12f ? dot * rsqrt_approx(n2) : 0.f;  // correlation.cpp:22
                dA = dB;
                nA = nB;
            }
        }
        __syncwarp();  // dots are rewritten by the next tile
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
    corr_tma_kernel<<<grid, kThreads, kSmemBytes, stream>>>(maps[0], maps[1], maps[2], maps[3], maps[4], p);
    return cudaGetLastError();
}

}  // namespace pvo_dev
