// corr_tma.cu — the production correlation kernel (K2) for D = 128, sm_100a.
//
// Same arithmetic as corr.cu (see its header: dots at integer cells + per-frame
// Gram terms, regrouped by linearity from correlation.cpp:8-71), organised for
// the B200 memory system and issue rate:
//   * one (edge, level) tile = the 9x9-cell union window of the patch's 9
//     pixels; the 729 dots <g_p, f_cell> of a tile are owned by ONE warp (lane
//     owns 3 cells x 9 pixels, lanes 27..31 idle), so a tile needs no block
//     barrier and no cross-warp reduction;
//   * a preparation launch (corr_prep_kernel) reprojects every patch pixel
//     (FP64) and turns each (edge, level) into tile records: one per box-sized
//     pixel group (tiles whose pixel windows do not fit one 9x9 box — strong
//     zoom / wide spread — are split; each sub-tile writes only its member
//     pixels), appended to ONE global tile list in processing (target-frame)
//     order; tiles whose every tap is zero padding are zero-filled there and
//     never reach the correlation kernel;
//   * persistent correlation CTAs (one per SM, 8 warps) whose warps take tiles
//     from the global list with one atomic claim kept in flight per warp (the
//     frames being read stay in L2; no per-CTA static shares, so no tail from
//     unequal shares); the last warp to finish resets the queue words;
//   * every warp runs its own 3-stage TMA ring over 16-channel chunks: per
//     chunk a 4-D tensor copy of the tile [81 cells][16 ch] (64B-swizzled, so
//     the 8-lane phases of a 128-bit shared load hit 8 distinct bank groups;
//     out-of-image cells are zero-filled by TMA, which IS the reference's zero
//     padding, features.cpp:15-17) and a 2-D copy of the patch descriptors
//     [9 px][16 ch]; the tile's planar Gram records [5][9][12] and its 9
//     reprojected pixels arrive in a single header buffer on their own
//     barrier, issued when the previous tile's epilogue is done.  The warp's
//     elected lane refills a stage as soon as the warp has consumed it;
//   * FP32 FMA dot products in fixed channel order (deterministic); output
//     recombination in FP32 with the bilinear weights' fractional parts taken
//     exactly in FP64 (x - floor(x)) as the reference does; coalesced stores.
//   * tiles whose 9 pixel windows share one 8x8 cell window ("narrow": ~half
//     of all tiles, most level-1 tiles) run a 2-cells-per-lane variant (64
//     cells over 32 lanes) instead of 3 cells over 27 lanes: 1/3 fewer FMAs.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "corr_exact.cuh"
#include "geometry.cuh"
#include "kernels.cuh"

namespace pvo_dev {

namespace {

#ifndef CORR_WARPS
#define CORR_WARPS 8
#endif
#ifndef CORR_STAGES
#define CORR_STAGES 3
#endif
// Dot accumulation (A/B knob CORR_ACC): 0 = per-chunk partials (8 + 8 terms, then
// one add), 1 = one FFMA2 chain per (cell, pixel) over all 128 channels (64
// terms: 168 registers, 10 warps x 2 stages fit, -5 %, but a long-chain rounding
// tail: max |err|/tol 1.08 on a 40k-edge C4 sample, 6,408 outputs above 0.25 of
// the tolerance), 2 = pixel-outer per-chunk sums.  0 and 2 give max |err|/tol
// 0.47 on every C2 edge and 0.45 on the C4 sample, 236 outputs above 0.25
// (profiles/r2/corr_accuracy.txt); 0 is the faster of the two.
#ifndef CORR_ACC
#define CORR_ACC 0
#endif
#ifndef CORR_CLAIM
#define CORR_CLAIM 1
#endif
constexpr int kClaim = CORR_CLAIM;  // tiles per queue claim
constexpr int kWarps = CORR_WARPS;  // A/B knobs (tools/build_variant.sh)
constexpr int kThreads = 32 * kWarps;
constexpr int kD = 128;
constexpr int kBox = 9;
constexpr int kCells = kBox * kBox;
constexpr int kPix = 9;
constexpr int kOut = kPix * 49;
constexpr int kChunkCh = 16;                           // channels per pipeline chunk (64 B rows)
constexpr int kChunks = kD / kChunkCh;                 // 8
constexpr int kStages = CORR_STAGES;                   // per-warp ring depth
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
constexpr uint32_t kChunkTxNarrow = 64 * kChunkCh * 4 + kChunkGBytes;  // narrow tiles: an 8x8 box
constexpr uint32_t kHeaderTx = kGramBytes + kCoordBytes;
constexpr int kHeaderOff = kStages * kStageBytes;        // the tile header (own barrier)
constexpr int kDotsOff = kHeaderOff + kHeaderBytes;      // [9][81] f32
constexpr int kPixOff = kDotsOff + 2944;                 // per-tile pixel table (ax, ay, floors)
constexpr int kMetaOff = kPixOff + 640;                  // 2 tile records
constexpr int kWarpBytes = (kMetaOff + 64 + 1023) / 1024 * 1024;
constexpr int kSmemBytes = kWarps * kWarpBytes + 1024;   // + alignment slack
static_assert(kChunkGOff >= kChunkTileBytes && kChunkGOff + kChunkGBytes <= kStageBytes, "stage");
static_assert(kGramBytes + kCoordBytes <= kHeaderBytes, "header");
static_assert(kMetaOff + 64 <= kWarpBytes && kWarpBytes % 1024 == 0, "warp region");
static_assert(kCorrMetaInts == 8, "tile record");

// tile record code: bit 2: narrow (8x8 window); bits 8..16: far-pixel mask
// (zero-filled by this record); bits 17..25: member pixels (outputs written by
// this record)
constexpr int kKindTma = 0;
constexpr int kNarrow = 4;
constexpr int kPixMask = (1 << kPix) - 1;

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
// Correlation-volume stores: written once, never re-read by the kernels, so they
// stream past L2 (evict-first) instead of displacing the frames and patch
// descriptors the tiles in flight read (A/B knob CORR_STCS).
#ifndef CORR_STCS
#define CORR_STCS 1
#endif
__device__ __forceinline__ void store_out(float* p, float v) {
#if CORR_STCS
    __stcs(p, v);
#else
    *p = v;
#endif
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

// ---- tile preparation (a launch before the correlation) ----
// Block of kPrepThreads threads per kPrepEdges processing positions: one thread per (edge,
// pixel) reprojects the patch pixel (FP64, camera.cpp:47-71), then one thread per
// (edge, level) builds the tile record(s) — one per box-sized pixel group — and
// the block appends them to the global tile list in one atomic; tiles whose
// every tap is zero padding are zero-filled here and never enter the list.
#ifndef CORR_PREP_THREADS
#define CORR_PREP_THREADS 128
#endif
constexpr int kPrepThreads = CORR_PREP_THREADS;
constexpr int kPrepEdges = kPrepThreads / kPix;  // 14 at 128 threads
constexpr int kPrepTiles = 2 * kPrepEdges;
__global__ void __launch_bounds__(kPrepThreads) corr_prep_kernel(CorrTmaParams a) {
    __shared__ double s_xy[kPrepEdges * kPix * 2];
    __shared__ int4 s_rec[kPrepTiles * kPix * 2];  // <= 9 pixel groups per tile
    __shared__ int s_zero[kPrepTiles];
    __shared__ int s_nrec, s_nzero, s_base;
    const int t = threadIdx.x;
    const int base = blockIdx.x * kPrepEdges;
    // the correlation launch that follows is a programmatic dependent: its CTAs
    // may set up as SMs free up and wait (griddepcontrol.wait) for this grid
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (t == 0) {
        s_nrec = 0;
        s_nzero = 0;
    }
    if (t < kPrepEdges * kPix) {
        const int pos = base + t / kPix, pix = t % kPix;
        if (pos < a.n_edges) {
            const int e = a.order ? a.order[pos] : pos;
            double xy[2];
            edge_pixel(a, e, pix, xy);
            s_xy[2 * t] = xy[0];
            s_xy[2 * t + 1] = xy[1];
            a.coords[(size_t)e * 18 + 2 * pix] = xy[0];
            a.coords[(size_t)e * 18 + 2 * pix + 1] = xy[1];
        }
    }
    __syncthreads();
    const int pos = base + (t >> 1), level = t & 1;
    if (t < kPrepTiles && pos < a.n_edges) {
        const int e = a.order ? a.order[pos] : pos;
        const double* xy = s_xy + (t >> 1) * kPix * 2;
        const double inv_scale = level ? 1.0 / 16.0 : 1.0 / 4.0;  // 1 / kFeatureStride^(level+1) (features.hpp:46)
        const int W = level ? a.w1 : a.w0, H = level ? a.h1 : a.h0;
        int fxs[kPix], fys[kPix];
        bool finite = true;
        int far = 0;  // pixels whose whole 8x8 tap window lies outside the grid: all 49 outputs are 0
#pragma unroll
        for (int p = 0; p < kPix; ++p) {
            const double x = xy[2 * p], y = xy[2 * p + 1];
            finite = finite && isfinite(x) && isfinite(y);
            fxs[p] = clamp_floor(x * inv_scale, W);  // x / 4 or x / 16, exact
            fys[p] = clamp_floor(y * inv_scale, H);
            if (fxs[p] + 4 < 0 || fxs[p] - 3 >= W || fys[p] + 4 < 0 || fys[p] - 3 >= H) far |= 1 << p;
        }
        const int fslot = a.e_slot ? a.e_slot[e] : a.pose_slot[a.e_pose[e]];
        const int grow = (a.e_patch[e] * 2 + level) * kPix;
        if (!finite) {
            atomicOr(a.status, 1 << kDevBadCoords);  // correlation.cpp:43-45
        } else if (far == kPixMask) {              // every tap of every pixel is zero padding
            s_zero[atomicAdd(&s_nzero, 1)] = e * 2 + level;
        } else {
            // Pixel groups that each fit one 9x9 box: a box at origin (X0, Y0) holds the
            // 8x8 window of pixel q iff fx_q - 3 in {X0, X0+1} and fy_q - 3 in {Y0, Y0+1}.
            // Greedy: seed = lowest remaining pixel; of the 4 boxes containing its window
            // take the one covering most remaining pixels.  Group 0 (usually the whole
            // tile) also zero-fills the far pixels.
            int rest = kPixMask & ~far;
            bool first = true;
            while (rest) {
                const int p0 = __ffs(rest) - 1;
                int best = 0, bx = 0, by = 0;
#pragma unroll
                for (int cand = 0; cand < 4; ++cand) {
                    const int X0 = fxs[p0] - 3 - (cand & 1), Y0 = fys[p0] - 3 - (cand >> 1);
                    int m = 0;
#pragma unroll
                    for (int q = 0; q < kPix; ++q) {
                        const int dx = fxs[q] - 3 - X0, dy = fys[q] - 3 - Y0;
                        if (((rest >> q) & 1) && (unsigned)dx <= 1u && (unsigned)dy <= 1u) m |= 1 << q;
                    }
                    if (__popc(m) > __popc(best)) {
                        best = m;
                        bx = X0;
                        by = Y0;
                    }
                }
                // narrow: every member's window is the same 8x8 block -> origin = that block
                int xl = 1 << 30, xh = -(1 << 30), yl = 1 << 30, yh = -(1 << 30);
#pragma unroll
                for (int q = 0; q < kPix; ++q)
                    if ((best >> q) & 1) {
                        xl = min(xl, fxs[q]);
                        xh = max(xh, fxs[q]);
                        yl = min(yl, fys[q]);
                        yh = max(yh, fys[q]);
                    }
                int code = kKindTma | (best << 17) | (first ? far << 8 : 0);
                if (xl == xh && yl == yh) {
                    code |= kNarrow;
                    bx = xl - 3;
                    by = yl - 3;
                }
                const int i = atomicAdd(&s_nrec, 1);
                s_rec[2 * i] = make_int4(bx, by, code, fslot);
                s_rec[2 * i + 1] = make_int4(grow, e, level, 0);
                first = false;
                rest &= ~best;
            }
        }
    }
    __syncthreads();
    if (t == 0) s_base = atomicAdd(a.ctl, s_nrec);  // < list capacity: at most 9 records per tile
    __syncthreads();
    int4* list = reinterpret_cast<int4*>(a.meta) + 2 * (size_t)s_base;
    for (int i = t; i < 2 * s_nrec; i += kPrepThreads) list[i] = s_rec[i];
    for (int z = t >> 5; z < s_nzero; z += kPrepThreads / 32) {  // a warp per zero tile, coalesced
        float* o = a.out + (size_t)s_zero[z] * kOut;
        for (int i = t & 31; i < kOut; i += 32) store_out(o + i, 0.f);
    }
}

__global__ void __launch_bounds__(kThreads, 1)
    corr_tma_kernel(const __grid_constant__ CUtensorMap feat0, const __grid_constant__ CUtensorMap feat1,
                    const __grid_constant__ CUtensorMap gram0, const __grid_constant__ CUtensorMap gram1,
                    const __grid_constant__ CUtensorMap patch, const __grid_constant__ CUtensorMap feat0n,
                    const __grid_constant__ CUtensorMap feat1n, CorrTmaParams a) {
    extern __shared__ unsigned char smem_raw[];
    // 1024-aligned base, derived by offset so the compiler keeps the shared address space
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t full[kWarps * kStages];
    __shared__ __align__(8) uint64_t hfull[kWarps];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid < kWarps * kStages) mbar_init(&full[tid], 1);
    if (tid < kWarps) mbar_init(&hfull[tid], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // launched as a programmatic dependent of the preparation grid: its tile
    // list, coordinates and zero fills are complete and visible after this
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    // one global tile list in processing order (target-frame sorted: the frames
    // in flight stay in L2)
    const int n_all = min(__ldcg(a.ctl), a.list_cap);

    // ================= per-warp pipeline =================
    unsigned char* wb = smem + warp * kWarpBytes;
    const uint32_t wbu = smem_u32(wb);                    // shared-window addresses, computed once
    const uint32_t baru = smem_u32(full + warp * kStages);  // stage s barrier: baru + 8 * s
    const uint32_t hbaru = smem_u32(hfull + warp);          // header barrier

    // issue cursor (warp-uniform): pending tile + its record, current tile, chunk.
    // Tiles come from the global queue; lane 0 keeps one claim in flight so the
    // atomic's latency hides behind a whole tile.
    // CORR_CLAIM consecutive tiles per atomic (A/B knob), the next claim kept in flight
    int pend = 0;
    int claim = 0;
    int cl_next = 0, cl_left = 0;  // warp-uniform: next tile of the current claim, tiles left in it
    if (lane == 0) claim = atomicAdd(a.ctl + 1, kClaim);
    int4 pr0 = make_int4(0, 0, 0, 0), pr1 = make_int4(0, 0, 0, 0);
    auto grab = [&]() {
        if (cl_left == 0) {
            cl_next = __shfl_sync(0xffffffffu, claim, 0);
            cl_left = kClaim;
            if (cl_next < n_all && lane == 0) claim = atomicAdd(a.ctl + 1, kClaim);
        }
        pend = cl_next++;
        --cl_left;
        if (pend < n_all) {
            const int4* src = reinterpret_cast<const int4*>(a.meta) + 2 * (size_t)pend;
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
        if (ichunk == kChunks) {  // advance to the next tile of the list
            if (pend >= n_all) {
                idone = true;
                return;
            }
            ir0 = pr0;
            ir1 = pr1;
            ichunk = 0;
            grab();
        }
        if (lane == 0) {
            const int level = ir1.z;
            const uint32_t bar = baru + 8 * is;
            const uint32_t st = wbu + is * kStageBytes;
            if (ichunk == 0) {
                int4* rec = reinterpret_cast<int4*>(wb + kMetaOff + 32 * (hi & 1));
                rec[0] = ir0;
                rec[1] = ir1;
            }
            const bool narrow = ir0.z & kNarrow;  // 8x8 box: the 64 cells the narrow variant reads
            mbar_expect_tx(bar, narrow ? kChunkTxNarrow : kChunkTx);
            tma_load_4d(st, narrow ? (level ? &feat1n : &feat0n) : (level ? &feat1 : &feat0), ichunk * kChunkCh,
                        ir0.x, ir0.y, ir0.w, bar);
            tma_load_2d(st + kChunkGOff, &patch, ichunk * kChunkCh, ir1.x, bar);
        }
        if (ichunk == 0) ++hi;
        ++ichunk;
        is = is == kStages - 1 ? 0 : is + 1;
    };
    // the tile header (Gram records + reprojected pixels) of tile hc, into the
    // warp's single header buffer: issued once the previous tile's epilogue is done
    auto issue_header = [&](int hc) {
        if (lane == 0) {
            const int4 r0 = *reinterpret_cast<const int4*>(wb + kMetaOff + 32 * (hc & 1));
            const int4 r1 = *reinterpret_cast<const int4*>(wb + kMetaOff + 32 * (hc & 1) + 16);
            const uint32_t hd = wbu + kHeaderOff;
            mbar_expect_tx(hbaru, kHeaderTx);
            // TMA needs a 16-byte aligned start in the innermost (x) dimension: start at
            // floor4(x0); the 12-wide box still covers x0 .. x0 + 8
            tma_load_4d(hd, r1.z ? &gram1 : &gram0, r0.x & ~3, r0.y, 0, r0.w, hbaru);
            bulk_load(hd + kGramBytes, a.coords + (size_t)r1.y * 18, kCoordBytes, hbaru);
        }
    };
    for (int k = 0; k < kStages; ++k) issue_one();
    __syncwarp();
    if (hi > 0) issue_header(0);

    float* dots = reinterpret_cast<float*>(wb + kDotsOff);
    int cs = 0;          // stage being consumed
    uint32_t cph = 0;    // its barrier phase parity
    // Dots <g_p, f_cell> of one tile, NC cells per lane: NC = 3 -> lanes 0..26 own
    // rows lane, lane+27, lane+54 of the 9x9 box (lanes 27..31 compute throwaway rows);
    // NC = 2 (narrow tile) -> lane owns cells (lane&7, lane>>3) and (lane&7, 4+(lane>>3))
    // of the 8x8 window at the box origin.  Results go to dots[p][box row].
    auto tile_dots = [&](auto nc_tag) {
        constexpr int NC = decltype(nc_tag)::value;
        int roff[NC], soff[NC];  // dots index (9-wide box rows) x 64; stage row offset (8-wide when narrow)
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            const int r = NC == 3 ? lane + 27 * k : ((lane >> 3) + 4 * k) * kBox + (lane & 7);
            const int rs = NC == 3 ? r : ((lane >> 3) + 4 * k) * 8 + (lane & 7);
            roff[k] = r * 64;
            soff[k] = rs * 64;
        }
        // (even, odd)-channel sums per (cell, pixel): packed FP32x2 FMAs (FFMA2)
        float2 acc[NC][kPix];
#pragma unroll
        for (int k = 0; k < NC; ++k)
#pragma unroll
            for (int p = 0; p < kPix; ++p) acc[k][p] = make_float2(0.f, 0.f);
        for (int c = 0; c < kChunks; ++c) {
            mbar_wait(baru + 8 * cs, cph);
            const unsigned char* st = wb + cs * kStageBytes;
            const float* g = reinterpret_cast<const float*>(st + kChunkGOff);
#if CORR_ACC == 2
            // pixel-outer: the chunk's 16 channels of the lane's cells stay in registers,
            // each (cell, pixel) sums its 16 channels in a short FFMA2 chain (8 terms per
            // component) and adds that once into the tile total — the accuracy of
            // per-chunk partials without holding a second [NC][9] accumulator set
            float4 v[NC][kChunkCh / 4];
#pragma unroll
            for (int k = 0; k < NC; ++k) {
                const int sw = (soff[k] >> 7) & 3;  // 64B swizzle: unit u of row r at u ^ ((r >> 1) & 3)
#pragma unroll
                for (int u = 0; u < kChunkCh / 4; ++u)
                    v[k][u] = *reinterpret_cast<const float4*>(st + soff[k] + ((u ^ sw) << 4));
            }
#pragma unroll
            for (int p = 0; p < kPix; ++p) {
                float4 gv[kChunkCh / 4];
#pragma unroll
                for (int u = 0; u < kChunkCh / 4; ++u) gv[u] = *reinterpret_cast<const float4*>(g + p * kChunkCh + 4 * u);
#pragma unroll
                for (int k = 0; k < NC; ++k) {
                    float2 t = __fmul2_rn(make_float2(v[k][0].x, v[k][0].y), make_float2(gv[0].x, gv[0].y));
                    t = __ffma2_rn(make_float2(v[k][0].z, v[k][0].w), make_float2(gv[0].z, gv[0].w), t);
#pragma unroll
                    for (int u = 1; u < kChunkCh / 4; ++u) {
                        t = __ffma2_rn(make_float2(v[k][u].x, v[k][u].y), make_float2(gv[u].x, gv[u].y), t);
                        t = __ffma2_rn(make_float2(v[k][u].z, v[k][u].w), make_float2(gv[u].z, gv[u].w), t);
                    }
                    acc[k][p] = __fadd2_rn(acc[k][p], t);
                }
            }
#else
#if CORR_ACC == 0
            float2 part[NC][kPix];  // per-chunk partials (r1): 8 + 8 terms per component
#endif
#pragma unroll
            for (int u = 0; u < kChunkCh / 4; ++u) {
                float4 v[NC], gv[kPix];
#pragma unroll
                for (int k = 0; k < NC; ++k) {
                    const int sw = (soff[k] >> 7) & 3;
                    v[k] = *reinterpret_cast<const float4*>(st + soff[k] + ((u ^ sw) << 4));
                }
#pragma unroll
                for (int p = 0; p < kPix; ++p) gv[p] = *reinterpret_cast<const float4*>(g + p * kChunkCh + 4 * u);
#if CORR_ACC == 1  // one chain per (cell, pixel, parity) over all 128 channels (64 terms)
#pragma unroll
                for (int k = 0; k < NC; ++k)
#pragma unroll
                    for (int p = 0; p < kPix; ++p)
                        acc[k][p] = __ffma2_rn(make_float2(v[k].x, v[k].y), make_float2(gv[p].x, gv[p].y), acc[k][p]);
#pragma unroll
                for (int k = 0; k < NC; ++k)
#pragma unroll
                    for (int p = 0; p < kPix; ++p)
                        acc[k][p] = __ffma2_rn(make_float2(v[k].z, v[k].w), make_float2(gv[p].z, gv[p].w), acc[k][p]);
#else
#pragma unroll
                for (int k = 0; k < NC; ++k)
#pragma unroll
                    for (int p = 0; p < kPix; ++p) {
                        const float2 va = make_float2(v[k].x, v[k].y), ga = make_float2(gv[p].x, gv[p].y);
                        part[k][p] = u == 0 ? __fmul2_rn(va, ga) : __ffma2_rn(va, ga, part[k][p]);
                    }
#pragma unroll
                for (int k = 0; k < NC; ++k)
#pragma unroll
                    for (int p = 0; p < kPix; ++p)
                        part[k][p] = __ffma2_rn(make_float2(v[k].z, v[k].w), make_float2(gv[p].z, gv[p].w), part[k][p]);
#endif
            }
#if CORR_ACC == 0
#pragma unroll
            for (int k = 0; k < NC; ++k)
#pragma unroll
                for (int p = 0; p < kPix; ++p) acc[k][p] = __fadd2_rn(acc[k][p], part[k][p]);
#endif
#endif
            __syncwarp();  // every lane is done with this stage: refill it
            if (++cs == kStages) {
                cs = 0;
                cph ^= 1;
            }
            issue_one();
        }
        if (NC == 2 || lane < 27) {
#pragma unroll
            for (int k = 0; k < NC; ++k)
#pragma unroll
                for (int p = 0; p < kPix; ++p) dots[p * kCells + (roff[k] >> 6)] = acc[k][p].x + acc[k][p].y;
        }
    };
    for (int hc = 0; hc < hi; ++hc) {
        const int hb = hc & 1;
        const int4 r0 = *reinterpret_cast<const int4*>(wb + kMetaOff + 32 * hb);
        const int4 r1 = *reinterpret_cast<const int4*>(wb + kMetaOff + 32 * hb + 16);
        if (r0.z & kNarrow)
            tile_dots(std::integral_constant<int, 2>{});
        else
            tile_dots(std::integral_constant<int, 3>{});

        // ---- epilogue ----
        mbar_wait(hbaru, hc & 1);
        const unsigned char* hd = wb + kHeaderOff;
        const float* gram = reinterpret_cast<const float*>(hd) + (r0.x & 3);  // box starts at floor4(x0)
        const double* tc = reinterpret_cast<const double*>(hd + kGramBytes);
        const int e = r1.y, level = r1.z, far = (r0.z >> 8) & kPixMask, member = (r0.z >> 17) & kPixMask;
        __syncwarp();
        // Separable bilinear recombination (correlation.cpp:8-23 regrouped): lane owns
        // the output column (pixel p, offset beta) and walks alpha = 0..6, carrying the
        // x-interpolated row terms of row alpha + 1 into the next step:
        //   fx(y)   = (1-ax) f[y][x] + ax f[y][x+1]
        //   dot     = (1-ay) <g, fx(y)> + ay <g, fx(y+1)>
        //   |f(x)|^2 = (1-ay)^2 |fx(y)|^2 + ay^2 |fx(y+1)|^2 + 2 ay (1-ay) <fx(y), fx(y+1)>
        // with |fx|^2 and <fx(y), fx(y+1)> from the Gram records (|f|^2, right, down,
        // diag, anti).  ax / ay are the reference's per-offset fractional parts (FP64).
        // per-pixel fractional offsets, computed once per tile (not per column):
        // ax[p][beta] = (bx + (beta-3)) - floor(...), ay[p][alpha] likewise, in FP64
        // exactly as the reference (features.cpp:10-13); 1/4 and 1/16 are exact
        const double inv_scale = level ? 1.0 / 16.0 : 1.0 / 4.0;  // kFeatureStride (features.hpp:46)
        const int W = level ? a.w1 : a.w0, H = level ? a.h1 : a.h0;
        float* s_ax = reinterpret_cast<float*>(wb + kPixOff);  // [9][7]
        float* s_ay = s_ax + kPix * 7;                          // [9][7]
        int* s_f = reinterpret_cast<int*>(s_ay + kPix * 7);     // [9][2] floor(bx), floor(by)
        for (int t = lane; t < kPix * 7; t += 32) {
            const int p = (t * 37) >> 8, q = t - 7 * p;
            const double bx = tc[2 * p] * inv_scale, by = tc[2 * p + 1] * inv_scale;
            const int fx = clamp_floor(bx, W), fy = clamp_floor(by, H);
            s_ax[t] = (float)((bx + (double)(q - 3)) - (double)(fx + q - 3));
            s_ay[t] = (float)((by + (double)(q - 3)) - (double)(fy + q - 3));
            if (q == 0) {
                s_f[2 * p] = fx;
                s_f[2 * p + 1] = fy;
            }
        }
        __syncwarp();
        float* out = a.out + ((size_t)e * 2 + level) * kOut;
        unsigned exact = 0;  // outputs to re-evaluate directly: bit 7 * (col >= 32) + alpha
#pragma unroll 1
        for (int col = lane; col < kPix * 7; col += 32) {
            const int p = (col * 37) >> 8, beta = col - 7 * p;  // col / 7 for col < 63
            float* o = out + p * 49 + beta;
            if (!((member >> p) & 1)) {
                if ((far >> p) & 1) {  // every tap of this pixel is zero padding
#pragma unroll
                    for (int alpha = 0; alpha < 7; ++alpha) store_out(o + alpha * 7, 0.f);
                }
                continue;  // else: another sub-tile of this (edge, level) writes it
            }
            const int fx = s_f[2 * p], fy = s_f[2 * p + 1];
            const float ax = s_ax[col];
            const float bx0 = 1.f - ax;
            const int cx = fx - 3 - r0.x + beta, cy = fy - 3 - r0.y;
            const float* d = dots + p * kCells + cy * kBox + cx;
            const float* G = gram + cy * kGramW + cx;
            const float qa = bx0 * bx0, qb = ax * ax, qc = 2.f * ax * bx0, qd = ax * bx0;
            // row terms of row y: <g, fx(y)>, |fx(y)|^2 and its diagonal part
            // sum_x w_x^2 |f(y, x)|^2 (the cancellation check's scale)
            float dA = fmaf(ax, d[1], bx0 * d[0]);
            float sA = fmaf(qb, G[1], qa * G[0]);
            float nA = fmaf(qc, G[kGramPlane], sA);
            const int ebit = col >= 32 ? 7 : 0;
#pragma unroll
            for (int alpha = 0; alpha < 7; ++alpha) {
                const float* dn = d + (alpha + 1) * kBox;
                const float* Gn = G + (alpha + 1) * kGramW;
                const float* Gc = G + alpha * kGramW;
                const float dB = fmaf(ax, dn[1], bx0 * dn[0]);
                const float sB = fmaf(qb, Gn[1], qa * Gn[0]);
                const float nB = fmaf(qc, Gn[kGramPlane], sB);
                // <fx(y), fx(y+1)> = (1-ax)^2 down[x] + ax^2 down[x+1] + ax(1-ax) (diag[x] + anti[x])
                const float cr = fmaf(qd, Gc[3 * kGramPlane] + Gc[4 * kGramPlane],
                                      fmaf(qb, Gc[2 * kGramPlane + 1], qa * Gc[2 * kGramPlane]));
                const float ay = s_ay[p * 7 + alpha];
                const float by0 = 1.f - ay;
                const float dot = fmaf(ay, dB, by0 * dA);
                const float wa = by0 * by0, wb = ay * ay;
                const float n2 = fmaf(2.f * ay * by0, cr, fmaf(wb, nB, wa * nA));
                if (corr_needs_exact(n2, fmaf(wb, sB, wa * sA)))
                    exact |= 1u << (ebit + alpha);  // written once, by the re-evaluation below
                else
                    store_out(o + alpha * 7, n2 > 1e-12f ? dot * rsqrt_approx(n2) : 0.f);  // correlation.cpp:22
                dA = dB;
                nA = nB;
                sA = sB;
            }
        }
        // cancelling taps: the warp re-evaluates those outputs the reference's way
        // (corr_exact.cuh); rare on real features, so the common path stays FP32
        unsigned todo = __ballot_sync(0xffffffffu, exact != 0);
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            unsigned m = __shfl_sync(0xffffffffu, exact, src);
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                const int col = src + (b >= 7 ? 32 : 0), alpha = b >= 7 ? b - 7 : b;
                const int p = (col * 37) >> 8, beta = col - 7 * p;
                const double x = tc[2 * p] * inv_scale + (double)(beta - 3);
                const double y = tc[2 * p + 1] * inv_scale + (double)(alpha - 3);
                const float* fr = (level ? a.feat1 : a.feat0) + (size_t)r0.w * W * H * kD;
                const float v = corr_exact_warp(a.patch_feats + (size_t)(r1.x + p) * kD, fr, W, H, kD, x, y);
                if (lane == 0) store_out(out + p * 49 + alpha * 7 + beta, v);
            }
        }
        __syncwarp();  // dots and the header are rewritten by the next tile
        if (hc + 1 < hi) issue_header(hc + 1);
    }
    // the last warp to finish leaves the queue words zero for the next launch
    if (lane == 0) {
        __threadfence();
        if (atomicAdd(a.ctl + 2, 1) == (int)gridDim.x * kWarps - 1) {
            a.ctl[0] = 0;
            a.ctl[1] = 0;
            a.ctl[2] = 0;
        }
    }
}

}  // namespace

int corr_tma_smem_bytes() { return kSmemBytes; }
int corr_tma_grid(int n_edges, int num_sms) { return n_edges < num_sms ? n_edges : num_sms; }
// worst case: every pixel of every tile in its own box -> 9 records per tile
int corr_tma_list_cap(int n_edges) { return 2 * kPix * n_edges; }

cudaError_t launch_corr_tma(const CorrTmaParams& p, const CUtensorMap* maps, int num_sms, cudaStream_t stream) {
    if (p.n_edges <= 0) return cudaSuccess;
    cudaError_t err = cudaFuncSetAttribute(corr_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (err != cudaSuccess) return err;
    const int grid = corr_tma_grid(p.n_edges, num_sms);
    if (p.list_cap < corr_tma_list_cap(p.n_edges) || !p.ctl) return cudaErrorInvalidValue;
    corr_prep_kernel<<<(p.n_edges + kPrepEdges - 1) / kPrepEdges, kPrepThreads, 0, stream>>>(p);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    err = cudaLaunchKernelEx(&cfg, corr_tma_kernel, maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], maps[6], p);
    if (err != cudaSuccess) return err;
    return cudaGetLastError();
}

}  // namespace pvo_dev
