// capi_common.hpp — host-side state and helpers shared by the capi_*.cu
// translation units of the extern "C" boundary (include/pvo_capi.h): the
// context (device, streams, frame store, TMA descriptors, scratch), the
// resident window / batch state, problem staging and kernel dispatch.
// The host code only validates, flattens and moves memory; every numeric
// result comes from the sm_100a kernels.  There is no CPU compute fallback.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "geometry.cuh"
#include "internal.hpp"
#include "kernels.cuh"

using namespace pvo_host;

struct BABuffers {
    DevBuf poses, free_slot, patch_src, px, py, depth, depth_slot, edge_begin, e_patch, e_pose, e_in, e_w, e_target,
        e_weight, cand_poses, cand_depth, patch_v, patch_h, patch_bd, partials, system, delta, norms, n_norms, dbg_h,
        dbg_b, K, status2, attempts, clocks;
    // large-window path (ba_large.cu)
    DevBuf g_begin, g_lo, g_nl, g_off, patch_group, g_part, g_res, A, mats, cmats, u_res, ctrl;
    void release() {
        DevBuf* all[] = {&poses,    &free_slot,  &patch_src, &px,        &py,       &depth,    &depth_slot,
                         &edge_begin, &e_patch,  &e_pose,    &e_in,      &e_w,      &e_target, &e_weight,
                         &cand_poses, &cand_depth, &patch_v, &patch_h,   &patch_bd, &partials, &system,
                         &delta,    &norms,      &n_norms,   &dbg_h,     &dbg_b,    &K,        &status2,
                         &attempts, &clocks,     &g_begin,   &g_lo,      &g_nl,     &g_off,    &patch_group,
                         &g_part,   &g_res,      &A,         &mats,      &cmats,    &u_res,    &ctrl};
        for (DevBuf* b : all) b->release();
    }
};

struct LogEntryHost {
    int removed = -1, anchor = -1;
    double relative[7];
    double ts = 0;
};

// Host-side plan of a flattened problem (edges grouped by patch).
struct Plan {
    int n_free_poses = 0, n_free_depths = 0;
    std::vector<int> free_slot, depth_slot, edge_begin, perm;  // perm: sorted edge -> input edge
    bool sorted = true;
    // large pose systems (> 16 free poses or > 128 poses): multi-kernel path (ba_large.cu)
    bool large = false;
    std::vector<int> g_begin, g_lo, g_nl, patch_group;
    std::vector<long long> g_off;
    long long g_part_doubles = 0;
    int max_nl = 0, bw = 0;
};

// Patch groups of the large path: runs of consecutive patches with one source
// pose, cut to <= 64 patches; the window of a run = the free pose slots its
// patches touch (source + edge targets).  The reduced system's half-bandwidth
// is the widest window - 1 (patch_graph.cpp:79 keeps edges within the radius).
#ifndef PVO_GROUP_PATCHES
#define PVO_GROUP_PATCHES 64
#endif
inline void plan_groups(const HostProblem& pr, Plan& pl) {
    constexpr int kGroupPatches = PVO_GROUP_PATCHES;  // A/B knob (assemble CTAs per run)
    pl.g_begin.assign(1, 0);
    pl.patch_group.assign(pr.n_patches, 0);
    int k = 0;
    while (k < pr.n_patches) {
        int r1 = k;
        while (r1 < pr.n_patches && pr.src[r1] == pr.src[k]) ++r1;
        int lo = 1 << 30, hi = -1;
        auto touch = [&](int pose) {
            const int f = pl.free_slot[pose];
            if (f >= 0) {
                lo = std::min(lo, f);
                hi = std::max(hi, f);
            }
        };
        for (int q = k; q < r1; ++q) {
            touch(pr.src[q]);
            for (int i = pl.edge_begin[q]; i < pl.edge_begin[q + 1]; ++i) touch(pr.e_pose[pl.perm[i]]);
        }
        const int nposes = hi >= lo ? hi - lo + 1 : 0;
        if (nposes > pvo_dev::kMaxLocalPoses) {
            fail(PVO_UNSUPPORTED, "ba: a patch run touches " + std::to_string(nposes) + " free poses (max " +
                                      std::to_string(pvo_dev::kMaxLocalPoses) + ")");
        }
        for (int c = k; c < r1; c += kGroupPatches) {
            const int c1 = std::min(r1, c + kGroupPatches);
            const int g = (int)pl.g_lo.size();
            for (int q = c; q < c1; ++q) pl.patch_group[q] = g;
            pl.g_begin.push_back(c1);
            pl.g_lo.push_back(nposes ? lo : 0);
            pl.g_nl.push_back(6 * nposes);
            pl.g_off.push_back(pl.g_part_doubles);
            const long long nl = 6 * nposes;
            pl.g_part_doubles += nl * (nl + 1) / 2 + nl;
            pl.max_nl = std::max(pl.max_nl, (int)nl);
        }
        k = r1;
    }
    pl.bw = pl.max_nl > 0 ? pl.max_nl - 1 : 0;
}

struct Window {
    bool loaded = false;
    int n_poses = 0, n_patches = 0, n_edges = 0;
    Plan plan;
    HostProblem shape;  // sizes, K, image size (pointers unused)
    DevBuf pose_slot, patch_feats, corr, init_poses, init_depth, order, flags;
    // host-loaded windows: the processing order of each half of the edge range
    // (edges [0, half) then [half, E)), so a host read-back of the volume can
    // start on the first half while the second is correlated (0: no split)
    DevBuf order_half;
    int half = 0;
};

// Batch of independent windows (config 5: many sequences per device).  All
// windows are concatenated into one set of arrays (window-local indices for
// the BA, global indices for the correlation); one correlation launch covers
// every edge and one batched BA launch runs a CTA per window.
struct Batch {
    bool loaded = false;
    int n_windows = 0, n_poses = 0, n_patches = 0, n_edges = 0, max_free = 0, max_poses = 0;
    int iterations = -1;
    double damping = 0.0;
    std::vector<int> pose_off, patch_off, edge_off;
    std::vector<pvo_dev::BAParams> hparams;
    static constexpr int kNormStride = 66;
    DevBuf poses, free_slot, src, px, py, depth, depth_slot, edge_begin, e_patch, e_pose, e_in, e_w, e_target,
        e_weight, cand_poses, cand_depth, patch_v, patch_h, patch_bd, partials, system, delta, norms, n_norms,
        status2, attempts, status, K, g_e_patch, g_e_pose, g_src, pose_slot, order, patch_feats, corr, params,
        init_poses, init_depth;
    // windows beyond 16 free poses / 128 poses: run one after another on the large-window
    // BA (ba_large.cu) with their own plans; the other windows share the batched kernel
    std::vector<int> large_idx;
    std::vector<Plan> large_plans;
    std::vector<pvo_dev::BAParams> small_params;
    int n_small = 0;
    BABuffers lb;  // the large windows' group arrays and scratch
    void release() {
        lb.release();
        DevBuf* all[] = {&poses,     &free_slot, &src,        &px,        &py,         &depth,     &depth_slot,
                         &edge_begin, &e_patch,  &e_pose,     &e_in,      &e_w,        &e_target,  &e_weight,
                         &cand_poses, &cand_depth, &patch_v,  &patch_h,   &patch_bd,   &partials,  &system,
                         &delta,     &norms,     &n_norms,    &status2,   &attempts,   &status,    &K,
                         &g_e_patch, &g_e_pose,  &g_src,      &pose_slot, &order,      &patch_feats, &corr,
                         &params,    &init_poses, &init_depth};
        for (DevBuf* b : all) b->release();
    }
};

// A host feature grid mirrored on the device (the reference-signature calls
// pvo_correlate / pvo_correlate_points take host FeatureGrids).  Keyed by the
// host address, shape and a fingerprint of sampled contents: the reference's
// providers build each pyramid once and never modify it (flow_provider.cpp
// add_frame), so a pyramid is uploaded (and its Gram terms derived) once
// instead of on every call.  LRU within a byte budget (PVO_GRID_CACHE_MB).
struct GridEntry {
    const void* host = nullptr;
    int w = 0, h = 0, C = 0;
    uint64_t fp = 0;
    DevBuf feat, gram;
    bool has_gram = false;
    uint64_t tick = 0;
    size_t bytes = 0;
};

struct pvo_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int num_sms = 0;
    int64_t launches = 0;
    int* d_status = nullptr;
    // frame store
    int nf = 0, w0 = 0, h0 = 0, w1 = 0, h1 = 0, C = 0;
    DevBuf feat0, feat1, gram0, gram1;
    // direct-op scratch
    DevBuf s0, s1, s2, s3, s4, s5, s6, s7, s8;
    // TMA descriptors of the frame store (feat0, feat1, gram0, gram1) and the
    // production correlation kernel's scratch
    CUtensorMap maps[7];  // feat0, feat1, gram0, gram1, patch descriptors (per call), feat0/feat1 8x8 boxes
    bool maps_ok = false;
    const void* patch_map_base = nullptr;
    int patch_map_rows = 0;
    DevBuf c_coords, c_meta, c_over, c_order;
    BABuffers ba;
    Window win;
    Batch bat;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    // copy stream: device->host read-back of the correlation volume overlaps the BA kernels
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_corr = nullptr, ev_copy = nullptr, ev_corr2 = nullptr;
    bool timing_pending = false;
    bool tracing = false;  // record BA phase clocks (pvo_ctx_set_tracing)
    bool timing = true;    // record the per-iteration timing events (pvo_ctx_set_timing)
    // FP64 neighbour-Gram maps of the frame store for the provider measurement
    // ([slot][H][W][kGram25] per level, launch_gram25), derived lazily per slot
    DevBuf g25_0, g25_1;
    std::vector<uint8_t> g25_valid;
    DevBuf replay;  // the measurement's exact-replay list (kept zeroed by the kernels)
    std::vector<GridEntry*> grids;  // host-grid cache (GridEntry above)
    uint64_t grid_tick = 0;
    size_t grid_bytes = 0;
    int64_t grid_hits = 0, grid_misses = 0;
    std::mt19937_64 oracle_rng{0};  // the oracle provider's RNG (flow_provider.cpp:10, rng_(noise.seed))
    int* d_corr_ctl = nullptr;      // correlation tile queue: [list length, queue head, warps done, -]
    void* h_stage = nullptr;        // page-locked staging for small read-backs (async copies, one sync)
    size_t h_stage_cap = 0;
    void* stage(size_t bytes) {
        if (bytes > h_stage_cap) {
            // same headroom policy as DevBuf::get: page-locking is the costliest allocation
            if (h_stage_cap)
                bytes = std::max(bytes, std::min(h_stage_cap + h_stage_cap / 2, bytes + (size_t(256) << 20)));
            const auto t0 = std::chrono::steady_clock::now();
            if (h_stage) cudaFreeHost(h_stage);
            h_stage = nullptr;
            const size_t old = h_stage_cap;
            h_stage_cap = 0;
            cuda_check(cudaMallocHost(&h_stage, bytes), "cudaMallocHost");
            h_stage_cap = bytes;
            if (pvo_host::DevBuf::trace_alloc())
                std::fprintf(stderr, "[pvo alloc] pinned staging %zu -> %zu bytes, %.3f ms\n", old, bytes,
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        }
        return h_stage;
    }
};

namespace pvo_host {

inline void bind(pvo_ctx* ctx) {
    if (!ctx) fail(PVO_INVALID_ARGUMENT, "null context");
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
}

template <typename T>
inline T* upload(pvo_ctx* ctx, DevBuf& buf, const T* host, size_t count) {
    T* d = buf.as<T>(count);
    if (count) cuda_check(cudaMemcpyAsync(d, host, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    return d;
}
template <typename T>
inline void download(pvo_ctx* ctx, T* host, const T* dev, size_t count) {
    if (count) cuda_check(cudaMemcpyAsync(host, dev, count * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
}
inline void sync(pvo_ctx* ctx) { cuda_check(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize"); }
// The per-iteration timing events (pvo_ctx_last_timing).  Under stream capture
// they are recorded as external event nodes, so a graph replay records them too.
inline void record_timing(pvo_ctx* ctx, int i) {
    if (!ctx->timing) return;
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cuda_check(cudaStreamIsCapturing(ctx->stream, &st), "cudaStreamIsCapturing");
    cuda_check(cudaEventRecordWithFlags(ctx->ev[i], ctx->stream,
                                        st == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0),
               "event");
}
// Page-locked (or registered) host memory: an async copy from it is still in
// flight when the call returns, so calls that read such caller buffers sync
// before returning (pageable sources are staged by the copy itself).
inline bool host_pinned(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

inline void reset_status(pvo_ctx* ctx) {
    cuda_check(cudaMemsetAsync(ctx->d_status, 0, sizeof(int), ctx->stream), "status reset");
}
inline int read_status(pvo_ctx* ctx) {
    int s = 0;
    cuda_check(cudaMemcpyAsync(&s, ctx->d_status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "status");
    sync(ctx);
    return s;
}
// BA status bits -> the reference's exception (bundle_adjust.cpp:65-92, :147-149).
inline void raise_ba_status(int s) {
    if (!s) return;
    using namespace pvo_dev;
    if (s & (1 << kDevNonFiniteResidual)) fail(PVO_DEGENERATE, "ba: non-finite residual");
    if (s & (1 << kDevNonPositiveDepth)) fail(PVO_DEGENERATE, "schur: non-positive damped depth-block entry");
    if (s & (1 << kDevFactorization)) fail(PVO_DEGENERATE, "schur: reduced camera system factorization failed");
    if (s & (1 << kDevNonFinitePose)) fail(PVO_DEGENERATE, "schur: non-finite pose update");
    if (s & (1 << kDevNonFiniteDepth)) fail(PVO_DEGENERATE, "schur: non-finite depth update");
    fail(PVO_CUDA_ERROR, "unknown device status");
}

inline bool finite2(const double* v) { return std::isfinite(v[0]) && std::isfinite(v[1]); }

// BAProblem::validate (bundle_adjust.cpp:11-36).
inline void validate(const HostProblem& pr) {
    if (pr.n_poses < 0 || pr.n_patches < 0 || pr.n_edges < 0) fail(PVO_INVALID_ARGUMENT, "ba: negative size");
    for (int e = 0; e < pr.n_edges; ++e) {
        if (pr.e_patch[e] < 0 || pr.e_patch[e] >= pr.n_patches || pr.e_pose[e] < 0 || pr.e_pose[e] >= pr.n_poses) {
            fail(PVO_INVALID_ARGUMENT, "ba: edge references an unknown patch or pose");
        }
        if (!finite2(pr.e_in + 2 * e)) fail(PVO_INVALID_ARGUMENT, "ba: non-finite edge target");
        const double wx = pr.e_w[2 * e], wy = pr.e_w[2 * e + 1];
        if (wx < 0 || wx >= 1 || wy < 0 || wy >= 1) fail(PVO_INVALID_ARGUMENT, "ba: edge weights must lie in [0, 1)");
    }
    for (int k = 0; k < pr.n_patches; ++k) {
        if (pr.src[k] < 0 || pr.src[k] >= pr.n_poses) fail(PVO_INVALID_ARGUMENT, "ba: patch source pose out of range");
    }
}

inline Plan make_plan(const HostProblem& pr, bool all_fixed) {
    Plan pl;
    pl.free_slot.assign(pr.n_poses, -1);
    for (int i = 0; i < pr.n_poses; ++i)
        if (!all_fixed && !pr.fixed[i]) pl.free_slot[i] = pl.n_free_poses++;
    pl.depth_slot.assign(pr.n_patches, -1);
    for (int k = 0; k < pr.n_patches; ++k)
        if (!pr.depth_free || pr.depth_free[k]) pl.depth_slot[k] = pl.n_free_depths++;
    // group edges by patch (stable): the kernel runs a warp per patch
    std::vector<int> count(pr.n_patches + 1, 0);
    for (int e = 0; e < pr.n_edges; ++e) count[pr.e_patch[e] + 1]++;
    pl.edge_begin.assign(pr.n_patches + 1, 0);
    for (int k = 0; k < pr.n_patches; ++k) pl.edge_begin[k + 1] = pl.edge_begin[k] + count[k + 1];
    std::vector<int> fill(pl.edge_begin.begin(), pl.edge_begin.end() - 1);
    pl.perm.assign(pr.n_edges, 0);
    for (int e = 0; e < pr.n_edges; ++e) {
        const int pos = fill[pr.e_patch[e]]++;
        pl.perm[pos] = e;
        if (pos != e) pl.sorted = false;
    }
    int max_edges = 0;
    for (int k = 0; k < pr.n_patches; ++k) max_edges = std::max(max_edges, pl.edge_begin[k + 1] - pl.edge_begin[k]);
    if (max_edges > pvo_dev::ba_max_edges_per_patch()) {
        fail(PVO_UNSUPPORTED, "ba: more than " + std::to_string(pvo_dev::ba_max_edges_per_patch()) +
                                  " edges on one patch");
    }
    if (pr.p != 3) fail(PVO_UNSUPPORTED, "ba: the kernels implement 3x3 patches");
    pl.large = pl.n_free_poses > pvo_dev::ba_max_free_poses() || pr.n_poses > pvo_dev::ba_max_poses();
    if (std::getenv("PVO_BA_LARGE")) pl.large = true;  // testing: force the multi-kernel path
    if (pl.large) plan_groups(pr, pl);
    return pl;
}

// Upload the problem into ctx->ba and fill the kernel parameter block.
inline pvo_dev::BAParams stage_problem(pvo_ctx* ctx, const HostProblem& pr, const Plan& pl, int extra_norms) {
    BABuffers& B = ctx->ba;
    const int pp = pr.p * pr.p;
    pvo_dev::BAParams a;
    a.n_poses = pr.n_poses;
    a.n_patches = pr.n_patches;
    a.n_edges = pr.n_edges;
    a.n_free_poses = pl.n_free_poses;
    a.n_free_depths = pl.n_free_depths;
    // the plan's host vectors go through the context's page-locked staging (async
    // copies; every caller synchronises before it returns)
    const size_t nfs = pl.free_slot.size(), nds = pl.depth_slot.size(), neb = pl.edge_begin.size();
    int* stg = static_cast<int*>(ctx->stage(sizeof(int) * (nfs + nds + neb)));
    std::memcpy(stg, pl.free_slot.data(), sizeof(int) * nfs);
    std::memcpy(stg + nfs, pl.depth_slot.data(), sizeof(int) * nds);
    std::memcpy(stg + nfs + nds, pl.edge_begin.data(), sizeof(int) * neb);
    a.poses = upload(ctx, B.poses, pr.poses, (size_t)pr.n_poses * 7);
    a.pose_free_slot = upload(ctx, B.free_slot, static_cast<const int*>(stg), nfs);
    a.patch_src = upload(ctx, B.patch_src, pr.src, pr.n_patches);
    a.patch_x = upload(ctx, B.px, pr.px, (size_t)pr.n_patches * pp);
    a.patch_y = upload(ctx, B.py, pr.py, (size_t)pr.n_patches * pp);
    a.depth = upload(ctx, B.depth, pr.depth, pr.n_patches);
    a.depth_slot = upload(ctx, B.depth_slot, static_cast<const int*>(stg + nfs), nds);
    a.patch_edge_begin = upload(ctx, B.edge_begin, static_cast<const int*>(stg + nfs + nds), neb);
    if (pl.sorted) {
        a.e_patch = upload(ctx, B.e_patch, pr.e_patch, pr.n_edges);
        a.e_pose = upload(ctx, B.e_pose, pr.e_pose, pr.n_edges);
        a.e_in = upload(ctx, B.e_in, pr.e_in, (size_t)pr.n_edges * 2);
        a.e_weight_in = upload(ctx, B.e_w, pr.e_w, (size_t)pr.n_edges * 2);
    } else {
        std::vector<int> ep(pr.n_edges), eo(pr.n_edges);
        std::vector<double> ein(2 * (size_t)pr.n_edges), ew(2 * (size_t)pr.n_edges);
        for (int i = 0; i < pr.n_edges; ++i) {
            const int e = pl.perm[i];
            ep[i] = pr.e_patch[e];
            eo[i] = pr.e_pose[e];
            ein[2 * i] = pr.e_in[2 * e];
            ein[2 * i + 1] = pr.e_in[2 * e + 1];
            ew[2 * i] = pr.e_w[2 * e];
            ew[2 * i + 1] = pr.e_w[2 * e + 1];
        }
        a.e_patch = upload(ctx, B.e_patch, ep.data(), ep.size());
        a.e_pose = upload(ctx, B.e_pose, eo.data(), eo.size());
        a.e_in = upload(ctx, B.e_in, ein.data(), ein.size());
        a.e_weight_in = upload(ctx, B.e_w, ew.data(), ew.size());
        sync(ctx);  // the temporaries die here
    }
    const int np = 6 * pl.n_free_poses;
    a.e_target = B.e_target.as<double>((size_t)pr.n_edges * 2);
    a.e_weight = B.e_weight.as<double>((size_t)pr.n_edges * 2);
    a.cand_poses = B.cand_poses.as<double>((size_t)pr.n_poses * 7);
    a.cand_depth = B.cand_depth.as<double>(pr.n_patches);
    a.patch_v = B.patch_v.as<double>((size_t)pr.n_patches * std::max(np, 1));
    a.patch_h = B.patch_h.as<double>(pr.n_patches);
    a.patch_bd = B.patch_bd.as<double>(pr.n_patches);
    if (pl.large) {
        upload(ctx, B.g_begin, pl.g_begin.data(), pl.g_begin.size());
        upload(ctx, B.g_lo, pl.g_lo.data(), pl.g_lo.size());
        upload(ctx, B.g_nl, pl.g_nl.data(), pl.g_nl.size());
        upload(ctx, B.g_off, pl.g_off.data(), pl.g_off.size());
        upload(ctx, B.patch_group, pl.patch_group.data(), pl.patch_group.size());
    }
    a.status2 = B.status2.as<int>(2);
    a.attempts = B.attempts.as<int>(1);
    a.phase_clocks = ctx->tracing ? B.clocks.as<long long>(128) : nullptr;
    if (!pl.large) {
        const int grid = pvo_dev::ba_grid_size(pr.n_patches, pl.n_free_poses, pr.n_poses, ctx->num_sms);
        a.partials = B.partials.as<double>(pvo_dev::ba_partials_doubles(pl.n_free_poses, grid));
        a.system = B.system.as<double>((size_t)np * (np + 1) / 2 + np + 1);
    }
    a.delta = B.delta.as<double>(std::max(np, 1));
    a.residual_norms = B.norms.as<double>(2 + extra_norms);
    a.n_norms = B.n_norms.as<int>(1);
    a.status = ctx->d_status;
    std::memcpy(a.K, pr.K, sizeof(a.K));
    a.image_w = pr.image_w;
    a.image_h = pr.image_h;
    a.damping = pr.damping;
    return a;
}

// Large-window parameter block over the context's buffers (groups uploaded by stage_problem).
inline pvo_dev::BALargeParams large_params(pvo_ctx* ctx, const pvo_dev::BAParams& a, const Plan& pl,
                                           BABuffers* bufs = nullptr) {
    BABuffers& B = bufs ? *bufs : ctx->ba;
    pvo_dev::BALargeParams p;
    p.a = a;
    const int np = 6 * pl.n_free_poses;
    p.a.patch_v = nullptr;
    p.n_groups = (int)pl.g_lo.size();
    p.g_begin = static_cast<const int*>(B.g_begin.p);
    p.g_lo = static_cast<const int*>(B.g_lo.p);
    p.g_nl = static_cast<const int*>(B.g_nl.p);
    p.g_off = static_cast<const long long*>(B.g_off.p);
    p.patch_group = static_cast<const int*>(B.patch_group.p);
    p.max_nl = pl.max_nl;
    p.bw = pl.bw;
    p.g_part = B.g_part.as<double>((size_t)std::max<long long>(1, pl.g_part_doubles));
    p.g_res = B.g_res.as<double>(2 * (size_t)std::max(1, p.n_groups));
    p.patch_vl = B.patch_v.as<double>((size_t)a.n_patches * std::max(1, pl.max_nl));
    p.A = B.A.as<double>((size_t)(np + 1) * (np + 1));
    p.mats = B.mats.as<double>(12 * (size_t)a.n_poses);
    p.cmats = B.cmats.as<double>(12 * (size_t)a.n_poses);
    p.n_update_ctas = std::max(1, std::min(2 * ctx->num_sms, (a.n_patches + 7) / 8));
    p.u_res = B.u_res.as<double>(2 * (size_t)p.n_update_ctas);
    p.ctrl = B.ctrl.as<int>(4);
    return p;
}

// bufs: the large path's group arrays / scratch (default: the resident window's)
inline void launch_ba_checked(pvo_ctx* ctx, pvo_dev::BAParams& a, const Plan& pl, BABuffers* bufs = nullptr) {
    NvtxRange range(pl.large ? "ba_large" : "ba");
    cuda_check(cudaMemsetAsync(a.n_norms, 0, sizeof(int), ctx->stream), "memset");
    if (pl.large) {
        if (a.gn_step_mode) fail(PVO_UNSUPPORTED, "gauss_newton_step: pose systems beyond 16 free poses");
        cuda_check(cudaMemsetAsync(a.attempts, 0, sizeof(int), ctx->stream), "memset");
        pvo_dev::BALargeParams p = large_params(ctx, a, pl, bufs);
        const char* dump = std::getenv("PVO_BA_LARGE_DUMP");
        const int np = 6 * pl.n_free_poses;
        if (dump) p.dbg_A = ctx->ba.dbg_h.as<double>((size_t)(np + 1) * (np + 1));
        int n = 0;
        cuda_check(pvo_dev::launch_ba_large(p, ctx->num_sms, ctx->stream, &n), "ba large kernels");
        ctx->launches += n;
        if (dump) {
            std::vector<double> h((size_t)(np + 1) * (np + 1)), dl(np);
            download(ctx, h.data(), p.dbg_A, h.size());
            download(ctx, dl.data(), a.delta, dl.size());
            sync(ctx);
            FILE* f = std::fopen(dump, "wb");
            std::fwrite(h.data(), 8, h.size(), f);
            std::fwrite(dl.data(), 8, dl.size(), f);
            std::fclose(f);
        }
        return;
    }
    int grid = 0;
    cuda_check(pvo_dev::launch_ba(a, ctx->num_sms, ctx->stream, &grid), "ba kernel");
    ctx->launches += 1;
}

inline void ensure_p3(int p) {
    if (p != 3) fail(PVO_UNSUPPORTED, "the sm_100a kernels implement 3x3 patches (p = 3)");
}

// A frame-store slot's features changed: its FP64 neighbour-Gram maps are stale.
inline void invalidate_g25(pvo_ctx* ctx, int slot) {
    if (slot >= 0 && slot < (int)ctx->g25_valid.size()) ctx->g25_valid[slot] = 0;
}

// The FP64 neighbour-Gram maps of every slot (the Gram-form measurement kernel
// reads them): allocated on first use, re-derived for the slots written since.
// PVO_MEASURE_DIRECT=1 selects the direct kernel instead (A/B).
inline void ensure_g25(pvo_ctx* ctx, pvo_dev::MeasureParams& m) {
    static const bool direct = std::getenv("PVO_MEASURE_DIRECT") != nullptr;
    if (direct) return;
    const size_t c0 = (size_t)ctx->w0 * ctx->h0, c1 = (size_t)ctx->w1 * ctx->h1;
    double* g0 = ctx->g25_0.as<double>((size_t)ctx->nf * c0 * pvo_dev::kGram25);
    double* g1 = ctx->g25_1.as<double>((size_t)ctx->nf * std::max<size_t>(c1, 1) * pvo_dev::kGram25);
    if ((int)ctx->g25_valid.size() != ctx->nf) ctx->g25_valid.assign(ctx->nf, 0);
    for (int s = 0; s < ctx->nf; ++s) {
        if (ctx->g25_valid[s]) continue;
        const float* f0 = static_cast<const float*>(ctx->feat0.p) + (size_t)s * c0 * ctx->C;
        const float* f1 = static_cast<const float*>(ctx->feat1.p) + (size_t)s * c1 * ctx->C;
        cuda_check(pvo_dev::launch_gram25(f0, ctx->w0, ctx->h0, ctx->C, g0 + (size_t)s * c0 * pvo_dev::kGram25,
                                          ctx->stream),
                   "gram25 kernel");
        cuda_check(pvo_dev::launch_gram25(f1, ctx->w1, ctx->h1, ctx->C, g1 + (size_t)s * c1 * pvo_dev::kGram25,
                                          ctx->stream),
                   "gram25 kernel");
        ctx->launches += c1 ? 2 : 1;
        ctx->g25_valid[s] = 1;
    }
    m.g25_0 = g0;
    m.g25_1 = g1;
    const size_t need = ((size_t)m.n_edges + 3) * sizeof(int);
    if (ctx->replay.cap < need) {  // (re)allocated: zero it once; the kernels leave it zero
        ctx->replay.get(need);
        cuda_check(cudaMemsetAsync(ctx->replay.p, 0, ctx->replay.cap, ctx->stream), "memset");
    }
    m.replay_done = static_cast<int*>(ctx->replay.p);  // [done, stat, count, edges...]
    m.replay_stat = m.replay_done + 1;
    m.replay = m.replay_done + 2;
}

inline void compute_gram(pvo_ctx* ctx, const float* f0, float* g0, const float* f1, float* g1, int w0, int h0, int w1,
                  int h1, int C) {
    if (w0 * h0 + w1 * h1 > 0) {
        cuda_check(pvo_dev::launch_gram(f0, g0, w0, h0, f1, g1, std::max(w1, 0), std::max(h1, 0), C, ctx->num_sms,
                                        ctx->stream),
                   "gram kernel");
        ctx->launches += 1;
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        cuda_check(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q),
                   "cudaGetDriverEntryPoint");
        if (q != cudaDriverEntryPointSuccess || !p) fail(PVO_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

inline bool encode_map(CUtensorMap* map, int rank, void* base, const uint64_t* dims, const uint32_t* box,
                CUtensorMapSwizzle swizzle) {
    cuuint64_t d[4], strides[3];
    cuuint32_t bx[4], estr[4];
    uint64_t stride = 4;
    for (int i = 0; i < rank; ++i) {
        d[i] = dims[i];
        bx[i] = box[i];
        estr[i] = 1;
        if (i > 0) strides[i - 1] = stride;
        stride *= dims[i];
    }
    const CUresult r = tensor_map_encoder()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, base, d, strides, bx, estr,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// (Re)build the frame-store TMA descriptors (layouts in kernels.cuh): feature
// tiles in 16-channel chunks with the 64B swizzle, planar Gram records with a
// 12 x 9 x 5 box (Gram rows padded to 4 cells).  C != 128 leaves the generic
// kernel in charge.
inline void encode_frame_maps(pvo_ctx* ctx) {
    ctx->maps_ok = false;
    ctx->patch_map_base = nullptr;
    if (ctx->C != 128 || ctx->w1 < 1 || ctx->h1 < 1) return;
    const uint64_t f0[4] = {128, (uint64_t)ctx->w0, (uint64_t)ctx->h0, (uint64_t)ctx->nf};
    const uint64_t f1[4] = {128, (uint64_t)ctx->w1, (uint64_t)ctx->h1, (uint64_t)ctx->nf};
    const uint64_t g0[4] = {(uint64_t)pvo_dev::gram_stride(ctx->w0), (uint64_t)ctx->h0, 8, (uint64_t)ctx->nf};
    const uint64_t g1[4] = {(uint64_t)pvo_dev::gram_stride(ctx->w1), (uint64_t)ctx->h1, 8, (uint64_t)ctx->nf};
    const uint32_t fbox[4] = {16, 9, 9, 1}, gbox[4] = {12, 9, 5, 1}, nbox[4] = {16, 8, 8, 1};
    ctx->maps_ok = encode_map(&ctx->maps[0], 4, ctx->feat0.p, f0, fbox, CU_TENSOR_MAP_SWIZZLE_64B) &&
                   encode_map(&ctx->maps[1], 4, ctx->feat1.p, f1, fbox, CU_TENSOR_MAP_SWIZZLE_64B) &&
                   encode_map(&ctx->maps[2], 4, ctx->gram0.p, g0, gbox, CU_TENSOR_MAP_SWIZZLE_NONE) &&
                   encode_map(&ctx->maps[3], 4, ctx->gram1.p, g1, gbox, CU_TENSOR_MAP_SWIZZLE_NONE) &&
                   encode_map(&ctx->maps[5], 4, ctx->feat0.p, f0, nbox, CU_TENSOR_MAP_SWIZZLE_64B) &&
                   encode_map(&ctx->maps[6], 4, ctx->feat1.p, f1, nbox, CU_TENSOR_MAP_SWIZZLE_64B);
}

// Descriptor of the patch-descriptor array [P * 2 * 9][128] (cached per base).
inline bool encode_patch_map(pvo_ctx* ctx, const float* base, int n_patches) {
    if (ctx->patch_map_base == base && ctx->patch_map_rows == n_patches * 18) return true;
    ctx->patch_map_base = nullptr;
    if (n_patches < 1 || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
    const uint64_t dims[2] = {128, (uint64_t)n_patches * 18};
    const uint32_t box[2] = {16, 9};
    if (!encode_map(&ctx->maps[4], 2, const_cast<float*>(base), dims, box, CU_TENSOR_MAP_SWIZZLE_NONE)) return false;
    ctx->patch_map_base = base;
    ctx->patch_map_rows = n_patches * 18;
    return true;
}

// Correlation of a batch of edges against the frame store: the TMA kernel for
// D = 128 (it splits wide tiles into sub-tiles itself), or the generic kernel
// for other channel counts.  `t` carries the inputs; scratch is filled in here.
inline void run_corr(pvo_ctx* ctx, pvo_dev::CorrTmaParams t, int index_edges = 0) {
    if (t.n_edges <= 0) return;
    NvtxRange range("corr");
    if (ctx->maps_ok && encode_patch_map(ctx, t.patch_feats, t.n_patches)) {
        t.w0 = ctx->w0;
        t.h0 = ctx->h0;
        t.w1 = ctx->w1;
        t.h1 = ctx->h1;
        t.feat0 = static_cast<const float*>(ctx->feat0.p);
        t.feat1 = static_cast<const float*>(ctx->feat1.p);
        t.coords = ctx->c_coords.as<double>((size_t)std::max(t.n_edges, index_edges) * 18);  // indexed by edge
        t.list_cap = pvo_dev::corr_tma_list_cap(t.n_edges);
        t.meta = ctx->c_meta.as<int>((size_t)t.list_cap * pvo_dev::kCorrMetaInts);
        t.ctl = ctx->d_corr_ctl;
        t.status = ctx->d_status;
        cuda_check(pvo_dev::launch_corr_tma(t, ctx->maps, ctx->num_sms, ctx->stream), "corr_tma kernel");
        ctx->launches += 2;  // tile preparation + correlation
        return;
    }
    pvo_dev::CorrParams cp;
    cp.n_edges = t.n_edges;
    cp.channels = ctx->C;
    cp.e_patch = t.e_patch;
    cp.e_pose = t.e_pose;
    cp.e_slot = t.e_slot;
    cp.pose_slot = t.pose_slot;
    cp.coords = t.coords_in;
    cp.poses = t.poses;
    cp.patch_src = t.patch_src;
    cp.patch_x = t.patch_x;
    cp.patch_y = t.patch_y;
    cp.depth = t.depth;
    cp.K = t.K;
    cp.feat0 = static_cast<const float*>(ctx->feat0.p);
    cp.feat1 = static_cast<const float*>(ctx->feat1.p);
    cp.gram0 = static_cast<const float*>(ctx->gram0.p);
    cp.gram1 = static_cast<const float*>(ctx->gram1.p);
    cp.w0 = ctx->w0;
    cp.h0 = ctx->h0;
    cp.w1 = ctx->w1;
    cp.h1 = ctx->h1;
    cp.patch_feats = t.patch_feats;
    cp.out = t.out;
    cp.status = ctx->d_status;
    cuda_check(pvo_dev::launch_corr(cp, ctx->stream), "corr kernel");
    ctx->launches += 1;
}

// Fingerprint of a host grid: its size and 256 evenly spaced samples.
inline uint64_t grid_fingerprint(const float* data, size_t n) {
    uint64_t h = 1469598103934665603ull ^ n;
    if (!n) return h;
    const size_t samples = std::min<size_t>(n, 256);
    for (size_t i = 0; i < samples; ++i) {
        uint32_t bits;
        std::memcpy(&bits, data + (samples == 1 ? 0 : i * (n - 1) / (samples - 1)), 4);
        h = (h ^ bits) * 1099511628211ull;
    }
    return h;
}

inline void grid_cache_clear(pvo_ctx* ctx) {
    for (GridEntry* e : ctx->grids) {
        e->feat.release();
        e->gram.release();
        delete e;
    }
    ctx->grids.clear();
    ctx->grid_bytes = 0;
}

// The device copy of host grid [h][w][C] (uploaded on a miss; Gram terms
// derived when `gram` is asked for).  Stream-ordered: the caller syncs before
// the host buffer may change.
inline GridEntry* cached_grid(pvo_ctx* ctx, const float* host, int w, int h, int C, bool gram) {
    const size_t n = (size_t)std::max(w, 0) * std::max(h, 0) * C;
    const uint64_t fp = grid_fingerprint(host, n);
    GridEntry* hit = nullptr;
    for (GridEntry* e : ctx->grids)
        if (e->host == host && e->w == w && e->h == h && e->C == C && e->fp == fp) hit = e;
    if (hit) {
        ++ctx->grid_hits;
    } else {
        ++ctx->grid_misses;
        const size_t bytes = sizeof(float) * (n + (size_t)std::max(pvo_dev::gram_stride(w) * h, 1) * 8);
        const char* mb = std::getenv("PVO_GRID_CACHE_MB");
        const size_t cap = (size_t)(mb ? std::max(1L, std::atol(mb)) : 4096L) << 20;
        while (ctx->grid_bytes + bytes > cap) {  // evict least recently used (never the one this call just used)
            auto lru = std::min_element(ctx->grids.begin(), ctx->grids.end(),
                                        [](const GridEntry* a, const GridEntry* b) { return a->tick < b->tick; });
            if (lru == ctx->grids.end() || (*lru)->tick == ctx->grid_tick) break;
            ctx->grid_bytes -= (*lru)->bytes;
            cuda_check(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");  // in-flight readers
            (*lru)->feat.release();
            (*lru)->gram.release();
            delete *lru;
            ctx->grids.erase(lru);
        }
        hit = new GridEntry;
        hit->host = host;
        hit->w = w;
        hit->h = h;
        hit->C = C;
        hit->fp = fp;
        hit->bytes = bytes;
        ctx->grids.push_back(hit);
        ctx->grid_bytes += bytes;
        upload(ctx, hit->feat, host, n);
    }
    hit->tick = ++ctx->grid_tick;
    if (gram && !hit->has_gram) {
        float* g = hit->gram.as<float>((size_t)std::max(pvo_dev::gram_stride(w) * h, 1) * 8);
        cuda_check(cudaMemsetAsync(g, 0, hit->gram.cap, ctx->stream), "memset");
        if (n) {
            cuda_check(pvo_dev::launch_gram(static_cast<const float*>(hit->feat.p), g, w, h, nullptr, nullptr, 0, 0, C,
                                            ctx->num_sms, ctx->stream),
                       "gram kernel");
            ctx->launches += 1;
        }
        hit->has_gram = true;
    }
    return hit;
}

// Stable order of edges by frame-store slot (L2 locality of the TMA kernel).
inline std::vector<int> slot_order(int n, const int* slot_of_edge) {
    // stable counting sort by frame slot (= std::stable_sort by slot, O(n))
    int lo = 0, hi = -1;
    for (int e = 0; e < n; ++e) {
        lo = e == 0 ? slot_of_edge[e] : std::min(lo, slot_of_edge[e]);
        hi = e == 0 ? slot_of_edge[e] : std::max(hi, slot_of_edge[e]);
    }
    std::vector<int> order(n);
    std::vector<int> start((size_t)std::max(hi - lo + 2, 1), 0);
    for (int e = 0; e < n; ++e) ++start[slot_of_edge[e] - lo + 1];
    for (size_t i = 1; i < start.size(); ++i) start[i] += start[i - 1];
    for (int e = 0; e < n; ++e) order[start[slot_of_edge[e] - lo]++] = e;
    return order;
}

}  // namespace pvo_host
