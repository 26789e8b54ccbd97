// capi.cu — the extern "C" boundary (include/pvo_capi.h): context, frame
// store, correlation, camera, bundle adjustment and the resident window.
//
// The host code here only validates, flattens and moves memory; every
// numeric result comes from the sm_100a kernels in corr.cu / ba.cu.  There
// is deliberately no CPU compute fallback.
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

namespace pvo_host {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace pvo_host

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
void plan_groups(const HostProblem& pr, Plan& pl) {
    constexpr int kGroupPatches = 64;
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
    void release() {
        DevBuf* all[] = {&poses,     &free_slot, &src,        &px,        &py,         &depth,     &depth_slot,
                         &edge_begin, &e_patch,  &e_pose,     &e_in,      &e_w,        &e_target,  &e_weight,
                         &cand_poses, &cand_depth, &patch_v,  &patch_h,   &patch_bd,   &partials,  &system,
                         &delta,     &norms,     &n_norms,    &status2,   &attempts,   &status,    &K,
                         &g_e_patch, &g_e_pose,  &g_src,      &pose_slot, &order,      &patch_feats, &corr,
                         &params,    &init_poses, &init_depth};
        for (DevBuf* b : all) b->release();
    }
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
    std::mt19937_64 oracle_rng{0};  // the oracle provider's RNG (flow_provider.cpp:10, rng_(noise.seed))
    int* d_corr_ctl = nullptr;      // correlation tile queue: [list length, queue head, warps done, -]
    void* h_stage = nullptr;        // page-locked staging for small read-backs (async copies, one sync)
    size_t h_stage_cap = 0;
    void* stage(size_t bytes) {
        if (bytes > h_stage_cap) {
            if (h_stage) cudaFreeHost(h_stage);
            h_stage = nullptr;
            h_stage_cap = 0;
            cuda_check(cudaMallocHost(&h_stage, bytes), "cudaMallocHost");
            h_stage_cap = bytes;
        }
        return h_stage;
    }
};

namespace {

void bind(pvo_ctx* ctx) {
    if (!ctx) fail(PVO_INVALID_ARGUMENT, "null context");
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
}

template <typename T>
T* upload(pvo_ctx* ctx, DevBuf& buf, const T* host, size_t count) {
    T* d = buf.as<T>(count);
    if (count) cuda_check(cudaMemcpyAsync(d, host, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream), "H2D");
    return d;
}
template <typename T>
void download(pvo_ctx* ctx, T* host, const T* dev, size_t count) {
    if (count) cuda_check(cudaMemcpyAsync(host, dev, count * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
}
void sync(pvo_ctx* ctx) { cuda_check(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize"); }
// The per-iteration timing events (pvo_ctx_last_timing).  Under stream capture
// they are recorded as external event nodes, so a graph replay records them too.
void record_timing(pvo_ctx* ctx, int i) {
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
bool host_pinned(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

void reset_status(pvo_ctx* ctx) {
    cuda_check(cudaMemsetAsync(ctx->d_status, 0, sizeof(int), ctx->stream), "status reset");
}
int read_status(pvo_ctx* ctx) {
    int s = 0;
    cuda_check(cudaMemcpyAsync(&s, ctx->d_status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "status");
    sync(ctx);
    return s;
}
// BA status bits -> the reference's exception (bundle_adjust.cpp:65-92, :147-149).
void raise_ba_status(int s) {
    if (!s) return;
    using namespace pvo_dev;
    if (s & (1 << kDevNonFiniteResidual)) fail(PVO_DEGENERATE, "ba: non-finite residual");
    if (s & (1 << kDevNonPositiveDepth)) fail(PVO_DEGENERATE, "schur: non-positive damped depth-block entry");
    if (s & (1 << kDevFactorization)) fail(PVO_DEGENERATE, "schur: reduced camera system factorization failed");
    if (s & (1 << kDevNonFinitePose)) fail(PVO_DEGENERATE, "schur: non-finite pose update");
    if (s & (1 << kDevNonFiniteDepth)) fail(PVO_DEGENERATE, "schur: non-finite depth update");
    fail(PVO_CUDA_ERROR, "unknown device status");
}

bool finite2(const double* v) { return std::isfinite(v[0]) && std::isfinite(v[1]); }

// BAProblem::validate (bundle_adjust.cpp:11-36).
void validate(const HostProblem& pr) {
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

Plan make_plan(const HostProblem& pr, bool all_fixed) {
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
pvo_dev::BAParams stage_problem(pvo_ctx* ctx, const HostProblem& pr, const Plan& pl, int extra_norms) {
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
pvo_dev::BALargeParams large_params(pvo_ctx* ctx, const pvo_dev::BAParams& a, const Plan& pl) {
    BABuffers& B = ctx->ba;
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

void launch_ba_checked(pvo_ctx* ctx, pvo_dev::BAParams& a, const Plan& pl) {
    cuda_check(cudaMemsetAsync(a.n_norms, 0, sizeof(int), ctx->stream), "memset");
    if (pl.large) {
        if (a.gn_step_mode) fail(PVO_UNSUPPORTED, "gauss_newton_step: pose systems beyond 16 free poses");
        cuda_check(cudaMemsetAsync(a.attempts, 0, sizeof(int), ctx->stream), "memset");
        pvo_dev::BALargeParams p = large_params(ctx, a, pl);
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

void ensure_p3(int p) {
    if (p != 3) fail(PVO_UNSUPPORTED, "the sm_100a kernels implement 3x3 patches (p = 3)");
}

void compute_gram(pvo_ctx* ctx, const float* f0, float* g0, const float* f1, float* g1, int w0, int h0, int w1,
                  int h1, int C) {
    if (w0 * h0 + w1 * h1 > 0) {
        cuda_check(pvo_dev::launch_gram(f0, g0, w0, h0, f1, g1, std::max(w1, 0), std::max(h1, 0), C, ctx->num_sms,
                                        ctx->stream),
                   "gram kernel");
        ctx->launches += 1;
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
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

bool encode_map(CUtensorMap* map, int rank, void* base, const uint64_t* dims, const uint32_t* box,
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
void encode_frame_maps(pvo_ctx* ctx) {
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
bool encode_patch_map(pvo_ctx* ctx, const float* base, int n_patches) {
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
void run_corr(pvo_ctx* ctx, pvo_dev::CorrTmaParams t, int index_edges = 0) {
    if (t.n_edges <= 0) return;
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

// Stable order of edges by frame-store slot (L2 locality of the TMA kernel).
std::vector<int> slot_order(int n, const int* slot_of_edge) {
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

}  // namespace

namespace pvo_host {

void run_ba(pvo_ctx* ctx, const HostProblem& pr, const BARun& run) {
    bind(ctx);
    validate(pr);
    if (run.gn_step_mode && pr.n_edges == 0) fail(PVO_INVALID_ARGUMENT, "ba: need at least one edge");
    const Plan pl = make_plan(pr, false);
    if (run.n_free_poses) *run.n_free_poses = pl.n_free_poses;
    if (run.n_free_depths) *run.n_free_depths = pl.n_free_depths;
    if (pr.n_edges == 0) {
        // nothing to optimise: state unchanged
        std::memcpy(run.out_poses, pr.poses, sizeof(double) * 7 * pr.n_poses);
        std::memcpy(run.out_depth, pr.depth, sizeof(double) * pr.n_patches);
        if (run.n_norms) *run.n_norms = 0;
        return;
    }
    pvo_dev::BAParams a = stage_problem(ctx, pr, pl, run.iterations + run.structure_only + 2);
    a.freeze_targets = run.freeze_targets;
    a.iterations = run.iterations;
    a.structure_only = run.structure_only;
    a.gn_step_mode = run.gn_step_mode;
    reset_status(ctx);
    if ((run.debug_h || run.debug_b) && pl.large) fail(PVO_UNSUPPORTED, "normal-equation capture: pose systems beyond 16 free poses");
    if (run.debug_h || run.debug_b) {
        const int n = 6 * pl.n_free_poses + pl.n_free_depths;
        double* dh = ctx->ba.dbg_h.as<double>((size_t)n * n);
        double* db = ctx->ba.dbg_b.as<double>(n);
        cuda_check(pvo_dev::launch_normal_equations_debug(a, dh, db, ctx->stream), "debug kernel");
        ctx->launches += 1;
        if (run.debug_h) download(ctx, run.debug_h, dh, (size_t)n * n);
        if (run.debug_b) download(ctx, run.debug_b, db, n);
    }
    launch_ba_checked(ctx, a, pl);
    const int status = read_status(ctx);
    raise_ba_status(status);
    download(ctx, run.out_poses, a.poses, (size_t)pr.n_poses * 7);
    download(ctx, run.out_depth, a.depth, pr.n_patches);
    int n_norms = 0;
    download(ctx, &n_norms, a.n_norms, 1);
    sync(ctx);
    if (run.residual_norms && n_norms > 0) {
        download(ctx, run.residual_norms, a.residual_norms, n_norms);
        sync(ctx);
    }
    if (run.n_norms) *run.n_norms = n_norms;
}

}  // namespace pvo_host

// ===========================================================================
// extern "C"
// ===========================================================================
extern "C" {

int pvo_version(void) { return 1; }
const char* pvo_last_error(void) { return pvo_host::g_last_error.c_str(); }

const char* pvo_status_string(int status) {
    switch (status) {
        case PVO_OK: return "ok";
        case PVO_INVALID_ARGUMENT: return "invalid_argument";
        case PVO_DEGENERATE: return "degenerate_problem";
        case PVO_DOMAIN_ERROR: return "domain_error";
        case PVO_OUT_OF_RANGE: return "out_of_range";
        case PVO_CUDA_ERROR: return "cuda_error";
        case PVO_UNSUPPORTED: return "unsupported";
        default: return "unknown";
    }
}

int pvo_ctx_create(int device, pvo_ctx** out) {
    return guarded([&] {
        if (!out) fail(PVO_INVALID_ARGUMENT, "null output");
        *out = nullptr;
        int n = 0;
        cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        if (device < 0 || device >= n) fail(PVO_CUDA_ERROR, "no CUDA device " + std::to_string(device));
        cudaDeviceProp prop{};
        cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (prop.major < 10) {
            fail(PVO_CUDA_ERROR, std::string("device ") + prop.name + " is not sm_100 (kernels are built for sm_100a)");
        }
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        auto* ctx = new pvo_ctx();
        ctx->device = device;
        ctx->num_sms = prop.multiProcessorCount;
        cuda_check(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "cudaStreamCreate");
        ctx->own_stream = true;
        cuda_check(cudaMalloc(&ctx->d_status, sizeof(int)), "cudaMalloc");
        cuda_check(cudaMalloc(&ctx->d_corr_ctl, 4 * sizeof(int)), "cudaMalloc");
        cuda_check(cudaMemset(ctx->d_corr_ctl, 0, 4 * sizeof(int)), "cudaMemset");  // kept zero between launches
        for (auto& e : ctx->ev) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
        cuda_check(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
        cuda_check(cudaEventCreateWithFlags(&ctx->ev_corr, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&ctx->ev_corr2, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&ctx->ev_copy, cudaEventDisableTiming), "cudaEventCreate");
        *out = ctx;
    });
}

int pvo_ctx_destroy(pvo_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        DevBuf* bufs[] = {&ctx->feat0, &ctx->feat1, &ctx->gram0, &ctx->gram1, &ctx->s0, &ctx->s1, &ctx->s2,
                          &ctx->s3,    &ctx->s4,    &ctx->s5,    &ctx->s6,    &ctx->s7, &ctx->s8,
                          &ctx->win.pose_slot, &ctx->win.patch_feats, &ctx->win.corr, &ctx->win.init_poses,
                          &ctx->win.init_depth, &ctx->win.order, &ctx->win.order_half, &ctx->win.flags, &ctx->c_coords, &ctx->c_meta,
                          &ctx->c_over, &ctx->c_order};
        for (DevBuf* b : bufs) b->release();
        ctx->ba.release();
        ctx->bat.release();
        if (ctx->d_status) cudaFree(ctx->d_status);
        if (ctx->d_corr_ctl) cudaFree(ctx->d_corr_ctl);
        if (ctx->h_stage) cudaFreeHost(ctx->h_stage);
        for (auto& e : ctx->ev)
            if (e) cudaEventDestroy(e);
        if (ctx->copy_stream) {
            cudaStreamSynchronize(ctx->copy_stream);
            cudaStreamDestroy(ctx->copy_stream);
        }
        if (ctx->ev_corr) cudaEventDestroy(ctx->ev_corr);
        if (ctx->ev_corr2) cudaEventDestroy(ctx->ev_corr2);
        if (ctx->ev_copy) cudaEventDestroy(ctx->ev_copy);
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

int pvo_ctx_set_stream(pvo_ctx* ctx, void* stream) {
    return guarded([&] {
        bind(ctx);
        if (ctx->own_stream) {
            cudaStreamSynchronize(ctx->stream);
            cudaStreamDestroy(ctx->stream);
            ctx->own_stream = false;
        }
        if (stream) {
            ctx->stream = static_cast<cudaStream_t>(stream);
        } else {
            cuda_check(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "cudaStreamCreate");
            ctx->own_stream = true;
        }
    });
}

int pvo_ctx_synchronize(pvo_ctx* ctx) {
    return guarded([&] {
        bind(ctx);
        sync(ctx);
    });
}

int64_t pvo_ctx_kernel_launches(pvo_ctx* ctx) { return ctx ? ctx->launches : -1; }

int pvo_ctx_set_timing(pvo_ctx* ctx, int on) {
    return guarded([&] {
        bind(ctx);
        ctx->timing = on != 0;
        if (!ctx->timing) ctx->timing_pending = false;
    });
}

int pvo_ctx_set_tracing(pvo_ctx* ctx, int on) {
    return guarded([&] {
        bind(ctx);
        ctx->tracing = on != 0;
        if (ctx->tracing) {
            long long* c = ctx->ba.clocks.as<long long>(128);
            cuda_check(cudaMemsetAsync(c, 0, 128 * sizeof(long long), ctx->stream), "memset");
        }
    });
}

int pvo_ctx_ba_phase_cycles(pvo_ctx* ctx, long long* out128) {
    return guarded([&] {
        bind(ctx);
        if (!ctx->tracing) fail(PVO_INVALID_ARGUMENT, "tracing is off (pvo_ctx_set_tracing)");
        download(ctx, out128, static_cast<const long long*>(ctx->ba.clocks.p), 128);
        sync(ctx);
    });
}

int pvo_ctx_ba_attempts(pvo_ctx* ctx, int* attempts) {
    return guarded([&] {
        bind(ctx);
        *attempts = 0;
        if (ctx->ba.attempts.p) {
            download(ctx, attempts, static_cast<const int*>(ctx->ba.attempts.p), 1);
            sync(ctx);
        }
    });
}

int pvo_ctx_last_timing(pvo_ctx* ctx, double* corr_ms, double* ba_ms) {
    return guarded([&] {
        bind(ctx);
        if (!ctx->timing_pending) fail(PVO_INVALID_ARGUMENT, "no timed iteration recorded");
        cuda_check(cudaEventSynchronize(ctx->ev[2]), "cudaEventSynchronize");
        float a = 0, b = 0;
        cuda_check(cudaEventElapsedTime(&a, ctx->ev[0], ctx->ev[1]), "cudaEventElapsedTime");
        cuda_check(cudaEventElapsedTime(&b, ctx->ev[1], ctx->ev[2]), "cudaEventElapsedTime");
        if (corr_ms) *corr_ms = a;
        if (ba_ms) *ba_ms = b;
    });
}

// ---- SE(3) host utilities ------------------------------------------------
int pvo_se3_exp(const double* xi, double* out) {
    return guarded([&] { pvo_dev::se3_store(pvo_dev::se3_exp(xi), out); });
}
int pvo_se3_log(const double* pose, double* xi) {
    return guarded([&] { se3_log_host(pose, xi); });
}
int pvo_se3_compose(const double* a, const double* b, double* out) {
    return guarded([&] {
        pvo_dev::se3_store(pvo_dev::se3_compose(pvo_dev::se3_load(a), pvo_dev::se3_load(b)), out);
    });
}
int pvo_se3_inverse(const double* a, double* out) {
    return guarded([&] { pvo_dev::se3_store(pvo_dev::se3_inverse(pvo_dev::se3_load(a)), out); });
}
int pvo_se3_retract(const double* a, const double* xi, double* out) {
    return guarded([&] { pvo_dev::se3_store(pvo_dev::se3_retract(pvo_dev::se3_load(a), xi), out); });
}

// ---- camera ----------------------------------------------------------------
int pvo_reproject_patches(pvo_ctx* ctx, int n, int p, const double* pi, const double* pj, const double* K,
                          const double* x, const double* y, const double* d, double* out_xy, uint8_t* behind) {
    return guarded([&] {
        bind(ctx);
        if (n < 0 || p < 1) fail(PVO_INVALID_ARGUMENT, "reproject: bad sizes");
        if (n == 0) return;
        const int pp = p * p;
        double* dpi = upload(ctx, ctx->s0, pi, (size_t)n * 7);
        double* dpj = upload(ctx, ctx->s1, pj, (size_t)n * 7);
        double* dK = upload(ctx, ctx->s2, K, 4);
        double* dx = upload(ctx, ctx->s3, x, (size_t)n * pp);
        double* dy = upload(ctx, ctx->s4, y, (size_t)n * pp);
        double* dd = upload(ctx, ctx->s5, d, n);
        double* dout = ctx->s6.as<double>((size_t)n * pp * 2);
        uint8_t* db = ctx->s7.as<uint8_t>(n);
        cuda_check(pvo_dev::launch_reproject(n, pp, dpi, dpj, dK, dx, dy, dd, dout, db, ctx->stream), "reproject");
        ctx->launches += 1;
        download(ctx, out_xy, dout, (size_t)n * pp * 2);
        download(ctx, behind, db, n);
        sync(ctx);
    });
}

int pvo_reprojection_jacobians(pvo_ctx* ctx, int n, int p, const double* pi, const double* pj, const double* K,
                               const double* x, const double* y, const double* d, double* out, uint8_t* behind) {
    return guarded([&] {
        bind(ctx);
        if (n < 0 || p < 1) fail(PVO_INVALID_ARGUMENT, "jacobians: bad sizes");
        if (n == 0) return;
        const int pp = p * p;
        double* dpi = upload(ctx, ctx->s0, pi, (size_t)n * 7);
        double* dpj = upload(ctx, ctx->s1, pj, (size_t)n * 7);
        double* dK = upload(ctx, ctx->s2, K, 4);
        double* dx = upload(ctx, ctx->s3, x, (size_t)n * pp);
        double* dy = upload(ctx, ctx->s4, y, (size_t)n * pp);
        double* dd = upload(ctx, ctx->s5, d, n);
        double* dout = ctx->s6.as<double>((size_t)n * 28);
        uint8_t* db = ctx->s7.as<uint8_t>(n);
        cuda_check(pvo_dev::launch_jacobians(n, pp, dpi, dpj, dK, dx, dy, dd, dout, db, ctx->stream), "jacobians");
        ctx->launches += 1;
        download(ctx, out, dout, (size_t)n * 28);
        download(ctx, behind, db, n);
        sync(ctx);
    });
}

// ---- correlation -------------------------------------------------------------
int pvo_correlate(pvo_ctx* ctx, int p, int C, const float* feats0, const float* feats1, const float* level0, int w0,
                  int h0, const float* level1, int w1, int h1, const double* coords, float* out) {
    return guarded([&] {
        bind(ctx);
        ensure_p3(p);
        if (C < 1 || w0 < 0 || h0 < 0 || w1 < 0 || h1 < 0) fail(PVO_INVALID_ARGUMENT, "correlate: bad sizes");
        for (int k = 0; k < p * p; ++k)
            if (!finite2(coords + 2 * k)) fail(PVO_INVALID_ARGUMENT, "correlate: non-finite reprojection");
        const size_t n0 = (size_t)w0 * h0 * C, n1 = (size_t)w1 * h1 * C;
        float* f0 = upload(ctx, ctx->s0, level0, n0);
        float* f1 = upload(ctx, ctx->s1, level1, n1);
        float* g0 = ctx->s2.as<float>((size_t)pvo_dev::gram_stride(w0) * h0 * 8);
        float* g1 = ctx->s3.as<float>((size_t)std::max(pvo_dev::gram_stride(w1) * h1, 1) * 8);
        compute_gram(ctx, f0, g0, f1, g1, w0, h0, w1, h1, C);
        float* pf = ctx->s4.as<float>((size_t)2 * 9 * C);
        cuda_check(cudaMemcpyAsync(pf, feats0, sizeof(float) * 9 * C, cudaMemcpyHostToDevice, ctx->stream), "H2D");
        cuda_check(cudaMemcpyAsync(pf + 9 * C, feats1, sizeof(float) * 9 * C, cudaMemcpyHostToDevice, ctx->stream),
                   "H2D");
        double* dc = upload(ctx, ctx->s5, coords, 18);
        int zero = 0;
        int* idx = upload(ctx, ctx->s6, &zero, 1);
        float* dout = ctx->s7.as<float>(2 * 9 * 49);
        reset_status(ctx);
        pvo_dev::CorrParams cp;
        cp.n_edges = 1;
        cp.channels = C;
        cp.e_patch = idx;
        cp.e_slot = idx;
        cp.coords = dc;
        cp.feat0 = f0;
        cp.feat1 = f1;
        cp.gram0 = g0;
        cp.gram1 = g1;
        cp.w0 = w0;
        cp.h0 = h0;
        cp.w1 = w1;
        cp.h1 = h1;
        cp.patch_feats = pf;
        cp.out = dout;
        cp.status = ctx->d_status;
        cuda_check(pvo_dev::launch_corr(cp, ctx->stream), "corr kernel");
        ctx->launches += 1;
        download(ctx, out, dout, 2 * 9 * 49);
        if (read_status(ctx)) fail(PVO_INVALID_ARGUMENT, "correlate: non-finite reprojection");
    });
}

int pvo_frames_reserve(pvo_ctx* ctx, int n_frames, int w0, int h0, int w1, int h1, int C) {
    return guarded([&] {
        bind(ctx);
        if (n_frames < 1 || w0 < 1 || h0 < 1 || w1 < 0 || h1 < 0 || C < 1) fail(PVO_INVALID_ARGUMENT, "frames: bad sizes");
        ctx->nf = n_frames;
        ctx->w0 = w0;
        ctx->h0 = h0;
        ctx->w1 = w1;
        ctx->h1 = h1;
        ctx->C = C;
        ctx->feat0.get(sizeof(float) * (size_t)n_frames * w0 * h0 * C);
        ctx->feat1.get(sizeof(float) * (size_t)n_frames * std::max(w1 * h1, 1) * C);
        const size_t gb0 = sizeof(float) * (size_t)n_frames * pvo_dev::gram_stride(w0) * h0 * 8;
        const size_t gb1 = sizeof(float) * (size_t)n_frames * std::max(pvo_dev::gram_stride(w1) * h1, 1) * 8;
        ctx->gram0.get(gb0);
        ctx->gram1.get(gb1);
        // row-pad cells of the Gram planes must read as zero (out of the image)
        cuda_check(cudaMemsetAsync(ctx->gram0.p, 0, gb0, ctx->stream), "memset");
        cuda_check(cudaMemsetAsync(ctx->gram1.p, 0, gb1, ctx->stream), "memset");
        encode_frame_maps(ctx);
    });
}

int pvo_frames_refresh(pvo_ctx* ctx, int slot) {
    return guarded([&] {
        bind(ctx);
        if (slot < 0 || slot >= ctx->nf) fail(PVO_OUT_OF_RANGE, "frames: slot out of range");
        const size_t c0 = (size_t)ctx->w0 * ctx->h0, c1 = (size_t)ctx->w1 * ctx->h1;
        float* f0 = static_cast<float*>(ctx->feat0.p) + slot * c0 * ctx->C;
        float* f1 = static_cast<float*>(ctx->feat1.p) + slot * c1 * ctx->C;
        float* g0 = static_cast<float*>(ctx->gram0.p) + (size_t)slot * pvo_dev::gram_stride(ctx->w0) * ctx->h0 * 8;
        float* g1 = static_cast<float*>(ctx->gram1.p) + (size_t)slot * pvo_dev::gram_stride(ctx->w1) * ctx->h1 * 8;
        compute_gram(ctx, f0, g0, f1, g1, ctx->w0, ctx->h0, ctx->w1, ctx->h1, ctx->C);
    });
}

int pvo_frames_upload(pvo_ctx* ctx, int slot, const float* level0, const float* level1, int memspace) {
    return guarded([&] {
        bind(ctx);
        if (slot < 0 || slot >= ctx->nf) fail(PVO_OUT_OF_RANGE, "frames: slot out of range");
        const size_t c0 = (size_t)ctx->w0 * ctx->h0, c1 = (size_t)ctx->w1 * ctx->h1;
        float* f0 = static_cast<float*>(ctx->feat0.p) + slot * c0 * ctx->C;
        float* f1 = static_cast<float*>(ctx->feat1.p) + slot * c1 * ctx->C;
        const cudaMemcpyKind kind = memspace == PVO_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        cuda_check(cudaMemcpyAsync(f0, level0, sizeof(float) * c0 * ctx->C, kind, ctx->stream), "frame upload");
        if (c1) cuda_check(cudaMemcpyAsync(f1, level1, sizeof(float) * c1 * ctx->C, kind, ctx->stream), "frame upload");
        float* g0 = static_cast<float*>(ctx->gram0.p) + (size_t)slot * pvo_dev::gram_stride(ctx->w0) * ctx->h0 * 8;
        float* g1 = static_cast<float*>(ctx->gram1.p) + (size_t)slot * pvo_dev::gram_stride(ctx->w1) * ctx->h1 * 8;
        compute_gram(ctx, f0, g0, f1, g1, ctx->w0, ctx->h0, ctx->w1, ctx->h1, ctx->C);
        if (memspace != PVO_DEVICE) sync(ctx);
    });
}

int pvo_frames_device_ptrs(pvo_ctx* ctx, float** level0, float** level1) {
    return guarded([&] {
        bind(ctx);
        if (level0) *level0 = static_cast<float*>(ctx->feat0.p);
        if (level1) *level1 = static_cast<float*>(ctx->feat1.p);
    });
}

int pvo_correlate_batch(pvo_ctx* ctx, int n_edges, int n_patches, int p, const int* e_patch, const int* e_slot,
                        const double* coords, const float* patch_feats, float* out, int memspace) {
    return guarded([&] {
        bind(ctx);
        ensure_p3(p);
        if (ctx->nf == 0) fail(PVO_INVALID_ARGUMENT, "correlate_batch: frame store is empty (pvo_frames_reserve)");
        if (n_edges < 0 || n_patches < 0) fail(PVO_INVALID_ARGUMENT, "correlate_batch: bad sizes");
        if (n_edges == 0) return;
        const int C = ctx->C;
        const int* dep;
        const int* des;
        const double* dc;
        const float* dpf;
        float* dout;
        if (memspace == PVO_DEVICE) {
            dep = e_patch;
            des = e_slot;
            dc = coords;
            dpf = patch_feats;
            dout = out;
        } else {
            for (int e = 0; e < n_edges; ++e) {
                if (e_patch[e] < 0 || e_patch[e] >= n_patches) fail(PVO_OUT_OF_RANGE, "correlate_batch: bad patch index");
                if (e_slot[e] < 0 || e_slot[e] >= ctx->nf) fail(PVO_OUT_OF_RANGE, "correlate_batch: bad frame slot");
            }
            dep = upload(ctx, ctx->s0, e_patch, n_edges);
            des = upload(ctx, ctx->s1, e_slot, n_edges);
            dc = upload(ctx, ctx->s2, coords, (size_t)n_edges * 18);
            dpf = upload(ctx, ctx->s3, patch_feats, (size_t)n_patches * 2 * 9 * C);
            dout = ctx->s4.as<float>((size_t)n_edges * 2 * 9 * 49);
        }
        const int* dorder = nullptr;
        if (memspace != PVO_DEVICE) {
            const std::vector<int> order = slot_order(n_edges, e_slot);
            dorder = upload(ctx, ctx->c_order, order.data(), order.size());
            sync(ctx);
        }
        reset_status(ctx);
        pvo_dev::CorrTmaParams t;
        t.n_edges = n_edges;
        t.order = dorder;
        t.e_patch = dep;
        t.e_slot = des;
        t.coords_in = dc;
        t.patch_feats = dpf;
        t.n_patches = n_patches;
        t.out = dout;
        run_corr(ctx, t);
        if (memspace != PVO_DEVICE) {
            download(ctx, out, dout, (size_t)n_edges * 2 * 9 * 49);
            if (read_status(ctx)) fail(PVO_INVALID_ARGUMENT, "correlate: non-finite reprojection");
        }
    });
}

// ---- bundle adjustment -----------------------------------------------------------
int pvo_gauss_newton_step(pvo_ctx* ctx, int n_poses, const double* poses, const uint8_t* fixed, int n_patches, int p,
                          const int* src, const double* px, const double* py, const double* depth,
                          const uint8_t* depth_free, int n_edges, const int* e_patch, const int* e_pose,
                          const double* e_target, const double* e_weight, const double* K, double damping,
                          double* out_poses, double* out_depth, double* residual_norms, double* debug_h,
                          double* debug_b, int* n_free_poses, int* n_free_depths) {
    return guarded([&] {
        HostProblem pr{n_poses, poses, fixed, n_patches, p, src, px, py, depth, depth_free, n_edges,
                       e_patch, e_pose, e_target, e_weight};
        std::memcpy(pr.K, K, sizeof(pr.K));
        pr.damping = damping;
        BARun run;
        run.iterations = 1;
        run.gn_step_mode = 1;
        run.out_poses = out_poses;
        run.out_depth = out_depth;
        run.residual_norms = residual_norms;
        run.debug_h = debug_h;
        run.debug_b = debug_b;
        run.n_free_poses = n_free_poses;
        run.n_free_depths = n_free_depths;
        run_ba(ctx, pr, run);
    });
}

int pvo_schur_solve(pvo_ctx* ctx, int np, int nd, const double* hpp, const double* hpd, const double* hdd,
                    const double* bp, const double* bd, double* dp, double* dd) {
    return guarded([&] {
        bind(ctx);
        if (np < 0 || nd < 0) fail(PVO_INVALID_ARGUMENT, "schur: bad sizes");
        for (int k = 0; k < nd; ++k)
            if (hdd[k] <= 0) fail(PVO_DEGENERATE, "schur: non-positive damped depth-block entry");
        double* d_hpp = upload(ctx, ctx->s0, hpp, (size_t)np * np);
        double* d_hpd = upload(ctx, ctx->s1, hpd, (size_t)np * nd);
        double* d_hdd = upload(ctx, ctx->s2, hdd, nd);
        double* d_bp = upload(ctx, ctx->s3, bp, np);
        double* d_bd = upload(ctx, ctx->s4, bd, nd);
        double* d_dp = ctx->s5.as<double>(std::max(np, 1));
        // dd followed by the reduced-system scratch (see launch_schur_dense)
        double* d_dd = ctx->s6.as<double>((size_t)nd + (size_t)np * (np + 1) / 2 + np + 1);
        reset_status(ctx);
        cuda_check(pvo_dev::launch_schur_dense(np, nd, d_hpp, d_hpd, d_hdd, d_bp, d_bd, d_dp, d_dd, ctx->d_status,
                                               ctx->stream),
                   "schur kernel");
        ctx->launches += 1;
        raise_ba_status(read_status(ctx));
        if (np) download(ctx, dp, d_dp, np);
        download(ctx, dd, d_dd, nd);
        sync(ctx);
    });
}

int pvo_ba_window(pvo_ctx* ctx, int n_poses, const double* poses, const uint8_t* fixed, int n_patches, int p,
                  const int* src, const double* px, const double* py, const double* depth, int n_edges,
                  const int* e_patch, const int* e_pose, const double* e_target, const double* e_weight,
                  const double* K, int image_w, int image_h, int freeze_targets, double damping, int iterations,
                  int structure_only, double* out_poses, double* out_depth, double* residual_norms, int* n_norms) {
    return guarded([&] {
        if (iterations < 0 || structure_only < 0) fail(PVO_INVALID_ARGUMENT, "ba: negative iteration count");
        HostProblem pr{n_poses, poses, fixed, n_patches, p, src, px, py, depth, nullptr, n_edges,
                       e_patch, e_pose, e_target, e_weight};
        std::memcpy(pr.K, K, sizeof(pr.K));
        pr.image_w = image_w;
        pr.image_h = image_h;
        pr.damping = damping;
        BARun run;
        run.freeze_targets = freeze_targets;
        run.iterations = iterations;
        run.structure_only = structure_only;
        run.out_poses = out_poses;
        run.out_depth = out_depth;
        run.residual_norms = residual_norms;
        run.n_norms = n_norms;
        if (freeze_targets) {
            // deltas are not validated as targets; validate() only checks finiteness
        }
        run_ba(ctx, pr, run);
    });
}

// ---- resident window ------------------------------------------------------------
int pvo_window_load(pvo_ctx* ctx, int n_poses, const double* poses, const uint8_t* fixed, const int* pose_slot,
                    int n_patches, int p, const int* src, const double* px, const double* py, const double* depth,
                    const float* patch_feats, int n_edges, const int* e_patch, const int* e_pose,
                    const double* e_delta, const double* e_weight, const double* K, int image_w, int image_h,
                    int memspace) {
    return guarded([&] {
        bind(ctx);
        if (memspace != PVO_HOST) fail(PVO_INVALID_ARGUMENT, "window_load: host arrays expected");
        if (ctx->nf == 0) fail(PVO_INVALID_ARGUMENT, "window_load: frame store is empty (pvo_frames_reserve)");
        HostProblem pr{n_poses, poses, fixed, n_patches, p, src, px, py, depth, nullptr, n_edges,
                       e_patch, e_pose, e_delta, e_weight};
        std::memcpy(pr.K, K, sizeof(pr.K));
        pr.image_w = image_w;
        pr.image_h = image_h;
        validate(pr);
        for (int i = 0; i < n_poses; ++i)
            if (pose_slot[i] < 0 || pose_slot[i] >= ctx->nf) fail(PVO_OUT_OF_RANGE, "window_load: bad frame slot");
        Window& w = ctx->win;
        // the inputs are valid: the resident window is replaced from here on (a
        // failure below leaves no window loaded).  The patch descriptors (the bulk
        // of the bytes) go first, so the transfer runs under the planning below.
        w.loaded = false;
        upload(ctx, w.patch_feats, patch_feats, (size_t)n_patches * 2 * 9 * ctx->C);
        w.plan = make_plan(pr, false);
        if (!w.plan.sorted) fail(PVO_INVALID_ARGUMENT, "window_load: edges must be grouped by patch (reference order)");
        w.shape = pr;
        w.n_poses = n_poses;
        w.n_patches = n_patches;
        w.n_edges = n_edges;
        stage_problem(ctx, pr, w.plan, 64);
        upload(ctx, w.pose_slot, pose_slot, n_poses);
        {
            std::vector<int> eslot(n_edges);
            for (int e = 0; e < n_edges; ++e) eslot[e] = pose_slot[e_pose[e]];
            const std::vector<int> order = slot_order(n_edges, eslot.data());
            upload(ctx, w.order, order.data(), order.size());  // pageable source: staged before return
            w.half = n_edges >= 4096 ? n_edges / 2 : 0;
            if (w.half) {
                std::vector<int> oh = slot_order(w.half, eslot.data());
                const std::vector<int> o2 = slot_order(n_edges - w.half, eslot.data() + w.half);
                for (int v : o2) oh.push_back(v + w.half);
                upload(ctx, w.order_half, oh.data(), oh.size());
            }
        }
        upload(ctx, w.init_poses, poses, (size_t)n_poses * 7);
        upload(ctx, w.init_depth, depth, n_patches);
        upload(ctx, ctx->ba.K, K, 4);
        w.corr.get(sizeof(float) * (size_t)n_edges * 2 * 9 * 49);
        sync(ctx);
        w.loaded = true;
    });
}

int pvo_window_set_state(pvo_ctx* ctx, const double* poses, const double* depth, int memspace) {
    return guarded([&] {
        bind(ctx);
        Window& w = ctx->win;
        if (!w.loaded) fail(PVO_INVALID_ARGUMENT, "window: nothing loaded");
        const cudaMemcpyKind kind = memspace == PVO_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        const double* sp = poses ? poses : static_cast<const double*>(w.init_poses.p);
        const double* sd = depth ? depth : static_cast<const double*>(w.init_depth.p);
        const cudaMemcpyKind kp = poses ? kind : cudaMemcpyDeviceToDevice;
        const cudaMemcpyKind kd = depth ? kind : cudaMemcpyDeviceToDevice;
        cuda_check(cudaMemcpyAsync(ctx->ba.poses.p, sp, sizeof(double) * 7 * w.n_poses, kp, ctx->stream), "state");
        cuda_check(cudaMemcpyAsync(ctx->ba.depth.p, sd, sizeof(double) * w.n_patches, kd, ctx->stream), "state");
    });
}

namespace {
pvo_dev::CorrTmaParams window_corr_params(pvo_ctx* ctx, float* out) {
    Window& w = ctx->win;
    pvo_dev::CorrTmaParams cp;
    cp.n_edges = w.n_edges;
    cp.order = static_cast<const int*>(w.order.p);
    cp.e_patch = static_cast<const int*>(ctx->ba.e_patch.p);
    cp.e_pose = static_cast<const int*>(ctx->ba.e_pose.p);
    cp.pose_slot = static_cast<const int*>(w.pose_slot.p);
    cp.poses = static_cast<const double*>(ctx->ba.poses.p);
    cp.patch_src = static_cast<const int*>(ctx->ba.patch_src.p);
    cp.patch_x = static_cast<const double*>(ctx->ba.px.p);
    cp.patch_y = static_cast<const double*>(ctx->ba.py.p);
    cp.depth = static_cast<const double*>(ctx->ba.depth.p);
    cp.K = static_cast<const double*>(ctx->ba.K.p);
    cp.patch_feats = static_cast<const float*>(w.patch_feats.p);
    cp.n_patches = w.n_patches;
    cp.out = out ? out : static_cast<float*>(w.corr.p);
    return cp;
}

pvo_dev::BAParams window_ba_params(pvo_ctx* ctx, int iterations, double damping) {
    Window& w = ctx->win;
    BABuffers& B = ctx->ba;
    const int np = 6 * w.plan.n_free_poses;
    pvo_dev::BAParams a;
    a.n_poses = w.n_poses;
    a.n_patches = w.n_patches;
    a.n_edges = w.n_edges;
    a.n_free_poses = w.plan.n_free_poses;
    a.n_free_depths = w.plan.n_free_depths;
    a.poses = static_cast<double*>(B.poses.p);
    a.pose_free_slot = static_cast<const int*>(B.free_slot.p);
    a.patch_src = static_cast<const int*>(B.patch_src.p);
    a.patch_x = static_cast<const double*>(B.px.p);
    a.patch_y = static_cast<const double*>(B.py.p);
    a.depth = static_cast<double*>(B.depth.p);
    a.depth_slot = static_cast<const int*>(B.depth_slot.p);
    a.patch_edge_begin = static_cast<const int*>(B.edge_begin.p);
    a.e_patch = static_cast<const int*>(B.e_patch.p);
    a.e_pose = static_cast<const int*>(B.e_pose.p);
    a.e_in = static_cast<const double*>(B.e_in.p);
    a.e_weight_in = static_cast<const double*>(B.e_w.p);
    a.e_target = static_cast<double*>(B.e_target.p);
    a.e_weight = static_cast<double*>(B.e_weight.p);
    a.cand_poses = static_cast<double*>(B.cand_poses.p);
    a.cand_depth = static_cast<double*>(B.cand_depth.p);
    a.patch_v = static_cast<double*>(B.patch_v.p);
    a.patch_h = static_cast<double*>(B.patch_h.p);
    a.patch_bd = static_cast<double*>(B.patch_bd.p);
    a.status2 = B.status2.as<int>(2);
    a.attempts = B.attempts.as<int>(1);
    a.phase_clocks = ctx->tracing ? B.clocks.as<long long>(128) : nullptr;
    if (!w.plan.large) {
        const int grid = pvo_dev::ba_grid_size(w.n_patches, w.plan.n_free_poses, w.n_poses, ctx->num_sms);
        a.partials = B.partials.as<double>(pvo_dev::ba_partials_doubles(w.plan.n_free_poses, grid));
        a.system = B.system.as<double>((size_t)np * (np + 1) / 2 + np + 1);
    }
    a.delta = B.delta.as<double>(std::max(np, 1));
    a.residual_norms = B.norms.as<double>(iterations + 2);
    a.n_norms = B.n_norms.as<int>(1);
    a.status = ctx->d_status;
    std::memcpy(a.K, w.shape.K, sizeof(a.K));
    a.image_w = w.shape.image_w;
    a.image_h = w.shape.image_h;
    a.freeze_targets = 1;
    a.damping = damping;
    a.iterations = iterations;
    return a;
}
}  // namespace

int pvo_window_correlate(pvo_ctx* ctx, float* out, int memspace) {
    return guarded([&] {
        bind(ctx);
        Window& w = ctx->win;
        if (!w.loaded) fail(PVO_INVALID_ARGUMENT, "window: nothing loaded");
        reset_status(ctx);
        run_corr(ctx, window_corr_params(ctx, memspace == PVO_DEVICE ? out : nullptr));
        if (out && memspace != PVO_DEVICE) {
            download(ctx, out, static_cast<float*>(w.corr.p), (size_t)w.n_edges * 2 * 9 * 49);
            if (read_status(ctx)) fail(PVO_INVALID_ARGUMENT, "correlate: non-finite reprojection");
        }
    });
}

int pvo_window_iteration(pvo_ctx* ctx, int iterations, double damping, float* corr_out, int corr_memspace) {
    return guarded([&] {
        bind(ctx);
        Window& w = ctx->win;
        if (!w.loaded) fail(PVO_INVALID_ARGUMENT, "window: nothing loaded");
        if (iterations < 0) fail(PVO_INVALID_ARGUMENT, "ba: negative iteration count");
        if (iterations > PVO_MAX_WINDOW_ITERATIONS) fail(PVO_INVALID_ARGUMENT, "ba: too many iterations");
        reset_status(ctx);
        record_timing(ctx, 0);
        const bool readback = corr_out && corr_memspace != PVO_DEVICE;
        const size_t vol_edge = (size_t)2 * 9 * 49;
        // the split needs the TMA path (the generic kernel has no edge order)
        const bool split = readback && w.half > 0 && ctx->maps_ok &&
                           encode_patch_map(ctx, static_cast<const float*>(w.patch_feats.p), w.n_patches);
        if (split) {
            // two launches over the halves of the edge range: the first half's
            // read-back runs on the copy stream while the second is correlated
            const int* oh = static_cast<const int*>(w.order_half.p);
            pvo_dev::CorrTmaParams c1 = window_corr_params(ctx, nullptr), c2 = c1;
            c1.n_edges = w.half;
            c1.order = oh;
            c2.n_edges = w.n_edges - w.half;
            c2.order = oh + w.half;
            run_corr(ctx, c1, w.n_edges);
            cuda_check(cudaEventRecord(ctx->ev_corr, ctx->stream), "event");
            run_corr(ctx, c2, w.n_edges);
            record_timing(ctx, 1);
            cuda_check(cudaEventRecord(ctx->ev_corr2, ctx->stream), "event");
            float* vol = static_cast<float*>(w.corr.p);
            cuda_check(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_corr, 0), "stream wait");
            cuda_check(cudaMemcpyAsync(corr_out, vol, sizeof(float) * w.half * vol_edge, cudaMemcpyDeviceToHost,
                                       ctx->copy_stream),
                       "D2H");
            cuda_check(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_corr2, 0), "stream wait");
            cuda_check(cudaMemcpyAsync(corr_out + (size_t)w.half * vol_edge, vol + (size_t)w.half * vol_edge,
                                       sizeof(float) * (size_t)(w.n_edges - w.half) * vol_edge, cudaMemcpyDeviceToHost,
                                       ctx->copy_stream),
                       "D2H");
            cuda_check(cudaEventRecord(ctx->ev_copy, ctx->copy_stream), "event");
        } else {
            run_corr(ctx, window_corr_params(ctx, corr_memspace == PVO_DEVICE ? corr_out : nullptr));
            record_timing(ctx, 1);
        }
        if (readback && !split) {  // the volume's D2H runs on the copy stream, under BA
            cuda_check(cudaEventRecord(ctx->ev_corr, ctx->stream), "event");
            cuda_check(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_corr, 0), "stream wait");
            cuda_check(cudaMemcpyAsync(corr_out, w.corr.p, sizeof(float) * (size_t)w.n_edges * 2 * 9 * 49,
                                       cudaMemcpyDeviceToHost, ctx->copy_stream),
                       "D2H");
            cuda_check(cudaEventRecord(ctx->ev_copy, ctx->copy_stream), "event");
        }
        pvo_dev::BAParams a = window_ba_params(ctx, iterations, damping);
        launch_ba_checked(ctx, a, w.plan);
        record_timing(ctx, 2);
        ctx->timing_pending = ctx->timing;
        if (readback) cuda_check(cudaStreamWaitEvent(ctx->stream, ctx->ev_copy, 0), "stream wait");
    });
}

// optimize_window's iterations on the resident window without the correlation
// pass (the per-frame pipeline: propose -> BA, pipeline.cpp:183-198)
int pvo_window_ba(pvo_ctx* ctx, int iterations, double damping) {
    return guarded([&] {
        bind(ctx);
        Window& w = ctx->win;
        if (!w.loaded) fail(PVO_INVALID_ARGUMENT, "window: nothing loaded");
        if (iterations < 0) fail(PVO_INVALID_ARGUMENT, "ba: negative iteration count");
        if (iterations > PVO_MAX_WINDOW_ITERATIONS) fail(PVO_INVALID_ARGUMENT, "ba: too many iterations");
        reset_status(ctx);
        pvo_dev::BAParams a = window_ba_params(ctx, iterations, damping);
        launch_ba_checked(ctx, a, w.plan);
    });
}

int pvo_window_read(pvo_ctx* ctx, double* poses, double* depth, double* residual_norms, int* n_norms) {
    return guarded([&] {
        bind(ctx);
        Window& w = ctx->win;
        if (!w.loaded) fail(PVO_INVALID_ARGUMENT, "window: nothing loaded");
        // status, state and norms: async copies into page-locked staging, one sync
        const size_t norms_cap = ctx->ba.norms.cap / sizeof(double);
        const size_t np7 = (size_t)w.n_poses * 7, nd = w.n_patches;
        double* st = static_cast<double*>(ctx->stage(sizeof(double) * (2 + np7 + nd + norms_cap)));
        int* st_i = reinterpret_cast<int*>(st);  // [status, n_norms]
        double* st_p = st + 2;
        double* st_d = st_p + np7;
        double* st_n = st_d + nd;
        download(ctx, st_i, ctx->d_status, 1);
        download(ctx, st_i + 1, static_cast<int*>(ctx->ba.n_norms.p), 1);
        if (poses) download(ctx, st_p, static_cast<double*>(ctx->ba.poses.p), np7);
        if (depth) download(ctx, st_d, static_cast<double*>(ctx->ba.depth.p), nd);
        if (residual_norms && norms_cap) download(ctx, st_n, static_cast<double*>(ctx->ba.norms.p), norms_cap);
        sync(ctx);
        const int status = st_i[0], n = st_i[1];
        if (status & (1 << pvo_dev::kDevBadCoords)) fail(PVO_INVALID_ARGUMENT, "correlate: non-finite reprojection");
        raise_ba_status(status);
        if (poses) std::memcpy(poses, st_p, sizeof(double) * np7);
        if (depth) std::memcpy(depth, st_d, sizeof(double) * nd);
        const size_t n_copy = std::min<size_t>(std::min<size_t>(n, norms_cap), PVO_MAX_WINDOW_ITERATIONS + 2);
        if (residual_norms && n > 0) std::memcpy(residual_norms, st_n, sizeof(double) * n_copy);
        if (n_norms) *n_norms = n;
    });
}

// ---- feature extraction (features.cpp:55-235) -----------
// The frame's pyramid from its image, on the device, into frame-store `slot`
// (+ its Gram terms).  The store must have been reserved with C = 25 * bc and
// level sizes (iw/4, ih/4), (iw/16, ih/16).
int pvo_frames_extract(pvo_ctx* ctx, int slot, const float* image, int iw, int ih, int base_channels, int memspace) {
    return guarded([&] {
        bind(ctx);
        if (base_channels != 1 && base_channels != 3) fail(PVO_INVALID_ARGUMENT, "features: base channel count must be 1 or 3");
        if (iw < 12 || ih < 12) fail(PVO_INVALID_ARGUMENT, "features: image too small");
        if (slot < 0 || slot >= ctx->nf) fail(PVO_OUT_OF_RANGE, "frames: slot out of range");
        if (ctx->C != 25 * base_channels || ctx->w0 != iw / 4 || ctx->h0 != ih / 4 || ctx->w1 != iw / 16 ||
            ctx->h1 != ih / 16)
            fail(PVO_INVALID_ARGUMENT, "frames_extract: frame store shape does not match the image / channels");
        const float* dimg = memspace == PVO_DEVICE ? image : upload(ctx, ctx->s0, image, (size_t)iw * ih);
        float* scratch = ctx->s1.as<float>(pvo_dev::extract_scratch_floats(iw, ih, base_channels));
        const size_t c0 = (size_t)ctx->w0 * ctx->h0, c1 = (size_t)ctx->w1 * ctx->h1;
        float* f0 = static_cast<float*>(ctx->feat0.p) + (size_t)slot * c0 * ctx->C;
        float* f1 = static_cast<float*>(ctx->feat1.p) + (size_t)slot * c1 * ctx->C;
        cuda_check(pvo_dev::launch_extract_features(dimg, iw, ih, base_channels, scratch, f0, f1, ctx->stream),
                   "feature extraction");
        ctx->launches += base_channels == 3 ? 8 : 7;
        float* g0 = static_cast<float*>(ctx->gram0.p) + (size_t)slot * pvo_dev::gram_stride(ctx->w0) * ctx->h0 * 8;
        float* g1 = static_cast<float*>(ctx->gram1.p) + (size_t)slot * pvo_dev::gram_stride(ctx->w1) * ctx->h1 * 8;
        compute_gram(ctx, f0, g0, f1, g1, ctx->w0, ctx->h0, ctx->w1, ctx->h1, ctx->C);
        if (memspace != PVO_DEVICE) sync(ctx);
    });
}

// A slot's pyramid back to the host (level0 [H0][W0][C], level1 [H1][W1][C]).
int pvo_frames_download(pvo_ctx* ctx, int slot, float* level0, float* level1) {
    return guarded([&] {
        bind(ctx);
        if (slot < 0 || slot >= ctx->nf) fail(PVO_OUT_OF_RANGE, "frames: slot out of range");
        const size_t c0 = (size_t)ctx->w0 * ctx->h0 * ctx->C, c1 = (size_t)ctx->w1 * ctx->h1 * ctx->C;
        if (level0) download(ctx, level0, static_cast<const float*>(ctx->feat0.p) + (size_t)slot * c0, c0);
        if (level1) download(ctx, level1, static_cast<const float*>(ctx->feat1.p) + (size_t)slot * c1, c1);
        sync(ctx);
    });
}

// crop_patch_features (features.cpp:204-224) of n patches from frame-store slot
// `slot`: centroids [n][2] -> the 3x3 grid (Patch::make) -> out [n][2][9][C].
int pvo_crop_patches(pvo_ctx* ctx, int slot, int n, const double* centroids, float* out, int memspace) {
    return guarded([&] {
        bind(ctx);
        if (slot < 0 || slot >= ctx->nf) fail(PVO_OUT_OF_RANGE, "frames: slot out of range");
        if (n <= 0) return;
        std::vector<double> px(9 * (size_t)n), py(9 * (size_t)n);
        for (int k = 0; k < n; ++k)
            for (int row = 0; row < 3; ++row)
                for (int col = 0; col < 3; ++col) {
                    px[9 * (size_t)k + 3 * row + col] = centroids[2 * k] + col - 1.0;
                    py[9 * (size_t)k + 3 * row + col] = centroids[2 * k + 1] + row - 1.0;
                }
        const double* dx = upload(ctx, ctx->s2, px.data(), px.size());
        const double* dy = upload(ctx, ctx->s3, py.data(), py.size());
        const size_t c0 = (size_t)ctx->w0 * ctx->h0, c1 = (size_t)ctx->w1 * ctx->h1;
        const float* f0 = static_cast<const float*>(ctx->feat0.p) + (size_t)slot * c0 * ctx->C;
        const float* f1 = static_cast<const float*>(ctx->feat1.p) + (size_t)slot * c1 * ctx->C;
        const size_t total = (size_t)n * 2 * 9 * ctx->C;
        float* dout = memspace == PVO_DEVICE ? out : ctx->s4.as<float>(total);
        cuda_check(pvo_dev::launch_crop_patches(n, dx, dy, f0, ctx->w0, ctx->h0, f1, ctx->w1, ctx->h1, ctx->C, dout,
                                                ctx->stream),
                   "crop");
        ctx->launches += 1;
        if (memspace != PVO_DEVICE) download(ctx, out, dout, total);
        sync(ctx);
    });
}

// ---- flow-provider measurement (flow_provider.cpp:150-312) -------------------
int pvo_measure_batch(pvo_ctx* ctx, int n_edges, int n_patches, int p, const int* e_patch, const int* e_slot,
                      const double* centers, const uint8_t* behind, const float* patch_feats, double* delta,
                      double* weight, uint8_t* flags) {
    return guarded([&] {
        bind(ctx);
        ensure_p3(p);
        if (ctx->nf == 0) fail(PVO_INVALID_ARGUMENT, "measure_batch: frame store is empty (pvo_frames_reserve)");
        if (n_edges < 0 || n_patches < 0) fail(PVO_INVALID_ARGUMENT, "measure_batch: bad sizes");
        if (n_edges == 0) return;
        if (ctx->C > 128) fail(PVO_UNSUPPORTED, "measure_batch: more than 128 channels");
        for (int e = 0; e < n_edges; ++e) {
            if (e_patch[e] < 0 || e_patch[e] >= n_patches) fail(PVO_OUT_OF_RANGE, "measure_batch: bad patch index");
            if (e_slot[e] < 0 || e_slot[e] >= ctx->nf) fail(PVO_OUT_OF_RANGE, "measure_batch: bad frame slot");
        }
        pvo_dev::MeasureParams m;
        m.n_edges = n_edges;
        m.channels = ctx->C;
        m.e_patch = upload(ctx, ctx->s0, e_patch, n_edges);
        m.e_slot = upload(ctx, ctx->s1, e_slot, n_edges);
        m.centers = upload(ctx, ctx->s2, centers, (size_t)n_edges * 2);
        m.behind = behind ? upload(ctx, ctx->s5, behind, n_edges) : nullptr;
        m.patch_feats = upload(ctx, ctx->s3, patch_feats, (size_t)n_patches * 2 * 9 * ctx->C);
        m.feat0 = static_cast<const float*>(ctx->feat0.p);
        m.feat1 = static_cast<const float*>(ctx->feat1.p);
        m.w0 = ctx->w0;
        m.h0 = ctx->h0;
        m.w1 = ctx->w1;
        m.h1 = ctx->h1;
        double* dd = ctx->s4.as<double>((size_t)n_edges * 4);
        m.delta = dd;
        m.weight = dd + (size_t)n_edges * 2;
        m.flags = ctx->s6.as<uint8_t>(n_edges);
        m.status = ctx->d_status;
        reset_status(ctx);
        cuda_check(pvo_dev::launch_measure(m, ctx->stream), "measure kernel");
        ctx->launches += 1;
        download(ctx, delta, m.delta, (size_t)n_edges * 2);
        download(ctx, weight, m.weight, (size_t)n_edges * 2);
        if (flags) download(ctx, flags, m.flags, n_edges);
        if (read_status(ctx) & (1 << pvo_dev::kDevBadCoords)) fail(PVO_INVALID_ARGUMENT, "measure: non-finite centre");
    });
}

// CorrelationFlowProvider::propose over the resident window's edges: measure at
// the current state and store the revisions (delta, weight) as the window's
// edge revisions, which the next pvo_window_iteration freezes into targets
// (pipeline.cpp:183-198: propose -> set_revision -> optimize_window).
int pvo_window_propose(pvo_ctx* ctx, double* delta_out, double* weight_out, uint8_t* flags_out) {
    return guarded([&] {
        bind(ctx);
        Window& w = ctx->win;
        if (!w.loaded) fail(PVO_INVALID_ARGUMENT, "window: nothing loaded");
        if (ctx->C > 128) fail(PVO_UNSUPPORTED, "window_propose: more than 128 channels");
        BABuffers& B = ctx->ba;
        pvo_dev::MeasureParams m;
        m.n_edges = w.n_edges;
        m.channels = ctx->C;
        m.e_patch = static_cast<const int*>(B.e_patch.p);
        m.e_pose = static_cast<const int*>(B.e_pose.p);
        m.pose_slot = static_cast<const int*>(w.pose_slot.p);
        m.poses = static_cast<const double*>(B.poses.p);
        m.patch_src = static_cast<const int*>(B.patch_src.p);
        m.patch_x = static_cast<const double*>(B.px.p);
        m.patch_y = static_cast<const double*>(B.py.p);
        m.depth = static_cast<const double*>(B.depth.p);
        m.K = static_cast<const double*>(B.K.p);
        m.patch_feats = static_cast<const float*>(w.patch_feats.p);
        m.feat0 = static_cast<const float*>(ctx->feat0.p);
        m.feat1 = static_cast<const float*>(ctx->feat1.p);
        m.w0 = ctx->w0;
        m.h0 = ctx->h0;
        m.w1 = ctx->w1;
        m.h1 = ctx->h1;
        m.delta = static_cast<double*>(B.e_in.p);  // the window's revisions, edge order = load order
        m.weight = static_cast<double*>(B.e_w.p);
        m.flags = w.flags.as<uint8_t>(w.n_edges);
        m.status = ctx->d_status;
        cuda_check(pvo_dev::launch_measure(m, ctx->stream), "measure kernel");
        ctx->launches += 1;
        if (delta_out) download(ctx, delta_out, m.delta, (size_t)w.n_edges * 2);
        if (weight_out) download(ctx, weight_out, m.weight, (size_t)w.n_edges * 2);
        if (flags_out) download(ctx, flags_out, m.flags, w.n_edges);
        if (delta_out || weight_out || flags_out) sync(ctx);
    });
}

// ---- OracleFlowProvider::propose (flow_provider.cpp:34-93) ---------------------
namespace {
struct V2Args {  // built as V2Args(a(), b()): the reference's Vec2(gauss(rng_), gauss(rng_)) evaluation order
    double x, y;
    V2Args(double a, double b) : x(a), y(b) {}
};
}  // namespace

int pvo_oracle_seed(pvo_ctx* ctx, uint64_t seed) {
    return guarded([&] { ctx->oracle_rng.seed(seed); });
}

// Simulator revisions for every edge of the resident window: ground truth
// (scene poses of the window's pose slots gt_poses [N][7], scene inverse depth
// gt_inv_depth [P]) minus the current reprojection, + N(0, sigma^2) noise,
// clamped to +-64 px, exactly floor(fraction * E) uniform outliers — the RNG
// stream is the reference's (a context-owned mt19937_64 that persists across
// calls, like the provider's member; the draws are consumed on the host in
// the reference's order between two device passes).  The revisions replace
// the window's deltas / weights (as pvo_window_propose).
int pvo_window_oracle_propose(pvo_ctx* ctx, const double* gt_poses, const double* gt_inv_depth, double flow_sigma,
                              double outlier_fraction, double* delta_out, double* weight_out) {
    return guarded([&] {
        bind(ctx);
        Window& w = ctx->win;
        if (!w.loaded) fail(PVO_INVALID_ARGUMENT, "window: nothing loaded");
        BABuffers& B = ctx->ba;
        const int E = w.n_edges;
        pvo_dev::OracleParams o;
        o.n_edges = E;
        o.e_patch = static_cast<const int*>(B.e_patch.p);
        o.e_pose = static_cast<const int*>(B.e_pose.p);
        o.patch_src = static_cast<const int*>(B.patch_src.p);
        o.patch_x = static_cast<const double*>(B.px.p);
        o.patch_y = static_cast<const double*>(B.py.p);
        o.depth = static_cast<const double*>(B.depth.p);
        o.poses = static_cast<const double*>(B.poses.p);
        o.K = static_cast<const double*>(B.K.p);
        o.gt_poses = upload(ctx, ctx->s0, gt_poses, 7 * (size_t)w.n_poses);
        o.gt_depth = upload(ctx, ctx->s1, gt_inv_depth, w.n_patches);
        o.flow_sigma = flow_sigma;
        o.weight_in_range = std::clamp(1.0 / (1.0 + flow_sigma * flow_sigma), 0.01, 0.99);
        o.behind = ctx->s5.as<uint8_t>(std::max(E, 1));
        o.delta = static_cast<double*>(B.e_in.p);
        o.weight = static_cast<double*>(B.e_w.p);
        cuda_check(pvo_dev::launch_oracle_propose(o, 0, ctx->stream), "oracle propose");
        std::vector<uint8_t> behind(E);
        download(ctx, behind.data(), o.behind, E);
        sync(ctx);
        // host: the RNG stream in the reference's order
        std::normal_distribution<double> gauss(0.0, flow_sigma);
        std::uniform_real_distribution<double> uniform(-32.0, 32.0);
        std::vector<double> noise(2 * (size_t)E, 0.0), odelta;
        std::vector<uint8_t> omask;
        if (flow_sigma > 0)
            for (int e = 0; e < E; ++e)
                if (!behind[e]) {
                    const V2Args n(gauss(ctx->oracle_rng), gauss(ctx->oracle_rng));
                    noise[2 * e] = n.x;
                    noise[2 * e + 1] = n.y;
                }
        const size_t num_outliers = static_cast<size_t>(outlier_fraction * static_cast<double>(E));
        if (num_outliers > 0) {
            std::vector<size_t> index(E);
            for (size_t i = 0; i < index.size(); ++i) index[i] = i;
            std::shuffle(index.begin(), index.end(), ctx->oracle_rng);
            omask.assign(E, 0);
            odelta.assign(2 * (size_t)E, 0.0);
            for (size_t i = 0; i < num_outliers; ++i) {
                const V2Args u(uniform(ctx->oracle_rng), uniform(ctx->oracle_rng));
                omask[index[i]] = 1;
                odelta[2 * index[i]] = u.x;
                odelta[2 * index[i] + 1] = u.y;
            }
            o.outlier = upload(ctx, ctx->s6, omask.data(), omask.size());
            o.outlier_delta = upload(ctx, ctx->s7, odelta.data(), odelta.size());
        }
        if (flow_sigma > 0) o.noise = upload(ctx, ctx->s8, noise.data(), noise.size());
        cuda_check(pvo_dev::launch_oracle_propose(o, 1, ctx->stream), "oracle propose");
        ctx->launches += 2;
        if (delta_out) download(ctx, delta_out, o.delta, 2 * (size_t)E);
        if (weight_out) download(ctx, weight_out, o.weight, 2 * (size_t)E);
        sync(ctx);
    });
}

// ---- batch of independent windows -------------------------------------------
int pvo_batch_load(pvo_ctx* ctx, int n_windows, const int* pose_off, const int* patch_off, const int* edge_off,
                   const double* poses, const uint8_t* fixed, const int* pose_slot, int p, const int* src,
                   const double* px, const double* py, const double* depth, const float* patch_feats,
                   const int* e_patch, const int* e_pose, const double* e_delta, const double* e_weight,
                   const double* K, int image_w, int image_h) {
    return guarded([&] {
        bind(ctx);
        if (ctx->nf == 0) fail(PVO_INVALID_ARGUMENT, "batch_load: frame store is empty (pvo_frames_reserve)");
        if (n_windows < 1) fail(PVO_INVALID_ARGUMENT, "batch_load: no windows");
        if (p != 3) fail(PVO_UNSUPPORTED, "the sm_100a kernels implement 3x3 patches (p = 3)");
        Batch& B = ctx->bat;
        B.loaded = false;
        B.n_windows = n_windows;
        B.pose_off.assign(pose_off, pose_off + n_windows + 1);
        B.patch_off.assign(patch_off, patch_off + n_windows + 1);
        B.edge_off.assign(edge_off, edge_off + n_windows + 1);
        for (int w = 0; w < n_windows; ++w)
            if (pose_off[w + 1] < pose_off[w] || patch_off[w + 1] < patch_off[w] || edge_off[w + 1] < edge_off[w] ||
                pose_off[0] != 0 || patch_off[0] != 0 || edge_off[0] != 0)
                fail(PVO_INVALID_ARGUMENT, "batch_load: offsets must start at 0 and be non-decreasing");
        const int NP = pose_off[n_windows], NK = patch_off[n_windows], NE = edge_off[n_windows];
        B.n_poses = NP;
        B.n_patches = NK;
        B.n_edges = NE;
        for (int i = 0; i < NP; ++i)
            if (pose_slot[i] < 0 || pose_slot[i] >= ctx->nf) fail(PVO_OUT_OF_RANGE, "batch_load: bad frame slot");
        // per-window plans (validation, free slots, CSR) on the window-local views
        std::vector<int> free_slot(NP), depth_slot(NK), edge_begin(NK + n_windows);
        std::vector<int> g_patch(NE), g_pose(NE), g_src(NK);
        std::vector<size_t> v_off(n_windows + 1, 0), part_off(n_windows + 1, 0), sys_off(n_windows + 1, 0);
        std::vector<int> n_free(n_windows), n_free_d(n_windows);
        B.max_free = 0;
        B.max_poses = 0;
        for (int w = 0; w < n_windows; ++w) {
            const int po = pose_off[w], ko = patch_off[w], eo = edge_off[w];
            HostProblem pr{pose_off[w + 1] - po, poses + 7 * (size_t)po, fixed + po, patch_off[w + 1] - ko, p,
                           src + ko, px + 9 * (size_t)ko, py + 9 * (size_t)ko, depth + ko, nullptr,
                           edge_off[w + 1] - eo, e_patch + eo, e_pose + eo, e_delta + 2 * (size_t)eo,
                           e_weight + 2 * (size_t)eo};
            std::memcpy(pr.K, K, sizeof(pr.K));
            pr.image_w = image_w;
            pr.image_h = image_h;
            validate(pr);
            const Plan pl = make_plan(pr, false);
            if (!pl.sorted) fail(PVO_INVALID_ARGUMENT, "batch_load: edges must be grouped by patch (reference order)");
            if (pl.large) fail(PVO_UNSUPPORTED, "batch_load: a window beyond 16 free poses / 128 poses");
            std::copy(pl.free_slot.begin(), pl.free_slot.end(), free_slot.begin() + po);
            std::copy(pl.depth_slot.begin(), pl.depth_slot.end(), depth_slot.begin() + ko);
            std::copy(pl.edge_begin.begin(), pl.edge_begin.end(), edge_begin.begin() + ko + w);
            for (int e = eo; e < edge_off[w + 1]; ++e) {
                g_patch[e] = e_patch[e] + ko;
                g_pose[e] = e_pose[e] + po;
            }
            for (int k = ko; k < patch_off[w + 1]; ++k) g_src[k] = src[k] + po;
            n_free[w] = pl.n_free_poses;
            n_free_d[w] = pl.n_free_depths;
            const int np = 6 * pl.n_free_poses;
            v_off[w + 1] = v_off[w] + (size_t)pr.n_patches * std::max(np, 1);
            part_off[w + 1] = part_off[w] + pvo_dev::ba_partials_doubles(pl.n_free_poses, 1);
            sys_off[w + 1] = sys_off[w] + (size_t)np * (np + 1) / 2 + np + 1;
            B.max_free = std::max(B.max_free, pl.n_free_poses);
            B.max_poses = std::max(B.max_poses, pr.n_poses);
        }
        // device arrays
        upload(ctx, B.poses, poses, (size_t)NP * 7);
        upload(ctx, B.init_poses, poses, (size_t)NP * 7);
        upload(ctx, B.free_slot, free_slot.data(), NP);
        upload(ctx, B.src, src, NK);
        upload(ctx, B.px, px, (size_t)NK * 9);
        upload(ctx, B.py, py, (size_t)NK * 9);
        upload(ctx, B.depth, depth, NK);
        upload(ctx, B.init_depth, depth, NK);
        upload(ctx, B.depth_slot, depth_slot.data(), NK);
        upload(ctx, B.edge_begin, edge_begin.data(), edge_begin.size());
        upload(ctx, B.e_patch, e_patch, NE);
        upload(ctx, B.e_pose, e_pose, NE);
        upload(ctx, B.e_in, e_delta, (size_t)NE * 2);
        upload(ctx, B.e_w, e_weight, (size_t)NE * 2);
        upload(ctx, B.g_e_patch, g_patch.data(), NE);
        upload(ctx, B.g_e_pose, g_pose.data(), NE);
        upload(ctx, B.g_src, g_src.data(), NK);
        upload(ctx, B.pose_slot, pose_slot, NP);
        upload(ctx, B.patch_feats, patch_feats, (size_t)NK * 2 * 9 * ctx->C);
        upload(ctx, B.K, K, 4);
        std::vector<int> eslot(NE);
        for (int e = 0; e < NE; ++e) eslot[e] = pose_slot[g_pose[e]];
        const std::vector<int> order = slot_order(NE, eslot.data());
        upload(ctx, B.order, order.data(), order.size());
        double* d_poses = static_cast<double*>(B.poses.p);
        double* e_target = B.e_target.as<double>((size_t)NE * 2);
        double* e_weff = B.e_weight.as<double>((size_t)NE * 2);
        double* cand_poses = B.cand_poses.as<double>((size_t)NP * 7);
        double* cand_depth = B.cand_depth.as<double>(NK);
        double* patch_v = B.patch_v.as<double>(std::max<size_t>(v_off[n_windows], 1));
        double* patch_h = B.patch_h.as<double>(NK);
        double* patch_bd = B.patch_bd.as<double>(NK);
        double* partials = B.partials.as<double>(std::max<size_t>(part_off[n_windows], 1));
        double* system = B.system.as<double>(std::max<size_t>(sys_off[n_windows], 1));
        double* delta = B.delta.as<double>((size_t)n_windows * std::max(6 * B.max_free, 1));
        double* norms = B.norms.as<double>((size_t)n_windows * Batch::kNormStride);
        int* n_norms = B.n_norms.as<int>(n_windows);
        int* status2 = B.status2.as<int>(2 * (size_t)n_windows);
        int* attempts = B.attempts.as<int>(n_windows);
        int* status = B.status.as<int>(n_windows);
        B.corr.get(sizeof(float) * (size_t)NE * 2 * 9 * 49);
        B.hparams.assign(n_windows, pvo_dev::BAParams{});
        for (int w = 0; w < n_windows; ++w) {
            const int po = pose_off[w], ko = patch_off[w], eo = edge_off[w];
            pvo_dev::BAParams& a = B.hparams[w];
            a.n_poses = pose_off[w + 1] - po;
            a.n_patches = patch_off[w + 1] - ko;
            a.n_edges = edge_off[w + 1] - eo;
            a.n_free_poses = n_free[w];
            a.n_free_depths = n_free_d[w];
            a.poses = d_poses + 7 * (size_t)po;
            a.pose_free_slot = static_cast<const int*>(B.free_slot.p) + po;
            a.patch_src = static_cast<const int*>(B.src.p) + ko;
            a.patch_x = static_cast<const double*>(B.px.p) + 9 * (size_t)ko;
            a.patch_y = static_cast<const double*>(B.py.p) + 9 * (size_t)ko;
            a.depth = static_cast<double*>(B.depth.p) + ko;
            a.depth_slot = static_cast<const int*>(B.depth_slot.p) + ko;
            a.patch_edge_begin = static_cast<const int*>(B.edge_begin.p) + ko + w;
            a.e_patch = static_cast<const int*>(B.e_patch.p) + eo;
            a.e_pose = static_cast<const int*>(B.e_pose.p) + eo;
            a.e_in = static_cast<const double*>(B.e_in.p) + 2 * (size_t)eo;
            a.e_weight_in = static_cast<const double*>(B.e_w.p) + 2 * (size_t)eo;
            a.e_target = e_target + 2 * (size_t)eo;
            a.e_weight = e_weff + 2 * (size_t)eo;
            std::memcpy(a.K, K, sizeof(a.K));
            a.image_w = image_w;
            a.image_h = image_h;
            a.freeze_targets = 1;
            a.cand_poses = cand_poses + 7 * (size_t)po;
            a.cand_depth = cand_depth + ko;
            a.patch_v = patch_v + v_off[w];
            a.patch_h = patch_h + ko;
            a.patch_bd = patch_bd + ko;
            a.partials = partials + part_off[w];
            a.system = system + sys_off[w];
            a.delta = delta + (size_t)w * std::max(6 * B.max_free, 1);
            a.residual_norms = norms + (size_t)w * Batch::kNormStride;
            a.n_norms = n_norms + w;
            a.status = status + w;
            a.status2 = status2 + 2 * w;
            a.attempts = attempts + w;
        }
        B.iterations = -1;
        sync(ctx);
        B.loaded = true;
    });
}

namespace {
void batch_params(pvo_ctx* ctx, int iterations, double damping) {
    Batch& B = ctx->bat;
    if (B.iterations == iterations && B.damping == damping) return;
    if (iterations + 2 > Batch::kNormStride) fail(PVO_INVALID_ARGUMENT, "batch: too many iterations");
    for (auto& a : B.hparams) {
        a.iterations = iterations;
        a.damping = damping;
    }
    upload(ctx, B.params, B.hparams.data(), B.hparams.size());
    B.iterations = iterations;
    B.damping = damping;
}
}  // namespace

int pvo_batch_reset(pvo_ctx* ctx) {
    return guarded([&] {
        bind(ctx);
        Batch& B = ctx->bat;
        if (!B.loaded) fail(PVO_INVALID_ARGUMENT, "batch: nothing loaded");
        cuda_check(cudaMemcpyAsync(B.poses.p, B.init_poses.p, sizeof(double) * 7 * B.n_poses,
                                   cudaMemcpyDeviceToDevice, ctx->stream), "state");
        cuda_check(cudaMemcpyAsync(B.depth.p, B.init_depth.p, sizeof(double) * B.n_patches, cudaMemcpyDeviceToDevice,
                                   ctx->stream), "state");
    });
}

int pvo_batch_iteration(pvo_ctx* ctx, int iterations, double damping, float* corr_out, int corr_memspace) {
    return guarded([&] {
        bind(ctx);
        Batch& B = ctx->bat;
        if (!B.loaded) fail(PVO_INVALID_ARGUMENT, "batch: nothing loaded");
        if (iterations < 0) fail(PVO_INVALID_ARGUMENT, "ba: negative iteration count");
        batch_params(ctx, iterations, damping);
        reset_status(ctx);
        cuda_check(cudaMemsetAsync(B.status.p, 0, sizeof(int) * B.n_windows, ctx->stream), "memset");
        cuda_check(cudaMemsetAsync(B.status2.p, 0, sizeof(int) * 2 * B.n_windows, ctx->stream), "memset");
        cuda_check(cudaMemsetAsync(B.n_norms.p, 0, sizeof(int) * B.n_windows, ctx->stream), "memset");
        record_timing(ctx, 0);
        pvo_dev::CorrTmaParams cp;
        cp.n_edges = B.n_edges;
        cp.order = static_cast<const int*>(B.order.p);
        cp.e_patch = static_cast<const int*>(B.g_e_patch.p);
        cp.e_pose = static_cast<const int*>(B.g_e_pose.p);
        cp.pose_slot = static_cast<const int*>(B.pose_slot.p);
        cp.poses = static_cast<const double*>(B.poses.p);
        cp.patch_src = static_cast<const int*>(B.g_src.p);
        cp.patch_x = static_cast<const double*>(B.px.p);
        cp.patch_y = static_cast<const double*>(B.py.p);
        cp.depth = static_cast<const double*>(B.depth.p);
        cp.K = static_cast<const double*>(B.K.p);
        cp.patch_feats = static_cast<const float*>(B.patch_feats.p);
        cp.n_patches = B.n_patches;
        float* vol = corr_memspace == PVO_DEVICE && corr_out ? corr_out : static_cast<float*>(B.corr.p);
        cp.out = vol;
        run_corr(ctx, cp);
        record_timing(ctx, 1);
        cuda_check(pvo_dev::launch_ba_batch(static_cast<const pvo_dev::BAParams*>(B.params.p), B.n_windows,
                                            B.max_free, B.max_poses, ctx->stream),
                   "ba batch kernel");
        ctx->launches += 1;
        record_timing(ctx, 2);
        ctx->timing_pending = ctx->timing;
        if (corr_out && corr_memspace != PVO_DEVICE) download(ctx, corr_out, vol, (size_t)B.n_edges * 2 * 9 * 49);
    });
}

int pvo_batch_read(pvo_ctx* ctx, double* poses, double* inv_depth, double* residual_norms, int* n_norms) {
    return guarded([&] {
        bind(ctx);
        Batch& B = ctx->bat;
        if (!B.loaded) fail(PVO_INVALID_ARGUMENT, "batch: nothing loaded");
        const int corr_status = read_status(ctx);
        if (corr_status & (1 << pvo_dev::kDevBadCoords)) fail(PVO_INVALID_ARGUMENT, "correlate: non-finite reprojection");
        std::vector<int> st(B.n_windows);
        download(ctx, st.data(), static_cast<const int*>(B.status.p), st.size());
        sync(ctx);
        for (int w = 0; w < B.n_windows; ++w)
            if (st[w]) {
                try {
                    raise_ba_status(st[w]);
                } catch (const Error& e) {
                    fail(e.status, "window " + std::to_string(w) + ": " + e.what());
                }
            }
        if (poses) download(ctx, poses, static_cast<const double*>(B.poses.p), (size_t)B.n_poses * 7);
        if (inv_depth) download(ctx, inv_depth, static_cast<const double*>(B.depth.p), B.n_patches);
        if (residual_norms)
            download(ctx, residual_norms, static_cast<const double*>(B.norms.p), (size_t)B.n_windows * Batch::kNormStride);
        if (n_norms) download(ctx, n_norms, static_cast<const int*>(B.n_norms.p), B.n_windows);
        sync(ctx);
    });
}

int pvo_batch_norm_stride(void) { return Batch::kNormStride; }

// ---- device-resident patch graph (dgraph.cu) -------------
}  // extern "C"

struct pvo_dgraph {
    pvo_ctx* ctx = nullptr;
    double K[4];
    int w = 0, h = 0, p = 3, C = 0;
    int next_id = 0;
    // host mirrors of the small, host-validated state
    std::vector<int> f_index, f_slot;
    std::vector<double> f_ts;
    std::vector<LogEntryHost> log;
    int P = 0, E = 0;
    // device state (double-buffered where a pass rewrites it)
    DevBuf f_idx_d, f_pose_d, f_slot_d;
    DevBuf p_id[2], p_src[2], p_x[2], p_y[2], p_d[2], p_feat[2];
    DevBuf ebeg[2], e_frame[2], e_has[2], e_rev[2];
    int cur = 0;  // which buffer set is live
    // scratch
    DevBuf t0, t1, t2, t3, t4, missing;
    // the last flattened window's extras (pose frames, fixed mask, patch ids, edge -> graph edge)
    DevBuf w_pose_frames, w_fixed, w_patch_ids, w_e_graph, w_nfixed;
    int wn_poses = 0, wn_patches = 0, wn_edges = 0;
    bool window_from_graph = false;

    pvo_dev::DGraphView view(int b) {
        pvo_dev::DGraphView v;
        v.F = static_cast<int>(f_index.size());
        v.P = P;
        v.f_index = static_cast<int*>(f_idx_d.p);
        v.f_pose = static_cast<double*>(f_pose_d.p);
        v.f_slot = static_cast<int*>(f_slot_d.p);
        v.p_id = static_cast<int*>(p_id[b].p);
        v.p_src = static_cast<int*>(p_src[b].p);
        v.p_x = static_cast<double*>(p_x[b].p);
        v.p_y = static_cast<double*>(p_y[b].p);
        v.p_d = static_cast<double*>(p_d[b].p);
        v.p_feat = static_cast<float*>(p_feat[b].p);
        v.feat_stride = (size_t)2 * 9 * C;
        v.ebeg = static_cast<int*>(ebeg[b].p);
        v.e_frame = static_cast<int*>(e_frame[b].p);
        v.e_has = static_cast<uint8_t*>(e_has[b].p);
        v.e_rev = static_cast<double*>(e_rev[b].p);
        return v;
    }
    // grow buffer set b to hold np patches / ne edges, preserving contents
    void reserve(int b, int np, int ne) {
        auto grow = [&](DevBuf& d, size_t bytes) {
            if (bytes <= d.cap) return;
            DevBuf n;
            n.get(std::max(bytes, 2 * d.cap));
            if (d.p) cuda_check(cudaMemcpyAsync(n.p, d.p, d.cap, cudaMemcpyDeviceToDevice, ctx->stream), "grow");
            cuda_check(cudaStreamSynchronize(ctx->stream), "grow");
            d.release();
            d = n;
            n.p = nullptr;
        };
        grow(p_id[b], 4 * (size_t)std::max(np, 1));
        grow(p_src[b], 4 * (size_t)std::max(np, 1));
        grow(p_x[b], 8 * 9 * (size_t)std::max(np, 1));
        grow(p_y[b], 8 * 9 * (size_t)std::max(np, 1));
        grow(p_d[b], 8 * (size_t)std::max(np, 1));
        grow(p_feat[b], 4 * (size_t)2 * 9 * C * std::max(np, 1));
        grow(ebeg[b], 4 * (size_t)(np + 1));
        grow(e_frame[b], 4 * (size_t)std::max(ne, 1));
        grow(e_has[b], (size_t)std::max(ne, 1));
        grow(e_rev[b], 32 * (size_t)std::max(ne, 1));
    }
    int position(int frame) const {
        auto it = std::lower_bound(f_index.begin(), f_index.end(), frame);
        if (it == f_index.end() || *it != frame) fail(PVO_INVALID_ARGUMENT, "patch graph: no frame " + std::to_string(frame));
        return static_cast<int>(it - f_index.begin());
    }
    void release() {
        DevBuf* all[] = {&f_idx_d, &f_pose_d, &f_slot_d, &t0, &t1, &t2, &t3, &t4, &missing, &w_pose_frames,
                         &w_fixed, &w_patch_ids, &w_e_graph, &w_nfixed};
        for (DevBuf* b : all) b->release();
        for (int b = 0; b < 2; ++b) {
            DevBuf* bs[] = {&p_id[b], &p_src[b], &p_x[b], &p_y[b], &p_d[b], &p_feat[b], &ebeg[b], &e_frame[b],
                            &e_has[b], &e_rev[b]};
            for (DevBuf* x : bs) x->release();
        }
    }
};

extern "C" {

int pvo_dgraph_create(pvo_ctx* ctx, const double* K, int w, int h, int p, int channels, pvo_dgraph** out) {
    return guarded([&] {
        bind(ctx);
        if (!out) fail(PVO_INVALID_ARGUMENT, "null output");
        ensure_p3(p);
        if (K[0] <= 0 || K[1] <= 0) fail(PVO_INVALID_ARGUMENT, "intrinsics: focal lengths must be positive");
        if (channels < 0) fail(PVO_INVALID_ARGUMENT, "dgraph: negative channel count");
        auto* g = new pvo_dgraph();
        g->ctx = ctx;
        std::memcpy(g->K, K, sizeof(g->K));
        g->w = w;
        g->h = h;
        g->C = channels;
        g->reserve(0, 64, 64);
        cuda_check(cudaMemsetAsync(g->ebeg[0].p, 0, sizeof(int), ctx->stream), "memset");
        *out = g;
    });
}

int pvo_dgraph_destroy(pvo_dgraph* g) {
    if (!g) return PVO_OK;
    cudaSetDevice(g->ctx->device);
    cudaStreamSynchronize(g->ctx->stream);
    g->release();
    delete g;
    return PVO_OK;
}

namespace {
void dg_upload_frames(pvo_dgraph* g, const std::vector<double>* poses_host) {
    pvo_ctx* ctx = g->ctx;
    const size_t F = g->f_index.size();
    upload(ctx, g->f_idx_d, g->f_index.data(), std::max<size_t>(F, 1));
    upload(ctx, g->f_slot_d, g->f_slot.data(), std::max<size_t>(F, 1));
    if (poses_host) upload(ctx, g->f_pose_d, poses_host->data(), poses_host->size());
}
}  // namespace

// patch_graph.cpp:27-34 (+ the frame-store slot holding the frame's pyramid)
int pvo_dgraph_add_frame(pvo_dgraph* g, double ts, const double* pose, int frame_slot, int* out_index) {
    return guarded([&] {
        pvo_ctx* ctx = g->ctx;
        bind(ctx);
        if (!g->f_ts.empty() && ts <= g->f_ts.back()) {
            fail(PVO_INVALID_ARGUMENT, "patch graph: timestamp must exceed the last frame's");
        }
        const int idx = g->f_index.empty() ? 0 : g->f_index.back() + 1;
        const size_t F = g->f_index.size();
        // poses live on the device (BA writes them back): append in place
        DevBuf grown;
        double* dp = static_cast<double*>(g->f_pose_d.p);
        if (g->f_pose_d.cap < 8 * 7 * (F + 1)) {
            grown.get(std::max<size_t>(8 * 7 * 2 * (F + 1), 8 * 7 * 64));
            if (F) cuda_check(cudaMemcpyAsync(grown.p, dp, 8 * 7 * F, cudaMemcpyDeviceToDevice, ctx->stream), "grow");
            sync(ctx);
            g->f_pose_d.release();
            g->f_pose_d = grown;
            grown.p = nullptr;
            dp = static_cast<double*>(g->f_pose_d.p);
        }
        cuda_check(cudaMemcpyAsync(dp + 7 * F, pose, 8 * 7, cudaMemcpyHostToDevice, ctx->stream), "H2D");
        g->f_index.push_back(idx);
        g->f_slot.push_back(frame_slot);
        g->f_ts.push_back(ts);
        dg_upload_frames(g, nullptr);  // stream-ordered; pageable sources are staged before return
        if (host_pinned(pose)) sync(ctx);
        if (out_index) *out_index = idx;
    });
}

// patch_graph.cpp:36-60 + Patch::make (camera.cpp:15-32); feats [n][2][9][C] or NULL
int pvo_dgraph_add_patches(pvo_dgraph* g, int frame, int n, const double* centroids, const double* depths,
                           const float* feats, int* out_ids) {
    return guarded([&] {
        pvo_ctx* ctx = g->ctx;
        bind(ctx);
        g->position(frame);
        for (int k = 0; k < n; ++k) {
            const double cx = centroids[2 * k], cy = centroids[2 * k + 1];
            if (cx - 1 < 0 || cy - 1 < 0 || cx + 1 > g->w - 1 || cy + 1 > g->h - 1) {
                fail(PVO_INVALID_ARGUMENT, "patch graph: centroid (" + std::to_string(cx) + ", " + std::to_string(cy) +
                                               ") leaves the image bounds");
            }
            if (depths[k] < 0) fail(PVO_INVALID_ARGUMENT, "patch: inverse depth must be >= 0");
        }
        if (n <= 0) return;
        const int b = g->cur, P0 = g->P;
        g->reserve(b, P0 + n, g->E);
        std::vector<int> ids(n), src(n, frame);
        std::vector<double> x(9 * (size_t)n), y(9 * (size_t)n);
        for (int k = 0; k < n; ++k) {
            ids[k] = g->next_id++;
            for (int row = 0; row < 3; ++row)
                for (int col = 0; col < 3; ++col) {
                    x[9 * (size_t)k + 3 * row + col] = centroids[2 * k] + col - 1.0;
                    y[9 * (size_t)k + 3 * row + col] = centroids[2 * k + 1] + row - 1.0;
                }
            if (out_ids) out_ids[k] = ids[k];
        }
        auto h2d = [&](DevBuf& d, const void* src_, size_t off, size_t bytes) {
            cuda_check(cudaMemcpyAsync(static_cast<char*>(d.p) + off, src_, bytes, cudaMemcpyHostToDevice, ctx->stream), "H2D");
        };
        h2d(g->p_id[b], ids.data(), 4 * (size_t)P0, 4 * (size_t)n);
        h2d(g->p_src[b], src.data(), 4 * (size_t)P0, 4 * (size_t)n);
        h2d(g->p_x[b], x.data(), 72 * (size_t)P0, 72 * (size_t)n);
        h2d(g->p_y[b], y.data(), 72 * (size_t)P0, 72 * (size_t)n);
        h2d(g->p_d[b], depths, 8 * (size_t)P0, 8 * (size_t)n);
        const size_t fs = 4 * (size_t)2 * 9 * g->C;
        if (fs) {
            if (feats)
                h2d(g->p_feat[b], feats, fs * P0, fs * n);
            else
                cuda_check(cudaMemsetAsync(static_cast<char*>(g->p_feat[b].p) + fs * P0, 0, fs * n, ctx->stream), "memset");
        }
        // the new patches have no edges yet: ebeg[P0+1 .. P0+n] = E
        std::vector<int> eb(n, g->E);
        h2d(g->ebeg[b], eb.data(), 4 * (size_t)(P0 + 1), 4 * (size_t)n);
        g->P = P0 + n;  // stream-ordered; the pageable temporaries were staged by the copies
        if (host_pinned(depths) || host_pinned(feats)) sync(ctx);
    });
}

// patch_graph.cpp:62-85
int pvo_dgraph_connect(pvo_dgraph* g, int radius, int* n_added) {
    return guarded([&] {
        pvo_ctx* ctx = g->ctx;
        bind(ctx);
        if (radius < 1) fail(PVO_INVALID_ARGUMENT, "patch graph: radius must be >= 1");
        const int b = g->cur, nb = 1 - b, P = g->P;
        if (P == 0) {
            if (n_added) *n_added = 0;
            return;
        }
        int* newlen = g->t0.as<int>(P);
        int* neb = g->ebeg[nb].as<int>(P + 1);
        cuda_check(pvo_dev::dg_connect(g->view(b), radius, 0, newlen, nullptr, nullptr, nullptr, nullptr, ctx->stream), "connect");
        cuda_check(pvo_dev::dg_scan(P, newlen, neb, ctx->stream), "scan");
        int E2 = 0;
        download(ctx, &E2, neb + P, 1);
        sync(ctx);
        g->reserve(nb, P, E2);
        neb = static_cast<int*>(g->ebeg[nb].p);
        // patch arrays are unchanged by connect: share them (copy into the other set)
        const size_t fs = 4 * (size_t)2 * 9 * g->C;
        auto d2d = [&](DevBuf& dst, DevBuf& srcb, size_t bytes) {
            if (bytes) cuda_check(cudaMemcpyAsync(dst.p, srcb.p, bytes, cudaMemcpyDeviceToDevice, ctx->stream), "D2D");
        };
        d2d(g->p_id[nb], g->p_id[b], 4 * (size_t)P);
        d2d(g->p_src[nb], g->p_src[b], 4 * (size_t)P);
        d2d(g->p_x[nb], g->p_x[b], 72 * (size_t)P);
        d2d(g->p_y[nb], g->p_y[b], 72 * (size_t)P);
        d2d(g->p_d[nb], g->p_d[b], 8 * (size_t)P);
        d2d(g->p_feat[nb], g->p_feat[b], fs * P);
        cuda_check(pvo_dev::dg_connect(g->view(b), radius, 1, nullptr, neb, static_cast<int*>(g->e_frame[nb].p),
                                       static_cast<uint8_t*>(g->e_has[nb].p), static_cast<double*>(g->e_rev[nb].p),
                                       ctx->stream),
                   "connect");
        if (n_added) *n_added = E2 - g->E;
        g->E = E2;
        g->cur = nb;
    });
}

// patch_graph.cpp:87-128
int pvo_dgraph_remove_frame(pvo_dgraph* g, int frame) {
    return guarded([&] {
        pvo_ctx* ctx = g->ctx;
        bind(ctx);
        const int pos = g->position(frame);
        const int F = static_cast<int>(g->f_index.size());
        if (pos >= F - 3) {
            fail(PVO_INVALID_ARGUMENT, "patch graph: frame " + std::to_string(frame) + " is among the most recent 3 keyframes");
        }
        if (pos == 0) fail(PVO_INVALID_ARGUMENT, "patch graph: the oldest frame has no predecessor to anchor");
        // relative-pose log entry (host; poses read back)
        std::vector<double> two(14);
        download(ctx, two.data(), static_cast<const double*>(g->f_pose_d.p) + 7 * (pos - 1), 14);
        sync(ctx);
        LogEntryHost le;
        le.removed = frame;
        le.anchor = g->f_index[pos - 1];
        le.ts = g->f_ts[pos];
        pvo_dev::se3_store(pvo_dev::se3_compose(pvo_dev::se3_load(two.data() + 7), pvo_dev::se3_inverse(pvo_dev::se3_load(two.data()))),
                           le.relative);
        g->log.push_back(le);
        const int b = g->cur, nb = 1 - b, P = g->P;
        if (P > 0) {
            int* keep = g->t0.as<int>(P);
            int* newlen = g->t1.as<int>(P);
            int* pidx = g->t2.as<int>(P + 1);
            int* neb = g->t3.as<int>(P + 1);
            pvo_dev::DGraphView v = g->view(b);
            cuda_check(pvo_dev::dg_remove(v, frame, 0, keep, newlen, nullptr, nullptr, v, ctx->stream), "remove");
            cuda_check(pvo_dev::dg_scan(P, keep, pidx, ctx->stream), "scan");
            cuda_check(pvo_dev::dg_scan(P, newlen, neb, ctx->stream), "scan");
            int cnt[2];
            download(ctx, &cnt[0], pidx + P, 1);
            download(ctx, &cnt[1], neb + P, 1);
            sync(ctx);
            g->reserve(nb, cnt[0], cnt[1]);
            pvo_dev::DGraphView out = g->view(nb);
            cuda_check(pvo_dev::dg_remove(g->view(b), frame, 1, nullptr, nullptr, pidx, neb, out, ctx->stream), "remove");
            // new CSR: ebeg_new[q] = neb[k] for kept k (neb is indexed by old patch): compact it
            std::vector<int> hk(P), hneb(P + 1);
            download(ctx, hk.data(), keep, P);
            download(ctx, hneb.data(), neb, P + 1);
            sync(ctx);
            std::vector<int> eb;
            eb.reserve(cnt[0] + 1);
            for (int k = 0; k < P; ++k)
                if (hk[k]) eb.push_back(hneb[k]);
            eb.push_back(cnt[1]);
            upload(g->ctx, g->ebeg[nb], eb.data(), eb.size());
            g->P = cnt[0];
            g->E = cnt[1];
            g->cur = nb;
        }
        // frames: drop position pos (poses shift down on the device)
        double* dp = static_cast<double*>(g->f_pose_d.p);
        if (pos + 1 < F)
            cuda_check(cudaMemcpyAsync(g->t4.as<double>(7 * (size_t)(F - pos - 1)), dp + 7 * (pos + 1),
                                       8 * 7 * (size_t)(F - pos - 1), cudaMemcpyDeviceToDevice, ctx->stream), "D2D");
        if (pos + 1 < F)
            cuda_check(cudaMemcpyAsync(dp + 7 * pos, g->t4.p, 8 * 7 * (size_t)(F - pos - 1), cudaMemcpyDeviceToDevice,
                                       ctx->stream), "D2D");
        g->f_index.erase(g->f_index.begin() + pos);
        g->f_slot.erase(g->f_slot.begin() + pos);
        g->f_ts.erase(g->f_ts.begin() + pos);
        dg_upload_frames(g, nullptr);
        sync(ctx);
    });
}

// patch_graph.cpp:153-164 for n keys (host arrays)
int pvo_dgraph_set_revisions(pvo_dgraph* g, int n, const int* patch_ids, const int* frames, const double* deltas,
                             const double* weights) {
    return guarded([&] {
        pvo_ctx* ctx = g->ctx;
        bind(ctx);
        if (n <= 0) return;
        std::vector<double> rev(4 * (size_t)n);
        for (int i = 0; i < n; ++i) {
            if (weights[2 * i] <= 0 || weights[2 * i] >= 1 || weights[2 * i + 1] <= 0 || weights[2 * i + 1] >= 1) {
                fail(PVO_INVALID_ARGUMENT, "patch graph: revision weights must lie in (0, 1)");
            }
            rev[4 * (size_t)i] = deltas[2 * i];
            rev[4 * (size_t)i + 1] = deltas[2 * i + 1];
            rev[4 * (size_t)i + 2] = weights[2 * i];
            rev[4 * (size_t)i + 3] = weights[2 * i + 1];
        }
        const int* di = upload(ctx, g->t0, patch_ids, n);
        const int* df = upload(ctx, g->t1, frames, n);
        const double* dr = upload(ctx, g->t4, rev.data(), rev.size());
        int* miss = g->missing.as<int>(1);
        const int big = 1 << 30;
        cuda_check(cudaMemcpyAsync(miss, &big, sizeof(int), cudaMemcpyHostToDevice, ctx->stream), "H2D");
        cuda_check(pvo_dev::dg_set_revisions(g->view(g->cur), n, di, df, dr, miss, ctx->stream), "set revisions");
        int m = 0;
        download(ctx, &m, miss, 1);
        sync(ctx);
        if (m != big) {
            fail(PVO_INVALID_ARGUMENT, "patch graph: no edge (" + std::to_string(patch_ids[m]) + ", " +
                                           std::to_string(frames[m]) + ")");
        }
    });
}

int pvo_dgraph_counts(pvo_dgraph* g, int* n_frames, int* n_patches, int* n_edges) {
    return guarded([&] {
        if (n_frames) *n_frames = static_cast<int>(g->f_index.size());
        if (n_patches) *n_patches = g->P;
        if (n_edges) *n_edges = g->E;
    });
}

// edges in key order (kk = patch id, jj = frame), rev [E][4], has_rev [E] (host copies)
int pvo_dgraph_edges(pvo_dgraph* g, int* kk, int* jj, double* rev, uint8_t* has_rev) {
    return guarded([&] {
        pvo_ctx* ctx = g->ctx;
        bind(ctx);
        const int b = g->cur, P = g->P, E = g->E;
        std::vector<int> ids(P), eb(P + 1);
        download(ctx, ids.data(), static_cast<const int*>(g->p_id[b].p), P);
        download(ctx, eb.data(), static_cast<const int*>(g->ebeg[b].p), P + 1);
        if (jj) download(ctx, jj, static_cast<const int*>(g->e_frame[b].p), E);
        if (rev) download(ctx, rev, static_cast<const double*>(g->e_rev[b].p), 4 * (size_t)E);
        if (has_rev) download(ctx, has_rev, static_cast<const uint8_t*>(g->e_has[b].p), E);
        sync(ctx);
        if (kk)
            for (int k = 0; k < P; ++k)
                for (int i = eb[k]; i < eb[k + 1]; ++i) kk[i] = ids[k];
    });
}

int pvo_dgraph_frames(pvo_dgraph* g, int* indices, double* poses) {
    return guarded([&] {
        bind(g->ctx);
        const size_t F = g->f_index.size();
        if (indices) std::copy(g->f_index.begin(), g->f_index.end(), indices);
        if (poses) {
            download(g->ctx, poses, static_cast<const double*>(g->f_pose_d.p), 7 * F);
            sync(g->ctx);
        }
    });
}

int pvo_dgraph_patches(pvo_dgraph* g, int* ids, int* src, double* inv_depth) {
    return guarded([&] {
        pvo_ctx* ctx = g->ctx;
        bind(ctx);
        const int b = g->cur;
        if (ids) download(ctx, ids, static_cast<const int*>(g->p_id[b].p), g->P);
        if (src) download(ctx, src, static_cast<const int*>(g->p_src[b].p), g->P);
        if (inv_depth) download(ctx, inv_depth, static_cast<const double*>(g->p_d[b].p), g->P);
        sync(ctx);
    });
}

// Pipeline::keyframe (pipeline.cpp:208-245): with >= 6 frames, the mean
// reprojected displacement between keyframes t-5 and t-3 over the patches
// seen in both; below threshold_px the candidate t-4 is removed.  removed =
// the removed frame index or -1; mean_flow / n_used report the statistic.
int pvo_dgraph_keyframe(pvo_dgraph* g, double threshold_px, int* removed, double* mean_flow, int* n_used) {
    return guarded([&] {
        pvo_ctx* ctx = g->ctx;
        bind(ctx);
        if (removed) *removed = -1;
        if (mean_flow) *mean_flow = 0.0;
        if (n_used) *n_used = 0;
        const int F = static_cast<int>(g->f_index.size());
        if (F < 6) return;  // need keyframes t-5 .. t
        const int frame_a = g->f_index[F - 6], frame_b = g->f_index[F - 4], candidate = g->f_index[F - 5];
        double* flow = g->t4.as<double>(std::max(g->P, 1));
        int* ok = g->t0.as<int>(std::max(g->P, 1));
        double* out = ctx->s6.as<double>(2);
        cuda_check(pvo_dev::dg_keyframe_flow(g->view(g->cur), frame_a, frame_b, g->K, flow, ok, out, ctx->stream),
                   "keyframe");
        double h[2];
        download(ctx, h, out, 2);
        sync(ctx);
        if (mean_flow) *mean_flow = h[0];
        if (n_used) *n_used = static_cast<int>(h[1]);
        if (h[1] == 0) return;
        if (h[0] < threshold_px) {
            const int st = pvo_dgraph_remove_frame(g, candidate);
            if (st != PVO_OK) fail(st, std::string("keyframe: ") + pvo_last_error());
            if (removed) *removed = candidate;
        }
    });
}

// The optimize_window problem build (bundle_adjust.cpp:231-307) on the device,
// loaded as the context's resident window (pvo_window_iteration / propose run
// on it next).  Revision deltas + raw weights: targets are frozen on the
// device by the BA (freeze_targets semantics).  all_active != 0 flattens every
// active edge (Pipeline::active_edges, pipeline.cpp:164-181: revised or not) —
// the set propose() measures; 0 keeps the revised ones (bundle_adjust.cpp:245).
// Windows beyond 16 free poses are not supported on this path yet.
int pvo_window_load_dgraph(pvo_ctx* ctx, pvo_dgraph* g, int window, int all_active, int* n_poses, int* n_patches,
                           int* n_edges) {
    return guarded([&] {
        bind(ctx);
        if (g->ctx != ctx) fail(PVO_INVALID_ARGUMENT, "window_load_dgraph: the graph belongs to another context");
        if (window < 1) fail(PVO_INVALID_ARGUMENT, "ba: window must be >= 1");
        if (ctx->nf == 0) fail(PVO_INVALID_ARGUMENT, "window_load: frame store is empty (pvo_frames_reserve)");
        if (g->C != 0 && g->C != ctx->C)
            fail(PVO_INVALID_ARGUMENT, "window_load_dgraph: descriptor channels differ from the frame store");
        Window& w = ctx->win;
        w.loaded = false;
        w.half = 0;  // the processing order is built on the device: no split read-back
        const int F = static_cast<int>(g->f_index.size()), P = g->P;
        const int window_start = std::max(F - window, 0), first_free = std::max(F - window, 1);
        pvo_dev::DGraphView v = g->view(g->cur);
        int* inc = g->t0.as<int>(std::max(P, 1));
        int* nrev = g->t1.as<int>(std::max(P, 1));
        int* pslot = g->t2.as<int>(P + 1);
        int* eoff = g->t3.as<int>(P + 1);
        int* used = ctx->s7.as<int>(std::max(F, 1));
        int* slot_of_pos = ctx->s8.as<int>(F + 1);
        int* nfix = g->w_nfixed.as<int>(1);
        cuda_check(cudaMemsetAsync(used, 0, sizeof(int) * std::max(F, 1), ctx->stream), "memset");
        cuda_check(pvo_dev::dg_window_pass0(v, window_start, all_active, inc, nrev, ctx->stream), "window");
        cuda_check(pvo_dev::dg_scan(P, inc, pslot, ctx->stream), "scan");
        cuda_check(pvo_dev::dg_scan(P, nrev, eoff, ctx->stream), "scan");
        cuda_check(pvo_dev::dg_window_used(v, inc, all_active, used, ctx->stream), "window");
        cuda_check(pvo_dev::dg_scan(F, used, slot_of_pos, ctx->stream), "scan");
        cuda_check(pvo_dev::dg_window_nfixed(v, first_free, used, nfix, ctx->stream), "window");
        int cnt[4];
        download(ctx, &cnt[0], slot_of_pos + F, 1);
        download(ctx, &cnt[1], pslot + P, 1);
        download(ctx, &cnt[2], eoff + P, 1);
        download(ctx, &cnt[3], nfix, 1);
        sync(ctx);
        const int N = cnt[0], Pw = cnt[1], Ew = cnt[2], nfixed = cnt[3];
        if (n_poses) *n_poses = N;
        if (n_patches) *n_patches = Pw;
        if (n_edges) *n_edges = Ew;
        g->window_from_graph = false;
        if (Pw == 0) return;  // nothing to optimise
        if (N - nfixed > pvo_dev::ba_max_free_poses() || N > pvo_dev::ba_max_poses())
            fail(PVO_UNSUPPORTED, "window_load_dgraph: windows beyond 16 free poses / 128 poses");
        BABuffers& B = ctx->ba;
        pvo_dev::WindowOut o;
        o.n_poses = N;
        o.n_patches = Pw;
        o.n_edges = Ew;
        o.pose_frames = g->w_pose_frames.as<int>(N);
        o.poses = B.poses.as<double>(7 * (size_t)N);
        o.fixed = g->w_fixed.as<uint8_t>(N);
        o.pose_slot = w.pose_slot.as<int>(N);
        o.free_slot = B.free_slot.as<int>(N);
        o.n_fixed_dev = nfix;
        o.patch_ids = g->w_patch_ids.as<int>(Pw);
        o.patch_src = B.patch_src.as<int>(Pw);
        o.px = B.px.as<double>(9 * (size_t)Pw);
        o.py = B.py.as<double>(9 * (size_t)Pw);
        o.depth = B.depth.as<double>(Pw);
        o.depth_slot = B.depth_slot.as<int>(Pw);
        o.edge_begin = B.edge_begin.as<int>(Pw + 1);
        o.patch_feats = w.patch_feats.as<float>((size_t)Pw * 2 * 9 * ctx->C);
        if (g->C == 0)  // a graph without descriptors: the window's are zero
            cuda_check(cudaMemsetAsync(o.patch_feats, 0, sizeof(float) * (size_t)Pw * 2 * 9 * ctx->C, ctx->stream), "memset");
        o.e_patch = B.e_patch.as<int>(Ew);
        o.e_pose = B.e_pose.as<int>(Ew);
        o.e_delta = B.e_in.as<double>(2 * (size_t)Ew);
        o.e_weight = B.e_w.as<double>(2 * (size_t)Ew);
        o.e_graph = g->w_e_graph.as<int>(Ew);
        o.order = w.order.as<int>(Ew);
        o.graph_patch = g->t4.as<int>(Pw);
        cuda_check(pvo_dev::dg_window_write(v, first_free, inc, all_active, pslot, eoff, used, slot_of_pos, o, ctx->nf,
                                            ctx->stream),
                   "window");
        ctx->launches += 8;
        // window bookkeeping as pvo_window_load (plan fields used by the kernels)
        w.n_poses = N;
        w.n_patches = Pw;
        w.n_edges = Ew;
        w.plan = Plan{};
        w.plan.n_free_poses = N - nfixed;
        w.plan.n_free_depths = Pw;
        w.shape = HostProblem{};
        std::memcpy(w.shape.K, g->K, sizeof(g->K));
        w.shape.image_w = g->w;
        w.shape.image_h = g->h;
        w.shape.n_poses = N;
        w.shape.n_patches = Pw;
        w.shape.n_edges = Ew;
        upload(ctx, B.K, g->K, 4);
        B.e_target.as<double>(2 * (size_t)Ew);
        B.e_weight.as<double>(2 * (size_t)Ew);
        B.cand_poses.as<double>(7 * (size_t)N);
        B.cand_depth.as<double>(Pw);
        B.patch_v.as<double>((size_t)Pw * std::max(6 * (N - nfixed), 1));
        B.patch_h.as<double>(Pw);
        B.patch_bd.as<double>(Pw);
        cuda_check(cudaMemcpyAsync(w.init_poses.as<double>(7 * (size_t)N), B.poses.p, 8 * 7 * (size_t)N,
                                   cudaMemcpyDeviceToDevice, ctx->stream), "D2D");
        cuda_check(cudaMemcpyAsync(w.init_depth.as<double>(Pw), B.depth.p, 8 * (size_t)Pw, cudaMemcpyDeviceToDevice,
                                   ctx->stream), "D2D");
        w.corr.get(sizeof(float) * (size_t)Ew * 2 * 9 * 49);
        g->wn_poses = N;
        g->wn_patches = Pw;
        g->wn_edges = Ew;
        g->window_from_graph = true;
        sync(ctx);
        w.loaded = true;
    });
}

// The window's current revisions (e.g. from pvo_window_propose) back into the
// graph's edges (has_rev set), and its BA state (free poses, every included
// depth) back into the graph (bundle_adjust.cpp:368-373).
int pvo_dgraph_store_window(pvo_ctx* ctx, pvo_dgraph* g, int revisions, int state) {
    return guarded([&] {
        bind(ctx);
        if (!g->window_from_graph || !ctx->win.loaded) fail(PVO_INVALID_ARGUMENT, "dgraph: no window loaded from this graph");
        pvo_dev::DGraphView v = g->view(g->cur);
        BABuffers& B = ctx->ba;
        if (revisions)
            cuda_check(pvo_dev::dg_store_revisions(v, g->wn_edges, static_cast<const int*>(g->w_e_graph.p),
                                                   static_cast<const double*>(B.e_in.p),
                                                   static_cast<const double*>(B.e_w.p), ctx->stream),
                       "store revisions");
        if (state)
            cuda_check(pvo_dev::dg_writeback(v, g->wn_poses, static_cast<const int*>(g->w_pose_frames.p),
                                             static_cast<const uint8_t*>(g->w_fixed.p),
                                             static_cast<const double*>(B.poses.p), g->wn_patches,
                                             static_cast<const int*>(g->w_patch_ids.p),
                                             static_cast<const double*>(B.depth.p), ctx->stream),
                       "writeback");
        sync(ctx);
    });
}

// Download the resident window's flattened problem (tests: compare with the host graph).
int pvo_window_problem_read(pvo_ctx* ctx, double* poses, uint8_t* fixed, int* pose_slot, int* patch_src, double* px,
                            double* py, double* depth, int* e_patch, int* e_pose, double* e_delta, double* e_weight) {
    return guarded([&] {
        bind(ctx);
        Window& w = ctx->win;
        if (!w.loaded) fail(PVO_INVALID_ARGUMENT, "window: nothing loaded");
        BABuffers& B = ctx->ba;
        const size_t N = w.n_poses, P = w.n_patches, E = w.n_edges;
        if (poses) download(ctx, poses, static_cast<const double*>(B.poses.p), 7 * N);
        if (fixed) {
            std::vector<int> fs(N);
            download(ctx, fs.data(), static_cast<const int*>(B.free_slot.p), N);
            sync(ctx);
            for (size_t i = 0; i < N; ++i) fixed[i] = fs[i] < 0;
        }
        if (pose_slot) download(ctx, pose_slot, static_cast<const int*>(w.pose_slot.p), N);
        if (patch_src) download(ctx, patch_src, static_cast<const int*>(B.patch_src.p), P);
        if (px) download(ctx, px, static_cast<const double*>(B.px.p), 9 * P);
        if (py) download(ctx, py, static_cast<const double*>(B.py.p), 9 * P);
        if (depth) download(ctx, depth, static_cast<const double*>(B.depth.p), P);
        if (e_patch) download(ctx, e_patch, static_cast<const int*>(B.e_patch.p), E);
        if (e_pose) download(ctx, e_pose, static_cast<const int*>(B.e_pose.p), E);
        if (e_delta) download(ctx, e_delta, static_cast<const double*>(B.e_in.p), 2 * E);
        if (e_weight) download(ctx, e_weight, static_cast<const double*>(B.e_w.p), 2 * E);
        sync(ctx);
    });
}

int pvo_window_corr_ptr(pvo_ctx* ctx, float** corr) {
    return guarded([&] {
        bind(ctx);
        if (!ctx->win.loaded) fail(PVO_INVALID_ARGUMENT, "window: nothing loaded");
        *corr = static_cast<float*>(ctx->win.corr.p);
    });
}

}  // extern "C"
