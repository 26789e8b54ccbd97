// capi_batch.cu — extern "C" boundary: batches of independent windows (config 5).
#include "capi_common.hpp"

extern "C" {

// ---- batch of independent windows -------------------------------------------
int pvo_batch_load(pvo_ctx* ctx, int n_windows, const int* pose_off, const int* patch_off, const int* edge_off,
                   const double* poses, const uint8_t* fixed, const int* pose_slot, int p, const int* src,
                   const double* px, const double* py, const double* depth, const float* patch_feats,
                   const int* e_patch, const int* e_pose, const double* e_delta, const double* e_weight,
                   const double* K, int image_w, int image_h) {
    return guarded(__func__, [&] {
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
        B.large_idx.clear();
        B.large_plans.clear();
        int max_free_large = 0;
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
            Plan pl = make_plan(pr, false);
            if (!pl.sorted) fail(PVO_INVALID_ARGUMENT, "batch_load: edges must be grouped by patch (reference order)");
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
            if (pl.large) {  // its own plan and scratch (Batch::lb); no batched-kernel buffers
                v_off[w + 1] = v_off[w];
                part_off[w + 1] = part_off[w];
                sys_off[w + 1] = sys_off[w];
                max_free_large = std::max(max_free_large, pl.n_free_poses);
                B.large_idx.push_back(w);
                B.large_plans.push_back(std::move(pl));
                continue;
            }
            v_off[w + 1] = v_off[w] + (size_t)pr.n_patches * std::max(np, 1);
            part_off[w + 1] = part_off[w] + pvo_dev::ba_partials_doubles(pl.n_free_poses, 1);
            sys_off[w + 1] = sys_off[w] + (size_t)np * (np + 1) / 2 + np + 1;
            B.max_free = std::max(B.max_free, pl.n_free_poses);
            B.max_poses = std::max(B.max_poses, pr.n_poses);
        }
        B.n_small = n_windows - (int)B.large_idx.size();
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
            a.delta = delta + (size_t)w * std::max(6 * B.max_free, 1);  // (large windows: Batch::lb.delta)
            a.residual_norms = norms + (size_t)w * Batch::kNormStride;
            a.n_norms = n_norms + w;
            a.status = status + w;
            a.status2 = status2 + 2 * w;
            a.attempts = attempts + w;
        }
        if (!B.large_idx.empty()) B.lb.delta.as<double>((size_t)6 * max_free_large);
        for (size_t i = 0; i < B.large_idx.size(); ++i) {  // the large path's per-window buffers
            pvo_dev::BAParams& a = B.hparams[B.large_idx[i]];
            a.partials = nullptr;
            a.system = nullptr;
            a.patch_v = nullptr;
            a.delta = static_cast<double*>(B.lb.delta.p);
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
    // the batched kernel's windows: every window that is not on the large path
    std::vector<pvo_dev::BAParams>& small = B.small_params;  // kept: the H2D copy reads it
    small.clear();
    size_t li = 0;
    for (int w = 0; w < B.n_windows; ++w) {
        if (li < B.large_idx.size() && B.large_idx[li] == w) {
            ++li;
            continue;
        }
        small.push_back(B.hparams[w]);
    }
    if (!small.empty()) upload(ctx, B.params, small.data(), small.size());
    B.iterations = iterations;
    B.damping = damping;
}
}  // namespace

int pvo_batch_reset(pvo_ctx* ctx) {
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
        bind(ctx);
        Batch& B = ctx->bat;
        if (!B.loaded) fail(PVO_INVALID_ARGUMENT, "batch: nothing loaded");
        if (iterations < 0) fail(PVO_INVALID_ARGUMENT, "ba: negative iteration count");
        batch_params(ctx, iterations, damping);
        reset_status(ctx);
        cuda_check(cudaMemsetAsync(B.status.p, 0, sizeof(int) * B.n_windows, ctx->stream), "memset");
        cuda_check(cudaMemsetAsync(B.status2.p, 0, sizeof(int) * 2 * B.n_windows, ctx->stream), "memset");
        cuda_check(cudaMemsetAsync(B.n_norms.p, 0, sizeof(int) * B.n_windows, ctx->stream), "memset");
        cuda_check(cudaMemsetAsync(B.norms.p, 0, sizeof(double) * B.n_windows * Batch::kNormStride, ctx->stream),
                   "memset");
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
        if (B.n_small > 0) {
            NvtxRange range("ba_batch");
            cuda_check(pvo_dev::launch_ba_batch(static_cast<const pvo_dev::BAParams*>(B.params.p), B.n_small,
                                                B.max_free, B.max_poses, ctx->stream),
                       "ba batch kernel");
            ctx->launches += 1;
        }
        for (size_t i = 0; i < B.large_idx.size(); ++i) {  // stream-ordered, sharing Batch::lb
            const Plan& pl = B.large_plans[i];
            upload(ctx, B.lb.g_begin, pl.g_begin.data(), pl.g_begin.size());
            upload(ctx, B.lb.g_lo, pl.g_lo.data(), pl.g_lo.size());
            upload(ctx, B.lb.g_nl, pl.g_nl.data(), pl.g_nl.size());
            upload(ctx, B.lb.g_off, pl.g_off.data(), pl.g_off.size());
            upload(ctx, B.lb.patch_group, pl.patch_group.data(), pl.patch_group.size());
            pvo_dev::BAParams a = B.hparams[B.large_idx[i]];
            launch_ba_checked(ctx, a, pl, &B.lb);
        }
        record_timing(ctx, 2);
        ctx->timing_pending = ctx->timing;
        if (corr_out && corr_memspace != PVO_DEVICE) download(ctx, corr_out, vol, (size_t)B.n_edges * 2 * 9 * 49);
    });
}

int pvo_batch_read(pvo_ctx* ctx, double* poses, double* inv_depth, double* residual_norms, int* n_norms) {
    return guarded(__func__, [&] {
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

}  // extern "C"
