// capi_window.cu — extern "C" boundary: the resident window (the per-frame hot path).
#include "capi_common.hpp"

extern "C" {

// ---- resident window ------------------------------------------------------------
int pvo_window_load(pvo_ctx* ctx, int n_poses, const double* poses, const uint8_t* fixed, const int* pose_slot,
                    int n_patches, int p, const int* src, const double* px, const double* py, const double* depth,
                    const float* patch_feats, int n_edges, const int* e_patch, const int* e_pose,
                    const double* e_delta, const double* e_weight, const double* K, int image_w, int image_h,
                    int memspace) {
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
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
        // the read-back copies the whole norms buffer: no uninitialised tail
        cuda_check(cudaMemsetAsync(a.residual_norms, 0, ctx->ba.norms.cap, ctx->stream), "memset");
        launch_ba_checked(ctx, a, w.plan);
        record_timing(ctx, 2);
        ctx->timing_pending = ctx->timing;
        if (readback) cuda_check(cudaStreamWaitEvent(ctx->stream, ctx->ev_copy, 0), "stream wait");
    });
}

// optimize_window's iterations on the resident window without the correlation
// pass (the per-frame pipeline: propose -> BA, pipeline.cpp:183-198)
int pvo_window_ba(pvo_ctx* ctx, int iterations, double damping) {
    return guarded(__func__, [&] {
        bind(ctx);
        Window& w = ctx->win;
        if (!w.loaded) fail(PVO_INVALID_ARGUMENT, "window: nothing loaded");
        if (iterations < 0) fail(PVO_INVALID_ARGUMENT, "ba: negative iteration count");
        if (iterations > PVO_MAX_WINDOW_ITERATIONS) fail(PVO_INVALID_ARGUMENT, "ba: too many iterations");
        reset_status(ctx);
        pvo_dev::BAParams a = window_ba_params(ctx, iterations, damping);
        // the read-back copies the whole norms buffer: no uninitialised tail
        cuda_check(cudaMemsetAsync(a.residual_norms, 0, ctx->ba.norms.cap, ctx->stream), "memset");
        launch_ba_checked(ctx, a, w.plan);
    });
}

int pvo_window_read(pvo_ctx* ctx, double* poses, double* depth, double* residual_norms, int* n_norms) {
    return guarded(__func__, [&] {
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

int pvo_window_problem_read(pvo_ctx* ctx, double* poses, uint8_t* fixed, int* pose_slot, int* patch_src, double* px,
                            double* py, double* depth, int* e_patch, int* e_pose, double* e_delta, double* e_weight) {
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
        bind(ctx);
        if (!ctx->win.loaded) fail(PVO_INVALID_ARGUMENT, "window: nothing loaded");
        *corr = static_cast<float*>(ctx->win.corr.p);
    });
}

}  // extern "C"

