// capi_provider.cu — extern "C" boundary: feature extraction, the correlation flow provider
// (measure / propose) and the simulator oracle provider.
#include "capi_common.hpp"

extern "C" {

// ---- feature extraction (features.cpp:55-235) -----------
// The frame's pyramid from its image, on the device, into frame-store `slot`
// (+ its Gram terms).  The store must have been reserved with C = 25 * bc and
// level sizes (iw/4, ih/4), (iw/16, ih/16).
int pvo_frames_extract(pvo_ctx* ctx, int slot, const float* image, int iw, int ih, int base_channels, int memspace) {
    return guarded(__func__, [&] {
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
        invalidate_g25(ctx, slot);
        if (memspace != PVO_DEVICE) sync(ctx);
    });
}

// A slot's pyramid back to the host (level0 [H0][W0][C], level1 [H1][W1][C]).
int pvo_frames_download(pvo_ctx* ctx, int slot, float* level0, float* level1) {
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
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
        ensure_g25(ctx, m);
        cuda_check(pvo_dev::launch_measure(m, ctx->stream), "measure kernel");
        ctx->launches += m.g25_0 ? 2 : 1;  // Gram-form kernel + exact replay
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
    return guarded(__func__, [&] {
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
        ensure_g25(ctx, m);
        cuda_check(pvo_dev::launch_measure(m, ctx->stream), "measure kernel");
        ctx->launches += m.g25_0 ? 2 : 1;  // Gram-form kernel + exact replay
        if (delta_out) download(ctx, delta_out, m.delta, (size_t)w.n_edges * 2);
        if (weight_out) download(ctx, weight_out, m.weight, (size_t)w.n_edges * 2);
        if (flags_out) download(ctx, flags_out, m.flags, w.n_edges);
        if (delta_out || weight_out || flags_out) sync(ctx);
    });
}

int pvo_measure_replayed(pvo_ctx* ctx, int* count) {
    return guarded(__func__, [&] {
        bind(ctx);
        if (!count) fail(PVO_INVALID_ARGUMENT, "measure_replayed: null output");
        *count = 0;
        if (ctx->replay.cap < 3 * sizeof(int)) return;
        cuda_check(cudaMemcpyAsync(count, static_cast<int*>(ctx->replay.p) + 1, sizeof(int), cudaMemcpyDeviceToHost,
                                   ctx->stream),
                   "replay count");
        sync(ctx);
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
    return guarded(__func__, [&] { ctx->oracle_rng.seed(seed); });
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
    return guarded(__func__, [&] {
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

}  // extern "C"
