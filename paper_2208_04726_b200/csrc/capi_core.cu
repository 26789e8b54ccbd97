// capi_core.cu — extern "C" boundary: library / context, SE(3) host
// utilities, camera, single-patch and batched correlation, the frame store,
// gauss_newton_step / schur_solve / the optimize_window loop on flat problems.
#include "capi_common.hpp"

namespace pvo_host {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace pvo_host

namespace pvo_host {

// Patches of any odd width p on the 3 x 3 kernels: the bundle adjustment reads a
// patch only through (a) its centre pixel p*p/2 — the Jacobian centre
// Patch::center(), the frozen-target and WRMS centre PatchReprojection::center()
// (camera.cpp:34-44, camera.hpp:49), one and the same pixel for odd p — and
// (b) the behind-camera test "any pixel with q_z <= eps" (camera.cpp:47-71).  q_z
// is affine in the pixel coordinates and the patch grid is axis-aligned, so its
// minimum over the p x p grid is attained at one of the 4 corners: the 3 x 3
// stand-in {first, centre, last column} x {first, centre, last row} carries
// exactly the pixels the reference's decisions depend on.  (Even widths use the
// pixel mean as the Jacobian centre but pixel p*p/2 for targets: unsupported.)
static HostProblem as_3x3(const HostProblem& pr, std::vector<double>& px9, std::vector<double>& py9) {
    if (pr.p < 1) fail(PVO_INVALID_ARGUMENT, "patch: width must be >= 1");
    if (pr.p == 3) return pr;
    if (pr.p % 2 == 0) fail(PVO_UNSUPPORTED, "ba: even patch widths (the Jacobian centre is not a pixel)");
    const int p = pr.p, cols[3] = {0, p / 2, p - 1};
    px9.resize((size_t)pr.n_patches * 9);
    py9.resize((size_t)pr.n_patches * 9);
    for (int k = 0; k < pr.n_patches; ++k)
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                const size_t src = (size_t)k * p * p + (size_t)cols[r] * p + cols[c];
                px9[(size_t)k * 9 + 3 * r + c] = pr.px[src];
                py9[(size_t)k * 9 + 3 * r + c] = pr.py[src];
            }
    HostProblem q = pr;
    q.p = 3;
    q.px = px9.data();
    q.py = py9.data();
    return q;
}

void run_ba(pvo_ctx* ctx, const HostProblem& pr_in, const BARun& run) {
    bind(ctx);
    std::vector<double> px9, py9;
    const HostProblem pr = as_3x3(pr_in, px9, py9);
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
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        DevBuf* bufs[] = {&ctx->feat0, &ctx->feat1, &ctx->gram0, &ctx->gram1, &ctx->g25_0, &ctx->g25_1, &ctx->replay, &ctx->s0, &ctx->s1, &ctx->s2,
                          &ctx->s3,    &ctx->s4,    &ctx->s5,    &ctx->s6,    &ctx->s7, &ctx->s8,
                          &ctx->win.pose_slot, &ctx->win.patch_feats, &ctx->win.corr, &ctx->win.init_poses,
                          &ctx->win.init_depth, &ctx->win.order, &ctx->win.order_half, &ctx->win.flags, &ctx->c_coords, &ctx->c_meta,
                          &ctx->c_over, &ctx->c_order};
        for (DevBuf* b : bufs) b->release();
        ctx->ba.release();
        ctx->bat.release();
        grid_cache_clear(ctx);
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
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
        bind(ctx);
        sync(ctx);
    });
}

int64_t pvo_ctx_kernel_launches(pvo_ctx* ctx) { return ctx ? ctx->launches : -1; }

int pvo_ctx_set_timing(pvo_ctx* ctx, int on) {
    return guarded(__func__, [&] {
        bind(ctx);
        ctx->timing = on != 0;
        if (!ctx->timing) ctx->timing_pending = false;
    });
}

int pvo_ctx_set_tracing(pvo_ctx* ctx, int on) {
    return guarded(__func__, [&] {
        bind(ctx);
        ctx->tracing = on != 0;
        if (ctx->tracing) {
            long long* c = ctx->ba.clocks.as<long long>(128);
            cuda_check(cudaMemsetAsync(c, 0, 128 * sizeof(long long), ctx->stream), "memset");
        }
    });
}

int pvo_ctx_ba_phase_cycles(pvo_ctx* ctx, long long* out128) {
    return guarded(__func__, [&] {
        bind(ctx);
        if (!ctx->tracing) fail(PVO_INVALID_ARGUMENT, "tracing is off (pvo_ctx_set_tracing)");
        download(ctx, out128, static_cast<const long long*>(ctx->ba.clocks.p), 128);
        sync(ctx);
    });
}

int pvo_ctx_ba_attempts(pvo_ctx* ctx, int* attempts) {
    return guarded(__func__, [&] {
        bind(ctx);
        *attempts = 0;
        if (ctx->ba.attempts.p) {
            download(ctx, attempts, static_cast<const int*>(ctx->ba.attempts.p), 1);
            sync(ctx);
        }
    });
}

int pvo_ctx_last_timing(pvo_ctx* ctx, double* corr_ms, double* ba_ms) {
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] { pvo_dev::se3_store(pvo_dev::se3_exp(xi), out); });
}
int pvo_se3_log(const double* pose, double* xi) {
    return guarded(__func__, [&] { se3_log_host(pose, xi); });
}
int pvo_se3_compose(const double* a, const double* b, double* out) {
    return guarded(__func__, [&] {
        pvo_dev::se3_store(pvo_dev::se3_compose(pvo_dev::se3_load(a), pvo_dev::se3_load(b)), out);
    });
}
int pvo_se3_inverse(const double* a, double* out) {
    return guarded(__func__, [&] { pvo_dev::se3_store(pvo_dev::se3_inverse(pvo_dev::se3_load(a)), out); });
}
int pvo_se3_retract(const double* a, const double* xi, double* out) {
    return guarded(__func__, [&] { pvo_dev::se3_store(pvo_dev::se3_retract(pvo_dev::se3_load(a), xi), out); });
}

// ---- camera ----------------------------------------------------------------
int pvo_reproject_patches(pvo_ctx* ctx, int n, int p, const double* pi, const double* pj, const double* K,
                          const double* x, const double* y, const double* d, double* out_xy, uint8_t* behind) {
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
        bind(ctx);
        if (p < 1 || C < 1 || w0 < 0 || h0 < 0 || w1 < 0 || h1 < 0) fail(PVO_INVALID_ARGUMENT, "correlate: bad sizes");
        const int pp = p * p;
        for (int k = 0; k < pp; ++k)
            if (!finite2(coords + 2 * k)) fail(PVO_INVALID_ARGUMENT, "correlate: non-finite reprojection");
        // the pyramid stays on the device between calls (grid cache); Gram terms only for the 3x3 kernel
        GridEntry* g0 = cached_grid(ctx, level0, w0, h0, C, p == 3);
        GridEntry* g1 = cached_grid(ctx, level1, w1, h1, C, p == 3);
        const float* f0 = static_cast<const float*>(g0->feat.p);
        const float* f1 = static_cast<const float*>(g1->feat.p);
        float* pf = ctx->s4.as<float>((size_t)2 * pp * C);
        cuda_check(cudaMemcpyAsync(pf, feats0, sizeof(float) * pp * C, cudaMemcpyHostToDevice, ctx->stream), "H2D");
        cuda_check(cudaMemcpyAsync(pf + (size_t)pp * C, feats1, sizeof(float) * pp * C, cudaMemcpyHostToDevice,
                                   ctx->stream),
                   "H2D");
        double* dc = upload(ctx, ctx->s5, coords, (size_t)2 * pp);
        float* dout = ctx->s7.as<float>((size_t)2 * pp * 49);
        if (p != 3) {  // any other width: the direct FP64 form of correlation.cpp:8-71
            cuda_check(pvo_dev::launch_corr_direct(pp, C, pf, dc, f0, w0, h0, f1, w1, h1, dout, ctx->stream),
                       "corr_direct kernel");
            ctx->launches += 1;
            download(ctx, out, dout, (size_t)2 * pp * 49);
            sync(ctx);
            return;
        }
        int zero = 0;
        int* idx = upload(ctx, ctx->s6, &zero, 1);
        reset_status(ctx);
        pvo_dev::CorrParams cp;
        cp.n_edges = 1;
        cp.channels = C;
        cp.e_patch = idx;
        cp.e_slot = idx;
        cp.coords = dc;
        cp.feat0 = f0;
        cp.feat1 = f1;
        cp.gram0 = static_cast<const float*>(g0->gram.p);
        cp.gram1 = static_cast<const float*>(g1->gram.p);
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

int pvo_correlate_points(pvo_ctx* ctx, int n, int C, const float* features, const float* grid, int w, int h,
                         const double* xy, int cubic, double* out) {
    return guarded(__func__, [&] {
        bind(ctx);
        if (n < 0 || C < 1 || w < 0 || h < 0) fail(PVO_INVALID_ARGUMENT, "correlate_at: bad sizes");
        if (n == 0) return;
        GridEntry* g = cached_grid(ctx, grid, w, h, C, false);
        pvo_dev::PointsParams a;
        a.n = n;
        a.channels = C;
        a.cubic = cubic ? 1 : 0;
        a.features = upload(ctx, ctx->s0, features, (size_t)n * C);
        a.xy = upload(ctx, ctx->s1, xy, (size_t)n * 2);
        a.grid = static_cast<const float*>(g->feat.p);
        a.W = w;
        a.H = h;
        a.out = ctx->s2.as<double>(n);
        cuda_check(pvo_dev::launch_points(a, ctx->stream), "points kernel");
        ctx->launches += 1;
        download(ctx, out, a.out, n);
        sync(ctx);
    });
}

int pvo_grid_cache_stats(pvo_ctx* ctx, int64_t* hits, int64_t* misses, int* entries, int64_t* bytes) {
    return guarded(__func__, [&] {
        if (!ctx) fail(PVO_INVALID_ARGUMENT, "null context");
        if (hits) *hits = ctx->grid_hits;
        if (misses) *misses = ctx->grid_misses;
        if (entries) *entries = (int)ctx->grids.size();
        if (bytes) *bytes = (int64_t)ctx->grid_bytes;
    });
}

int pvo_grid_cache_clear(pvo_ctx* ctx) {
    return guarded(__func__, [&] {
        bind(ctx);
        sync(ctx);
        grid_cache_clear(ctx);
    });
}

int pvo_frames_reserve(pvo_ctx* ctx, int n_frames, int w0, int h0, int w1, int h1, int C) {
    return guarded(__func__, [&] {
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
        ctx->g25_valid.assign(n_frames, 0);
        // row-pad cells of the Gram planes must read as zero (out of the image)
        cuda_check(cudaMemsetAsync(ctx->gram0.p, 0, gb0, ctx->stream), "memset");
        cuda_check(cudaMemsetAsync(ctx->gram1.p, 0, gb1, ctx->stream), "memset");
        encode_frame_maps(ctx);
    });
}

int pvo_frames_refresh(pvo_ctx* ctx, int slot) {
    return guarded(__func__, [&] {
        bind(ctx);
        if (slot < 0 || slot >= ctx->nf) fail(PVO_OUT_OF_RANGE, "frames: slot out of range");
        const size_t c0 = (size_t)ctx->w0 * ctx->h0, c1 = (size_t)ctx->w1 * ctx->h1;
        float* f0 = static_cast<float*>(ctx->feat0.p) + slot * c0 * ctx->C;
        float* f1 = static_cast<float*>(ctx->feat1.p) + slot * c1 * ctx->C;
        float* g0 = static_cast<float*>(ctx->gram0.p) + (size_t)slot * pvo_dev::gram_stride(ctx->w0) * ctx->h0 * 8;
        float* g1 = static_cast<float*>(ctx->gram1.p) + (size_t)slot * pvo_dev::gram_stride(ctx->w1) * ctx->h1 * 8;
        compute_gram(ctx, f0, g0, f1, g1, ctx->w0, ctx->h0, ctx->w1, ctx->h1, ctx->C);
        invalidate_g25(ctx, slot);
    });
}

int pvo_frames_upload(pvo_ctx* ctx, int slot, const float* level0, const float* level1, int memspace) {
    return guarded(__func__, [&] {
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
        invalidate_g25(ctx, slot);
        if (memspace != PVO_DEVICE) sync(ctx);
    });
}

int pvo_frames_device_ptrs(pvo_ctx* ctx, float** level0, float** level1) {
    return guarded(__func__, [&] {
        bind(ctx);
        if (level0) *level0 = static_cast<float*>(ctx->feat0.p);
        if (level1) *level1 = static_cast<float*>(ctx->feat1.p);
    });
}

int pvo_correlate_batch(pvo_ctx* ctx, int n_edges, int n_patches, int p, const int* e_patch, const int* e_slot,
                        const double* coords, const float* patch_feats, float* out, int memspace) {
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
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

}  // extern "C"
