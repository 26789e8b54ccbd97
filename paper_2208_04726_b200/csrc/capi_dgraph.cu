// capi_dgraph.cu — extern "C" boundary: the device-resident patch graph.
#include "capi_common.hpp"

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
    // grow d to at least `bytes` (doubling), preserving its contents
    void grow(DevBuf& d, size_t bytes) {
        if (bytes <= d.cap) return;
        DevBuf n;
        n.get(std::max(bytes, 2 * d.cap));
        // zero the new allocation first: the copy below moves the old capacity, whose
        // tail past the live entries was never written (compute-sanitizer initcheck)
        cuda_check(cudaMemsetAsync(n.p, 0, n.cap, ctx->stream), "grow");
        if (d.p) cuda_check(cudaMemcpyAsync(n.p, d.p, d.cap, cudaMemcpyDeviceToDevice, ctx->stream), "grow");
        cuda_check(cudaStreamSynchronize(ctx->stream), "grow");
        d.release();
        d = n;
        n.p = nullptr;
    }
    // grow buffer set b to hold np patches / ne edges, preserving contents
    void reserve(int b, int np, int ne) {
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
    return guarded(__func__, [&] {
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

// Capacity hint: size every graph buffer (both buffer sets, the frame arrays and
// the pass scratch) for `patches` patches, `edges` edges and `frames` frames up
// front, so a long-running per-frame loop never allocates inside a frame (a
// cudaMalloc can stall the host for milliseconds, and cudaFree synchronises the
// device).  Growth past the hint stays automatic.
int pvo_dgraph_reserve(pvo_dgraph* g, int patches, int edges, int frames) {
    return guarded(__func__, [&] {
        if (!g) fail(PVO_INVALID_ARGUMENT, "null graph");
        pvo_ctx* ctx = g->ctx;
        bind(ctx);
        if (patches < 0 || edges < 0 || frames < 0) fail(PVO_INVALID_ARGUMENT, "dgraph reserve: negative capacity");
        for (int b = 0; b < 2; ++b) g->reserve(b, std::max(patches, g->P), std::max(edges, g->E));
        const size_t F = std::max<size_t>((size_t)frames, g->f_index.size()) + 1;
        g->grow(g->f_pose_d, 8 * 7 * F);
        g->grow(g->f_idx_d, 4 * F);
        g->grow(g->f_slot_d, 4 * F);
        const size_t P1 = (size_t)std::max(patches, g->P) + 1;
        DevBuf* scratch[] = {&g->t0, &g->t1, &g->t2, &g->t3};
        for (DevBuf* t : scratch) t->get(4 * P1);
        g->t4.get(std::max(8 * P1, 8 * 7 * F));
        g->missing.get(4);
        g->w_nfixed.get(4);
        g->w_pose_frames.get(4 * F);
        g->w_fixed.get(F);
        g->w_patch_ids.get(4 * P1);
        g->w_e_graph.get(4 * ((size_t)std::max(edges, g->E) + 1));
        sync(ctx);
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
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
        if (n_frames) *n_frames = static_cast<int>(g->f_index.size());
        if (n_patches) *n_patches = g->P;
        if (n_edges) *n_edges = g->E;
    });
}

// edges in key order (kk = patch id, jj = frame), rev [E][4], has_rev [E] (host copies)
int pvo_dgraph_edges(pvo_dgraph* g, int* kk, int* jj, double* rev, uint8_t* has_rev) {
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
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
    return guarded(__func__, [&] {
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
// Windows beyond 16 free poses / 128 poses run on the large-window BA (its patch-group
// plan is built on the host from the device-flattened structure: one read-back).
int pvo_window_load_dgraph(pvo_ctx* ctx, pvo_dgraph* g, int window, int all_active, int* n_poses, int* n_patches,
                           int* n_edges) {
    return guarded(__func__, [&] {
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
        // windows beyond 16 free poses / 128 poses run on the multi-kernel large-window BA,
        // whose patch-group plan is built on the host from the flattened structure below
        const bool large = N - nfixed > pvo_dev::ba_max_free_poses() || N > pvo_dev::ba_max_poses();
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
        if (large) {
            // the large path's plan (plan_groups): patch runs by source pose, their free-pose
            // windows — from the device-flattened patch sources, edge CSR, edge poses and
            // free slots (edges are patch-contiguous: identity permutation)
            std::vector<int> src(Pw), ep(Ew);
            w.plan.edge_begin.resize(Pw + 1);
            w.plan.free_slot.resize(N);
            download(ctx, src.data(), o.patch_src, Pw);
            download(ctx, w.plan.edge_begin.data(), o.edge_begin, Pw + 1);
            download(ctx, ep.data(), o.e_pose, Ew);
            download(ctx, w.plan.free_slot.data(), o.free_slot, N);
            sync(ctx);
            w.plan.perm.resize(Ew);
            for (int e = 0; e < Ew; ++e) w.plan.perm[e] = e;
            HostProblem pr;
            pr.n_poses = N;
            pr.n_patches = Pw;
            pr.n_edges = Ew;
            pr.src = src.data();
            pr.e_pose = ep.data();
            w.plan.large = true;
            plan_groups(pr, w.plan);
            upload(ctx, B.g_begin, w.plan.g_begin.data(), w.plan.g_begin.size());
            upload(ctx, B.g_lo, w.plan.g_lo.data(), w.plan.g_lo.size());
            upload(ctx, B.g_nl, w.plan.g_nl.data(), w.plan.g_nl.size());
            upload(ctx, B.g_off, w.plan.g_off.data(), w.plan.g_off.size());
            upload(ctx, B.patch_group, w.plan.patch_group.data(), w.plan.patch_group.size());
        }
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
    return guarded(__func__, [&] {
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
}  // extern "C"
