// graph.cpp — host PatchGraph, window flattening, optimize_window driver and
// the host SE(3) log.
//
// The graph mirrors patch_graph.hpp:66-136 but is laid out for flattening:
// frames in a vector ordered by index (position = vector index), patches in
// a vector ordered by id (ids are issued increasing), and each patch owns
// its edges as a small vector ordered by frame index.  Iterating patches
// then edges therefore reproduces std::map<(patch, frame)> key order — the
// reference's edge order (patch-major, frame ascending) — without a tree.
// connect() visits only the positions within radius of the source
// (O(P * r) instead of the reference's O(P * F) scan) and produces the same
// edge set (patch_graph.cpp:62-85).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "geometry.cuh"
#include "internal.hpp"

using namespace pvo_host;
using pvo_dev::SE3;

namespace {

struct EdgeRec {
    int frame;
    bool has_rev;
    double delta[2], weight[2];
};
struct PatchRec {
    int id, src;
    std::vector<double> x, y;
    double d;
    std::vector<EdgeRec> edges;  // ordered by frame index
};
struct FrameRec {
    int index;
    double ts;
    double pose[7];
};
struct LogRec {
    int removed, anchor;
    double relative[7];
    double ts;
};

}  // namespace

struct pvo_graph {
    double K[4];
    int w, h, p;
    int next_id = 0;
    std::vector<FrameRec> frames;
    std::vector<PatchRec> patches;
    std::vector<LogRec> log;

    int position(int frame_index) const {
        auto it = std::lower_bound(frames.begin(), frames.end(), frame_index,
                                   [](const FrameRec& f, int v) { return f.index < v; });
        if (it == frames.end() || it->index != frame_index) {
            fail(PVO_OUT_OF_RANGE, "patch graph: no frame " + std::to_string(frame_index));
        }
        return static_cast<int>(it - frames.begin());
    }
    const FrameRec& frame(int frame_index) const { return frames[position(frame_index)]; }
    PatchRec& patch(int id) {
        auto it = std::lower_bound(patches.begin(), patches.end(), id,
                                   [](const PatchRec& p, int v) { return p.id < v; });
        if (it == patches.end() || it->id != id) fail(PVO_OUT_OF_RANGE, "patch graph: no patch " + std::to_string(id));
        return *it;
    }
};

namespace {

pvo_dev::Cam cam_of(const pvo_graph* g) { return {g->K[0], g->K[1], g->K[2], g->K[3]}; }

// reproject_patch center + behind (camera.cpp:47-71), host evaluation of the
// shared geometry.
void reproject_center_host(const pvo_graph* g, const PatchRec& pt, const double* pose_i, const double* pose_j,
                           double* cu, double* cv, bool* behind) {
    const SE3 pi = pvo_dev::se3_load(pose_i), pj = pvo_dev::se3_load(pose_j);
    const int pp = g->p * g->p;
    const int mid = pp / 2;
    if (pvo_dev::se3_equal(pi, pj)) {
        *cu = pt.x[mid];
        *cv = pt.y[mid];
        *behind = false;
        return;
    }
    const pvo_dev::Relative rel = pvo_dev::relative_pose(pi, pj);
    bool b = false;
    for (int k = 0; k < pp; ++k) {
        double u, v;
        const double qz = pvo_dev::reproject_point(rel, cam_of(g), pt.d, pt.x[k], pt.y[k], &u, &v);
        if (qz <= pvo_dev::kDepthEpsilon) b = true;
        if (k == mid) {
            *cu = u;
            *cv = v;
        }
    }
    *behind = b;
}

// The optimize_window problem build (bundle_adjust.cpp:231-307).
struct Flat {
    std::vector<int> pose_frames, patch_ids, src, e_patch, e_pose;
    std::vector<double> poses, px, py, depth, e_target, e_delta, e_weight;
    std::vector<uint8_t> fixed;
};

bool flatten(pvo_graph* g, int window, Flat& f) {
    if (window < 1) fail(PVO_INVALID_ARGUMENT, "ba: window must be >= 1");
    const int F = static_cast<int>(g->frames.size());
    const int window_start = std::max(F - window, 0);
    const int first_free = std::max(F - window, 1);
    const int pp = g->p * g->p;
    // included patches (ascending id) and their revised edges (frame order)
    std::vector<const PatchRec*> inc;
    for (const PatchRec& pt : g->patches) {
        if (g->position(pt.src) < window_start) continue;
        bool any = false;
        for (const EdgeRec& e : pt.edges) any = any || e.has_rev;
        if (any) inc.push_back(&pt);
    }
    if (inc.empty()) return false;
    // pose set = referenced frames in ascending index (slot order)
    std::vector<uint8_t> used(F, 0);
    for (const PatchRec* pt : inc) {
        used[g->position(pt->src)] = 1;
        for (const EdgeRec& e : pt->edges)
            if (e.has_rev) used[g->position(e.frame)] = 1;
    }
    std::vector<int> slot_of_pos(F, -1);
    for (int pos = 0; pos < F; ++pos) {
        if (!used[pos]) continue;
        slot_of_pos[pos] = static_cast<int>(f.pose_frames.size());
        f.pose_frames.push_back(g->frames[pos].index);
        f.poses.insert(f.poses.end(), g->frames[pos].pose, g->frames[pos].pose + 7);
        f.fixed.push_back(pos < first_free ? 1 : 0);
    }
    const double margin = 2.0 * 32.0;  // 2 * kMaxObservableMarginPx (bundle_adjust.hpp:18)
    for (size_t slot = 0; slot < inc.size(); ++slot) {
        const PatchRec& pt = *inc[slot];
        const int src_pos = g->position(pt.src);
        f.patch_ids.push_back(pt.id);
        f.src.push_back(slot_of_pos[src_pos]);
        f.px.insert(f.px.end(), pt.x.begin(), pt.x.begin() + pp);
        f.py.insert(f.py.end(), pt.y.begin(), pt.y.begin() + pp);
        f.depth.push_back(pt.d);
        for (const EdgeRec& e : pt.edges) {
            if (!e.has_rev) continue;
            const int tpos = g->position(e.frame);
            double cu, cv;
            bool behind;
            reproject_center_host(g, pt, g->frames[src_pos].pose, g->frames[tpos].pose, &cu, &cv, &behind);
            const bool observable = !behind && cu > -margin && cv > -margin && cu < g->w - 1 + margin &&
                                    cv < g->h - 1 + margin;
            f.e_patch.push_back(static_cast<int>(slot));
            f.e_pose.push_back(slot_of_pos[tpos]);
            f.e_target.push_back(cu + e.delta[0]);
            f.e_target.push_back(cv + e.delta[1]);
            f.e_delta.push_back(e.delta[0]);
            f.e_delta.push_back(e.delta[1]);
            f.e_weight.push_back(observable ? e.weight[0] : 0.0);
            f.e_weight.push_back(observable ? e.weight[1] : 0.0);
        }
    }
    return true;
}

}  // namespace

namespace pvo_host {

// se3.cpp:52-80
void se3_log_host(const double* pose, double* xi) {
    double qx = pose[0], qy = pose[1], qz = pose[2], qw = pose[3];
    if (qw < 0.0) {
        qx = -qx;
        qy = -qy;
        qz = -qz;
        qw = -qw;
    }
    const double vn = std::sqrt(qx * qx + qy * qy + qz * qz);
    const double theta = 2.0 * std::atan2(vn, qw);
    if (theta >= M_PI - 1e-6) fail(PVO_DOMAIN_ERROR, "se3 log: rotation angle within 1e-6 of pi");
    double o[3];
    if (theta < 1e-8 || vn < 1e-8) {
        o[0] = 2.0 * qx;
        o[1] = 2.0 * qy;
        o[2] = 2.0 * qz;
    } else {
        const double s = theta / vn;
        o[0] = s * qx;
        o[1] = s * qy;
        o[2] = s * qz;
    }
    const double t2 = o[0] * o[0] + o[1] * o[1] + o[2] * o[2];
    double c;
    if (t2 < 1e-16) {
        c = 1.0 / 12.0;
    } else {
        const double t = std::sqrt(t2);
        c = (1.0 - t * std::sin(t) / (2.0 * (1.0 - std::cos(t)))) / t2;
    }
    const double w[9] = {0, -o[2], o[1], o[2], 0, -o[0], -o[1], o[0], 0};
    double v[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const double ww = w[3 * i] * w[j] + w[3 * i + 1] * w[3 + j] + w[3 * i + 2] * w[6 + j];
            v[3 * i + j] = (i == j ? 1.0 : 0.0) - 0.5 * w[3 * i + j] + c * ww;
        }
    const double* t = pose + 4;
    for (int i = 0; i < 3; ++i) xi[i] = v[3 * i] * t[0] + v[3 * i + 1] * t[1] + v[3 * i + 2] * t[2];
    xi[3] = o[0];
    xi[4] = o[1];
    xi[5] = o[2];
}

}  // namespace pvo_host

extern "C" {

int pvo_graph_create(const double* K, int w, int h, int p, pvo_graph** out) {
    return guarded(__func__, [&] {
        if (!out) fail(PVO_INVALID_ARGUMENT, "null output");
        if (p < 1) fail(PVO_INVALID_ARGUMENT, "patch graph: patch width must be >= 1");
        if (K[0] <= 0 || K[1] <= 0) fail(PVO_INVALID_ARGUMENT, "intrinsics: focal lengths must be positive");
        auto* g = new pvo_graph();
        std::memcpy(g->K, K, sizeof(g->K));
        g->w = w;
        g->h = h;
        g->p = p;
        *out = g;
    });
}

int pvo_graph_destroy(pvo_graph* g) {
    delete g;
    return PVO_OK;
}

// patch_graph.cpp:27-34
int pvo_graph_add_frame(pvo_graph* g, double ts, const double* pose, int* out_index) {
    return guarded(__func__, [&] {
        if (!g->frames.empty() && ts <= g->frames.back().ts) {
            fail(PVO_INVALID_ARGUMENT, "patch graph: timestamp must exceed the last frame's");
        }
        FrameRec f;
        f.index = g->frames.empty() ? 0 : g->frames.back().index + 1;
        f.ts = ts;
        std::memcpy(f.pose, pose, sizeof(f.pose));
        g->frames.push_back(f);
        if (out_index) *out_index = f.index;
    });
}

// patch_graph.cpp:36-60 + Patch::make (camera.cpp:15-32)
int pvo_graph_add_patches(pvo_graph* g, int frame, int n, const double* centroids, const double* depths, int* out_ids) {
    return guarded(__func__, [&] {
        bool found = false;
        for (const FrameRec& f : g->frames) found = found || f.index == frame;
        if (!found) fail(PVO_INVALID_ARGUMENT, "patch graph: no frame " + std::to_string(frame));
        const double half = 0.5 * (g->p - 1);
        for (int k = 0; k < n; ++k) {
            const double cx = centroids[2 * k], cy = centroids[2 * k + 1];
            if (cx - half < 0 || cy - half < 0 || cx + half > g->w - 1 || cy + half > g->h - 1) {
                fail(PVO_INVALID_ARGUMENT, "patch graph: centroid (" + std::to_string(cx) + ", " + std::to_string(cy) +
                                               ") leaves the image bounds");
            }
        }
        for (int k = 0; k < n; ++k) {
            if (depths[k] < 0) fail(PVO_INVALID_ARGUMENT, "patch: inverse depth must be >= 0");
        }
        for (int k = 0; k < n; ++k) {
            PatchRec pt;
            pt.id = g->next_id++;
            pt.src = frame;
            pt.d = depths[k];
            const double cx = centroids[2 * k], cy = centroids[2 * k + 1];
            for (int row = 0; row < g->p; ++row)
                for (int col = 0; col < g->p; ++col) {
                    pt.x.push_back(cx + col - half);
                    pt.y.push_back(cy + row - half);
                }
            if (out_ids) out_ids[k] = pt.id;
            g->patches.push_back(std::move(pt));
        }
    });
}

// patch_graph.cpp:62-85: edge iff |pos(src) - pos(j)| <= r - 1.
int pvo_graph_connect(pvo_graph* g, int radius, int* n_added) {
    return guarded(__func__, [&] {
        if (radius < 1) fail(PVO_INVALID_ARGUMENT, "patch graph: radius must be >= 1");
        int added = 0;
        const int F = static_cast<int>(g->frames.size());
        for (PatchRec& pt : g->patches) {
            const int s = g->position(pt.src);
            const int lo = std::max(0, s - (radius - 1)), hi = std::min(F - 1, s + (radius - 1));
            // merge the position range into the (frame-ordered) edge list
            std::vector<EdgeRec> merged;
            merged.reserve(pt.edges.size() + (hi - lo + 1));
            size_t i = 0;
            for (int pos = lo; pos <= hi; ++pos) {
                const int fi = g->frames[pos].index;
                while (i < pt.edges.size() && pt.edges[i].frame < fi) merged.push_back(pt.edges[i++]);
                if (i < pt.edges.size() && pt.edges[i].frame == fi) {
                    merged.push_back(pt.edges[i++]);
                } else {
                    merged.push_back(EdgeRec{fi, false, {0, 0}, {0, 0}});
                    ++added;
                }
            }
            while (i < pt.edges.size()) merged.push_back(pt.edges[i++]);
            pt.edges.swap(merged);
        }
        if (n_added) *n_added = added;
    });
}

// patch_graph.cpp:87-128
int pvo_graph_remove_frame(pvo_graph* g, int frame) {
    return guarded(__func__, [&] {
        int pos = -1;
        for (size_t i = 0; i < g->frames.size(); ++i)
            if (g->frames[i].index == frame) pos = static_cast<int>(i);
        if (pos < 0) fail(PVO_INVALID_ARGUMENT, "patch graph: no frame " + std::to_string(frame));
        if (pos >= static_cast<int>(g->frames.size()) - 3) {
            fail(PVO_INVALID_ARGUMENT, "patch graph: frame " + std::to_string(frame) +
                                           " is among the most recent 3 keyframes");
        }
        if (pos == 0) fail(PVO_INVALID_ARGUMENT, "patch graph: the oldest frame has no predecessor to anchor");
        const FrameRec& cur = g->frames[pos];
        const FrameRec& pred = g->frames[pos - 1];
        LogRec lr;
        lr.removed = frame;
        lr.anchor = pred.index;
        lr.ts = cur.ts;
        pvo_dev::se3_store(pvo_dev::se3_compose(pvo_dev::se3_load(cur.pose), pvo_dev::se3_inverse(pvo_dev::se3_load(pred.pose))),
                           lr.relative);
        g->log.push_back(lr);
        std::vector<PatchRec> kept;
        for (PatchRec& pt : g->patches) {
            if (pt.src == frame) continue;
            pt.edges.erase(std::remove_if(pt.edges.begin(), pt.edges.end(),
                                          [frame](const EdgeRec& e) { return e.frame == frame; }),
                           pt.edges.end());
            kept.push_back(std::move(pt));
        }
        g->patches.swap(kept);
        g->frames.erase(g->frames.begin() + pos);
    });
}

// patch_graph.cpp:153-164
int pvo_graph_set_revision(pvo_graph* g, int patch_id, int frame, const double* delta, const double* weight) {
    return guarded(__func__, [&] {
        EdgeRec* hit = nullptr;
        for (PatchRec& pt : g->patches) {
            if (pt.id != patch_id) continue;
            for (EdgeRec& e : pt.edges)
                if (e.frame == frame) hit = &e;
        }
        if (!hit) {
            fail(PVO_INVALID_ARGUMENT, "patch graph: no edge (" + std::to_string(patch_id) + ", " +
                                           std::to_string(frame) + ")");
        }
        if (weight[0] <= 0 || weight[0] >= 1 || weight[1] <= 0 || weight[1] >= 1) {
            fail(PVO_INVALID_ARGUMENT, "patch graph: revision weights must lie in (0, 1)");
        }
        hit->has_rev = true;
        hit->delta[0] = delta[0];
        hit->delta[1] = delta[1];
        hit->weight[0] = weight[0];
        hit->weight[1] = weight[1];
    });
}

int pvo_graph_set_pose(pvo_graph* g, int frame, const double* pose) {
    return guarded(__func__, [&] { std::memcpy(g->frames[g->position(frame)].pose, pose, 7 * sizeof(double)); });
}
int pvo_graph_set_inverse_depth(pvo_graph* g, int patch_id, double d) {
    return guarded(__func__, [&] { g->patch(patch_id).d = d; });
}
int pvo_graph_num_frames(pvo_graph* g) { return static_cast<int>(g->frames.size()); }
int pvo_graph_num_patches(pvo_graph* g) { return static_cast<int>(g->patches.size()); }
int pvo_graph_num_edges(pvo_graph* g) {
    size_t n = 0;
    for (const PatchRec& pt : g->patches) n += pt.edges.size();
    return static_cast<int>(n);
}

int pvo_graph_edges(pvo_graph* g, int* kk, int* jj, double* rev, uint8_t* has_rev) {
    return guarded(__func__, [&] {
        size_t i = 0;
        for (const PatchRec& pt : g->patches) {
            for (const EdgeRec& e : pt.edges) {
                kk[i] = pt.id;
                jj[i] = e.frame;
                if (rev) {
                    rev[4 * i] = e.has_rev ? e.delta[0] : 0.0;
                    rev[4 * i + 1] = e.has_rev ? e.delta[1] : 0.0;
                    rev[4 * i + 2] = e.has_rev ? e.weight[0] : 0.0;
                    rev[4 * i + 3] = e.has_rev ? e.weight[1] : 0.0;
                }
                if (has_rev) has_rev[i] = e.has_rev ? 1 : 0;
                ++i;
            }
        }
    });
}

int pvo_graph_frames(pvo_graph* g, int* indices, double* poses) {
    return guarded(__func__, [&] {
        for (size_t i = 0; i < g->frames.size(); ++i) {
            indices[i] = g->frames[i].index;
            if (poses) std::memcpy(poses + 7 * i, g->frames[i].pose, 7 * sizeof(double));
        }
    });
}

int pvo_graph_patches(pvo_graph* g, int* ids, int* src, double* depth) {
    return guarded(__func__, [&] {
        for (size_t i = 0; i < g->patches.size(); ++i) {
            ids[i] = g->patches[i].id;
            if (src) src[i] = g->patches[i].src;
            if (depth) depth[i] = g->patches[i].d;
        }
    });
}

// Pipeline::active_edges (pipeline.cpp:164-181)
int pvo_graph_active_edges(pvo_graph* g, int window, int* kk, int* jj, int* n) {
    return guarded(__func__, [&] {
        int oldest = 0;
        if (!g->frames.empty() && window > 0) {
            const int F = static_cast<int>(g->frames.size());
            oldest = g->frames[std::max(F - window, 0)].index;
        }
        int i = 0;
        for (const PatchRec& pt : g->patches) {
            if (pt.src < oldest) continue;
            for (const EdgeRec& e : pt.edges) {
                if (kk) {
                    kk[i] = pt.id;
                    jj[i] = e.frame;
                }
                ++i;
            }
        }
        *n = i;
    });
}

// build_target (bundle_adjust.cpp:47-60)
int pvo_graph_build_target(pvo_graph* g, int patch_id, int frame, double* out) {
    return guarded(__func__, [&] {
        const EdgeRec* hit = nullptr;
        const PatchRec* owner = nullptr;
        for (const PatchRec& pt : g->patches) {
            if (pt.id != patch_id) continue;
            for (const EdgeRec& e : pt.edges)
                if (e.frame == frame) {
                    hit = &e;
                    owner = &pt;
                }
        }
        if (!hit) fail(PVO_INVALID_ARGUMENT, "build_target: no such edge");
        if (!hit->has_rev) fail(PVO_INVALID_ARGUMENT, "build_target: edge has no revision");
        double cu, cv;
        bool behind;
        reproject_center_host(g, *owner, g->frame(owner->src).pose, g->frame(frame).pose, &cu, &cv, &behind);
        out[0] = cu + hit->delta[0];
        out[1] = cv + hit->delta[1];
    });
}

int pvo_graph_window_problem(pvo_graph* g, int window, int* n_poses, int* n_patches, int* n_edges, int* pose_frames,
                             double* poses, uint8_t* fixed, int* patch_ids, int* patch_src, double* px, double* py,
                             double* depth, int* e_patch, int* e_pose, double* e_target, double* e_weight) {
    return guarded(__func__, [&] {
        Flat f;
        if (!flatten(g, window, f)) {
            *n_poses = *n_patches = *n_edges = 0;
            return;
        }
        *n_poses = static_cast<int>(f.pose_frames.size());
        *n_patches = static_cast<int>(f.patch_ids.size());
        *n_edges = static_cast<int>(f.e_patch.size());
        if (!pose_frames) return;
        std::copy(f.pose_frames.begin(), f.pose_frames.end(), pose_frames);
        std::copy(f.poses.begin(), f.poses.end(), poses);
        std::copy(f.fixed.begin(), f.fixed.end(), fixed);
        std::copy(f.patch_ids.begin(), f.patch_ids.end(), patch_ids);
        std::copy(f.src.begin(), f.src.end(), patch_src);
        std::copy(f.px.begin(), f.px.end(), px);
        std::copy(f.py.begin(), f.py.end(), py);
        std::copy(f.depth.begin(), f.depth.end(), depth);
        std::copy(f.e_patch.begin(), f.e_patch.end(), e_patch);
        std::copy(f.e_pose.begin(), f.e_pose.end(), e_pose);
        std::copy(f.e_target.begin(), f.e_target.end(), e_target);
        std::copy(f.e_weight.begin(), f.e_weight.end(), e_weight);
    });
}

// optimize_window (bundle_adjust.cpp:225-375): host flattening, device
// iterations (targets frozen on the device), write-back of free poses and
// every included depth (:368-373).
int pvo_optimize_window(pvo_ctx* ctx, pvo_graph* g, int window, int iterations, int structure_only, double damping,
                        double* residual_norms, int* n_norms, int* num_edges) {
    return guarded(__func__, [&] {
        Flat f;
        if (n_norms) *n_norms = 0;
        if (num_edges) *num_edges = 0;
        if (!flatten(g, window, f)) return;
        HostProblem pr;
        pr.n_poses = static_cast<int>(f.pose_frames.size());
        pr.poses = f.poses.data();
        pr.fixed = f.fixed.data();
        pr.n_patches = static_cast<int>(f.patch_ids.size());
        pr.p = g->p;
        pr.src = f.src.data();
        pr.px = f.px.data();
        pr.py = f.py.data();
        pr.depth = f.depth.data();
        pr.n_edges = static_cast<int>(f.e_patch.size());
        pr.e_patch = f.e_patch.data();
        pr.e_pose = f.e_pose.data();
        pr.e_in = f.e_delta.data();
        // freeze on the device: raw revision weights, observability applied there
        std::vector<double> raw_w;
        raw_w.reserve(f.e_weight.size());
        {
            size_t i = 0;
            for (const PatchRec& pt : g->patches) {
                bool included = std::binary_search(f.patch_ids.begin(), f.patch_ids.end(), pt.id);
                if (!included) continue;
                for (const EdgeRec& e : pt.edges) {
                    if (!e.has_rev) continue;
                    raw_w.push_back(e.weight[0]);
                    raw_w.push_back(e.weight[1]);
                    ++i;
                }
            }
        }
        pr.e_w = raw_w.data();
        std::memcpy(pr.K, g->K, sizeof(pr.K));
        pr.image_w = g->w;
        pr.image_h = g->h;
        pr.damping = damping;
        std::vector<double> out_poses(f.poses.size()), out_depth(f.depth.size());
        BARun run;
        run.freeze_targets = 1;
        run.iterations = iterations;
        run.structure_only = structure_only;
        run.out_poses = out_poses.data();
        run.out_depth = out_depth.data();
        run.residual_norms = residual_norms;
        run.n_norms = n_norms;
        run_ba(ctx, pr, run);
        for (size_t slot = 0; slot < f.pose_frames.size(); ++slot) {
            if (!f.fixed[slot]) std::memcpy(g->frames[g->position(f.pose_frames[slot])].pose, &out_poses[7 * slot], 7 * sizeof(double));
        }
        for (size_t slot = 0; slot < f.patch_ids.size(); ++slot) g->patch(f.patch_ids[slot]).d = out_depth[slot];
        if (num_edges) *num_edges = pr.n_edges;
    });
}

}  // extern "C"
