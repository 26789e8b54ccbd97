// oracle/_ref adapter — TEST INFRASTRUCTURE ONLY.
//
// Exports the same flat `orc_*` C surface as oracle/pvo_oracle.cpp (the
// restatement), but every entry calls the REFERENCE's own functions from
// /root/reference/proj/src, compiled unmodified by oracle/ref_build.py
// against the in-repo Eigen / doctest / json / png shims (oracle/ref_shim/).
// oracle/pyoracle.py prefers this library when it exists, so the parity
// tests compare the CUDA path with the reference itself.
//
// Only the argument marshalling lives here.  Two entry points have no
// counterpart in the reference's public API and restate a few lines of it on
// top of the reference's own operators (cited): orc_window_problem (the
// problem build inside optimize_window, bundle_adjust.cpp:231-307) and
// orc_ba_window (optimize_window's iteration loop, bundle_adjust.cpp:309-366,
// on a flat problem with frozen targets).  orc_graph_active_edges restates
// Pipeline::active_edges (pipeline.cpp:164-181), a Pipeline member.
// Poses cross the surface as 7 raw doubles and are reloaded bit for bit
// (see load_pose).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "pvo/bundle_adjust.hpp"
#include "pvo/camera.hpp"
#include "pvo/correlation.hpp"
#include "pvo/features.hpp"
#include "pvo/flow_provider.hpp"
#include "pvo/patch_graph.hpp"
#include "pvo/se3.hpp"

using namespace pvo;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const DegenerateProblem& e) {
        g_err = e.what();
        return 2;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

// The flat surface carries poses that came out of the reference's own
// operators (already normalised by Pose(q, t), se3.hpp:41).  Renormalising
// them again is not idempotent in the last ulp, so they are reloaded bit for
// bit: the member quaternion is written through rotation()'s reference (the
// Pose object itself is not const, so the const_cast is well defined).
Pose load_pose(const double* p) {
    Pose pose(Quat::Identity(), Vec3(p[4], p[5], p[6]));
    const_cast<Quat&>(pose.rotation()).coeffs() = Eigen::Vector4d(p[0], p[1], p[2], p[3]);
    return pose;
}
void store_pose(const Pose& p, double* o) {
    const auto& c = p.rotation().coeffs();  // x y z w
    o[0] = c(0);
    o[1] = c(1);
    o[2] = c(2);
    o[3] = c(3);
    o[4] = p.translation().x();
    o[5] = p.translation().y();
    o[6] = p.translation().z();
}
Intrinsics load_K(const double* k) { return Intrinsics(k[0], k[1], k[2], k[3]); }
Tangent load_xi(const double* xi) { return Tangent(Vec3(xi[0], xi[1], xi[2]), Vec3(xi[3], xi[4], xi[5])); }
Patch load_patch(int p, const double* x, const double* y, double d, int src) {
    Patch pt;
    pt.width = p;
    pt.source_frame = src;
    pt.inverse_depth = d;
    pt.x.assign(x, x + p * p);
    pt.y.assign(y, y + p * p);
    return pt;
}
FeatureGrid load_grid(const float* data, int w, int h, int c) {
    FeatureGrid g(w, h, c);
    std::memcpy(g.data.data(), data, sizeof(float) * g.data.size());
    return g;
}
PatchFeatures load_feats(int p, int channels, const float* g0, const float* g1) {
    PatchFeatures f;
    f.width = p;
    f.channels = channels;
    f.level0.assign(g0, g0 + static_cast<size_t>(p) * p * channels);
    f.level1.assign(g1, g1 + static_cast<size_t>(p) * p * channels);
    return f;
}

BAProblem load_problem(int n_poses, const double* poses, const uint8_t* fixed, int n_patches, int p,
                       const int* src, const double* px, const double* py, const double* depth,
                       const uint8_t* depth_free, int n_edges, const int* e_patch, const int* e_pose,
                       const double* e_target, const double* e_weight, const double* K, double damping) {
    BAProblem pr;
    for (int i = 0; i < n_poses; ++i) {
        pr.poses.push_back(load_pose(poses + 7 * i));
        pr.pose_fixed.push_back(fixed[i] != 0);
    }
    for (int k = 0; k < n_patches; ++k) {
        pr.patches.push_back(load_patch(p, px + k * p * p, py + k * p * p, depth[k], src[k]));
    }
    if (depth_free) {
        for (int k = 0; k < n_patches; ++k) pr.depth_free.push_back(depth_free[k] != 0);
    }
    for (int e = 0; e < n_edges; ++e) {
        BAEdge ed;
        ed.patch_id = e_patch[e];
        ed.target_pose = e_pose[e];
        ed.target_point = Vec2(e_target[2 * e], e_target[2 * e + 1]);
        ed.weight = Vec2(e_weight[2 * e], e_weight[2 * e + 1]);
        pr.edges.push_back(ed);
    }
    pr.intrinsics = load_K(K);
    pr.damping = damping;
    return pr;
}

// The oracle handle: the reference's PatchGraph plus the relative-pose log
// its remove_frame writes (patch_graph.hpp:105).
struct GraphHandle {
    PatchGraph graph;
    RelativePoseLog log;
};
PatchGraph& G(void* g) { return static_cast<GraphHandle*>(g)->graph; }

// Frame grids of a [F][H][W][C] store, materialised per frame on first use.
struct FrameCache {
    const float* base0;
    const float* base1;
    int w0, h0, w1, h1, c;
    std::map<int, std::unique_ptr<FeaturePyramid>> pyr;
    const FeaturePyramid& at(int f) {
        auto& slot = pyr[f];
        if (!slot) {
            slot = std::make_unique<FeaturePyramid>();
            slot->level0 = load_grid(base0 + static_cast<size_t>(f) * w0 * h0 * c, w0, h0, c);
            slot->level1 = load_grid(base1 + static_cast<size_t>(f) * w1 * h1 * c, w1, h1, c);
        }
        return *slot;
    }
};

template <class F>
void parallel_edges(int n_edges, int threads, F&& body) {
    const int nt = threads > 0 ? threads : 1;
    std::vector<std::string> errs(nt);
    auto work = [&](int t) {
        try {
            for (int e = t; e < n_edges; e += nt) body(e);
        } catch (const std::exception& ex) {
            errs[t] = ex.what();
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (auto& s : errs)
        if (!s.empty()) throw std::invalid_argument(s);
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
int orc_backend_is_reference() { return 1; }

// ---- se3 (se3.cpp) ----
int orc_se3_exp(const double* xi, double* pose) { return guard([&] { store_pose(pvo::exp(load_xi(xi)), pose); }); }
int orc_se3_log(const double* pose, double* xi) {
    return guard([&] {
        const Tangent t = pvo::log(load_pose(pose));
        const Vec6 v = t.vector();
        for (int i = 0; i < 6; ++i) xi[i] = v(i);
    });
}
int orc_se3_compose(const double* a, const double* b, double* out) {
    return guard([&] { store_pose(compose(load_pose(a), load_pose(b)), out); });
}
int orc_se3_inverse(const double* a, double* out) { return guard([&] { store_pose(inverse(load_pose(a)), out); }); }
int orc_se3_retract(const double* a, const double* xi, double* out) {
    return guard([&] { store_pose(retract(load_pose(a), load_xi(xi)), out); });
}
int orc_se3_pose_distance(const double* a, const double* b, double* dist, double* angle) {
    return guard([&] { *dist = pose_distance(load_pose(a), load_pose(b), angle); });
}
int orc_se3_make_pose(const double* q_xyzw, const double* t, double* out) {
    return guard([&] {
        store_pose(Pose(Quat(q_xyzw[3], q_xyzw[0], q_xyzw[1], q_xyzw[2]), Vec3(t[0], t[1], t[2])), out);
    });
}

// ---- camera (camera.cpp) ----
int orc_patch_make(double cx, double cy, int width, double inverse_depth, double* x, double* y) {
    return guard([&] {
        const Patch p = Patch::make(0, Vec2(cx, cy), width, inverse_depth);
        std::memcpy(x, p.x.data(), sizeof(double) * p.x.size());
        std::memcpy(y, p.y.data(), sizeof(double) * p.y.size());
    });
}
int orc_reproject_patch(const double* pi, const double* pj, const double* K, int p, const double* x,
                        const double* y, double inv_depth, double* out_xy, int* behind) {
    return guard([&] {
        const PatchReprojection r =
            reproject_patch(load_pose(pi), load_pose(pj), load_K(K), load_patch(p, x, y, inv_depth, 0));
        for (size_t k = 0; k < r.points.size(); ++k) {
            out_xy[2 * k] = r.points[k].x();
            out_xy[2 * k + 1] = r.points[k].y();
        }
        *behind = r.behind_camera ? 1 : 0;
    });
}
// out: center(2), d_pose_i(12, row-major 2x6), d_pose_j(12), d_inverse_depth(2)
int orc_reprojection_jacobians(const double* pi, const double* pj, const double* K, int p, const double* x,
                               const double* y, double inv_depth, double* out, int* behind) {
    return guard([&] {
        const ReprojectionJacobians j =
            reprojection_jacobians(load_pose(pi), load_pose(pj), load_K(K), load_patch(p, x, y, inv_depth, 0));
        out[0] = j.center.x();
        out[1] = j.center.y();
        for (int r = 0; r < 2; ++r)
            for (int c = 0; c < 6; ++c) {
                out[2 + 6 * r + c] = j.d_pose_i(r, c);
                out[14 + 6 * r + c] = j.d_pose_j(r, c);
            }
        out[26] = j.d_inverse_depth.x();
        out[27] = j.d_inverse_depth.y();
        *behind = j.behind_camera ? 1 : 0;
    });
}

// ---- features / correlation (features.cpp, correlation.cpp) ----
int orc_sample_zero_padded(const float* grid, int w, int h, int c, double x, double y, int ch, double* out) {
    return guard([&] { *out = load_grid(grid, w, h, c).sample_zero_padded(x, y, ch); });
}
int orc_sample_cubic(const float* grid, int w, int h, int c, double x, double y, int ch, double* out) {
    return guard([&] { *out = load_grid(grid, w, h, c).sample_cubic(x, y, ch); });
}
int orc_correlate_at(const float* feature, int channels, const float* grid, int w, int h, double x, double y,
                     double* out) {
    return guard([&] { *out = correlate_at(feature, channels, load_grid(grid, w, h, channels), x, y); });
}
int orc_correlate_at_cubic(const float* feature, int channels, const float* grid, int w, int h, double x,
                           double y, double* out) {
    return guard([&] { *out = correlate_at_cubic(feature, channels, load_grid(grid, w, h, channels), x, y); });
}
static void store_grid(const CorrelationGrid& cg, float* out) {
    const size_t n = cg.values[0].size();
    std::memcpy(out, cg.values[0].data(), sizeof(float) * n);
    std::memcpy(out + n, cg.values[1].data(), sizeof(float) * n);
}
static std::vector<Vec2> load_coords(int pp, const double* coords) {
    std::vector<Vec2> r;
    r.reserve(pp);
    for (int k = 0; k < pp; ++k) r.emplace_back(coords[2 * k], coords[2 * k + 1]);
    return r;
}
int orc_correlate(int p, int channels, const float* feats0, const float* feats1, const float* lvl0, int w0,
                  int h0, const float* lvl1, int w1, int h1, const double* coords, float* out) {
    return guard([&] {
        FeaturePyramid pyr;
        pyr.level0 = load_grid(lvl0, w0, h0, channels);
        pyr.level1 = load_grid(lvl1, w1, h1, channels);
        store_grid(correlate(load_feats(p, channels, feats0, feats1), pyr, load_coords(p * p, coords)), out);
    });
}
// frames [F][H][W][C], patch_feats [P][2][p*p][C], coords [E][p*p][2] -> out [E][2][p*p][49]
int orc_correlate_batch(int n_edges, const int* e_patch, const int* e_frame, const double* coords, int p,
                        int channels, const float* patch_feats, const float* frames0, int w0, int h0,
                        const float* frames1, int w1, int h1, float* out, int threads) {
    return guard([&] {
        const size_t pp = static_cast<size_t>(p) * p;
        FrameCache cache{frames0, frames1, w0, h0, w1, h1, channels, {}};
        for (int e = 0; e < n_edges; ++e) cache.at(e_frame[e]);  // materialise before the threads read
        parallel_edges(n_edges, threads, [&](int e) {
            const float* g = patch_feats + static_cast<size_t>(e_patch[e]) * 2 * pp * channels;
            const CorrelationGrid cg = correlate(load_feats(p, channels, g, g + pp * channels), cache.at(e_frame[e]),
                                                 load_coords(static_cast<int>(pp), coords + e * pp * 2));
            store_grid(cg, out + static_cast<size_t>(e) * 2 * pp * kCorrSize * kCorrSize);
        });
    });
}
// CorrelationFlowProvider::measure per edge (flow_provider.cpp:211-287; the
// behind-camera branch of propose, :301-302).  flags: 1 flat, 2 out of range, 4 behind.
int orc_measure_batch(int n_edges, const int* e_patch, const int* e_frame, const double* centers,
                      const uint8_t* behind, int p, int channels, const float* patch_feats, const float* frames0,
                      int w0, int h0, const float* frames1, int w1, int h1, double* delta, double* weight,
                      uint8_t* flags, int threads) {
    return guard([&] {
        const size_t pp = static_cast<size_t>(p) * p;
        FrameCache cache{frames0, frames1, w0, h0, w1, h1, channels, {}};
        for (int e = 0; e < n_edges; ++e) cache.at(e_frame[e]);
        const CorrelationFlowProvider provider(channels == 75 ? 3 : 1);  // measure() ignores channels_
        parallel_edges(n_edges, threads, [&](int e) {
            CorrelationFlowProvider::Measurement m;
            uint8_t fl = 0;
            if (behind && behind[e]) {
                fl = 4;
            } else {
                const float* g = patch_feats + static_cast<size_t>(e_patch[e]) * 2 * pp * channels;
                m = provider.measure(load_feats(p, channels, g, g + pp * channels), cache.at(e_frame[e]),
                                     Vec2(centers[2 * e], centers[2 * e + 1]));
                fl = (m.flat ? 1 : 0) | (m.out_of_range ? 2 : 0);
            }
            delta[2 * e] = m.delta.x();
            delta[2 * e + 1] = m.delta.y();
            weight[2 * e] = m.weight.x();
            weight[2 * e + 1] = m.weight.y();
            flags[e] = fl;
        });
    });
}
int orc_extract_features(const float* image, int iw, int ih, int bc, float* level0, float* level1) {
    return guard([&] {
        Image img(iw, ih);
        std::memcpy(img.pixels.data(), image, sizeof(float) * img.pixels.size());
        const FeaturePyramid pyr = extract_features(img, bc);
        std::memcpy(level0, pyr.level0.data.data(), sizeof(float) * pyr.level0.data.size());
        std::memcpy(level1, pyr.level1.data.data(), sizeof(float) * pyr.level1.data.size());
    });
}
// crop_patch_features (features.cpp:216-235): out [n][2][9][C]
int orc_crop_patches(int n, const double* px, const double* py, const float* l0, int w0, int h0, const float* l1,
                     int w1, int h1, int C, float* out) {
    return guard([&] {
        FeaturePyramid pyr;
        pyr.level0 = load_grid(l0, w0, h0, C);
        pyr.level1 = load_grid(l1, w1, h1, C);
        for (int k = 0; k < n; ++k) {
            const PatchFeatures f = crop_patch_features(pyr, load_patch(3, px + 9 * k, py + 9 * k, 0.0, 0));
            float* o = out + static_cast<size_t>(k) * 2 * 9 * C;
            std::memcpy(o, f.level0.data(), sizeof(float) * 9 * C);
            std::memcpy(o + 9 * C, f.level1.data(), sizeof(float) * 9 * C);
        }
    });
}

// ---- patch graph (patch_graph.cpp) ----
void* orc_graph_create(const double* K, int w, int h, int p) {
    try {
        return new GraphHandle{PatchGraph(load_K(K), w, h, p), {}};
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void orc_graph_destroy(void* g) { delete static_cast<GraphHandle*>(g); }
int orc_graph_add_frame(void* g, double ts, const double* pose, int* out_index) {
    return guard([&] { *out_index = G(g).add_frame(ts, load_pose(pose)); });
}
int orc_graph_add_patches(void* g, int frame, int n, const double* centroids, const double* depths, int* out_ids) {
    return guard([&] {
        std::vector<Vec2> c;
        for (int i = 0; i < n; ++i) c.emplace_back(centroids[2 * i], centroids[2 * i + 1]);
        const auto ids = G(g).add_patches(frame, c, std::vector<double>(depths, depths + n));
        if (out_ids) std::memcpy(out_ids, ids.data(), sizeof(int) * ids.size());
    });
}
int orc_graph_connect(void* g, int radius, int* n_added) {
    return guard([&] { *n_added = static_cast<int>(G(g).connect(radius).size()); });
}
int orc_graph_remove_frame(void* g, int frame) {
    return guard([&] { G(g).remove_frame(frame, static_cast<GraphHandle*>(g)->log); });
}
int orc_graph_set_revision(void* g, int patch, int frame, const double* delta, const double* weight) {
    return guard([&] {
        FlowRevision r;
        r.delta = Vec2(delta[0], delta[1]);
        r.weight = Vec2(weight[0], weight[1]);
        G(g).set_revision({patch, frame}, r);
    });
}
int orc_graph_num_edges(void* g) { return static_cast<int>(G(g).edges().size()); }
int orc_graph_num_frames(void* g) { return static_cast<int>(G(g).frames().size()); }
int orc_graph_num_patches(void* g) { return static_cast<int>(G(g).patches().size()); }
int orc_graph_edges(void* g, int* kk, int* jj, double* rev, uint8_t* has_rev) {
    return guard([&] {
        size_t i = 0;
        for (const auto& [key, r] : G(g).edges()) {
            kk[i] = key.first;
            jj[i] = key.second;
            if (rev) {
                rev[4 * i] = r ? r->delta.x() : 0.0;
                rev[4 * i + 1] = r ? r->delta.y() : 0.0;
                rev[4 * i + 2] = r ? r->weight.x() : 0.0;
                rev[4 * i + 3] = r ? r->weight.y() : 0.0;
            }
            if (has_rev) has_rev[i] = r.has_value() ? 1 : 0;
            ++i;
        }
    });
}
int orc_graph_frames(void* g, int* indices, double* poses) {
    return guard([&] {
        size_t i = 0;
        for (const auto& [idx, node] : G(g).frames()) {
            indices[i] = idx;
            if (poses) store_pose(node.pose, poses + 7 * i);
            ++i;
        }
    });
}
int orc_graph_patches(void* g, int* ids, int* src, double* depth) {
    return guard([&] {
        size_t i = 0;
        for (const auto& [id, p] : G(g).patches()) {
            ids[i] = id;
            if (src) src[i] = p.source_frame;
            if (depth) depth[i] = p.inverse_depth;
            ++i;
        }
    });
}
int orc_graph_set_pose(void* g, int frame, const double* pose) {
    return guard([&] { G(g).set_pose(frame, load_pose(pose)); });
}
int orc_graph_set_inverse_depth(void* g, int patch, double d) {
    return guard([&] { G(g).set_inverse_depth(patch, d); });
}
// Pipeline::active_edges (pipeline.cpp:164-181): edges of patches sourced in
// the newest `window` frames, in key order.
int orc_graph_active_edges(void* g, int window, int* kk, int* jj, int* n) {
    return guard([&] {
        const PatchGraph& graph = G(g);
        std::vector<int> recent;
        for (auto it = graph.frames().rbegin(); it != graph.frames().rend() && static_cast<int>(recent.size()) < window;
             ++it)
            recent.push_back(it->first);
        const int oldest = recent.empty() ? 0 : recent.back();
        int i = 0;
        for (const auto& [key, revision] : graph.edges()) {
            if (graph.patch(key.first).source_frame < oldest) continue;
            if (kk) {
                kk[i] = key.first;
                jj[i] = key.second;
            }
            ++i;
        }
        *n = i;
    });
}
int orc_graph_build_target(void* g, int patch, int frame, double* out) {
    return guard([&] {
        const Vec2 t = build_target(G(g), {patch, frame});
        out[0] = t.x();
        out[1] = t.y();
    });
}

// The BAProblem optimize_window builds (bundle_adjust.cpp:231-307), restated
// over the reference graph's accessors + reproject_patch (sizes first with
// null arrays).  Edge targets use build_target's formula via the reference.
int orc_window_problem(void* g, int window, double damping, int* n_poses, int* n_patches, int* n_edges,
                       int* pose_frames, double* poses, uint8_t* fixed, int* patch_ids, int* patch_src,
                       double* patch_x, double* patch_y, double* depth, int* e_patch, int* e_pose,
                       double* e_target, double* e_weight) {
    return guard([&] {
        (void)damping;
        if (window < 1) throw std::invalid_argument("ba: window must be >= 1");
        const PatchGraph& graph = G(g);
        std::map<int, int> position;
        {
            int pos = 0;
            for (const auto& [index, node] : graph.frames()) position[index] = pos++;
        }
        const int num_frames = static_cast<int>(graph.frames().size());
        const int window_start = std::max(num_frames - window, 0);
        const int first_free = std::max(num_frames - window, 1);
        std::vector<int> ids;
        std::vector<std::pair<PatchGraph::EdgeKey, const FlowRevision*>> active;
        for (const auto& [patch_id, patch] : graph.patches()) {
            if (position.at(patch.source_frame) < window_start) continue;
            bool any = false;
            for (const auto& key : graph.edges_of_patch(patch_id)) {
                const auto& revision = graph.edges().at(key);
                if (!revision.has_value()) continue;
                active.emplace_back(key, &*revision);
                any = true;
            }
            if (any) ids.push_back(patch_id);
        }
        std::map<int, int> pose_index;
        for (int id : ids) pose_index.emplace(graph.patch(id).source_frame, 0);
        for (const auto& [key, r] : active) pose_index.emplace(key.second, 0);
        {
            int slot = 0;
            for (auto& [f, idx] : pose_index) idx = slot++;
        }
        std::map<int, int> patch_index;
        for (size_t k = 0; k < ids.size(); ++k) patch_index[ids[k]] = static_cast<int>(k);
        *n_poses = static_cast<int>(pose_index.size());
        *n_patches = static_cast<int>(ids.size());
        *n_edges = static_cast<int>(active.size());
        if (!pose_frames || active.empty()) return;
        const int pp = graph.patch_width() * graph.patch_width();
        for (const auto& [f, slot] : pose_index) {
            pose_frames[slot] = f;
            store_pose(graph.frame(f).pose, poses + 7 * slot);
            fixed[slot] = position.at(f) < first_free ? 1 : 0;
        }
        for (size_t k = 0; k < ids.size(); ++k) {
            const Patch& pt = graph.patch(ids[k]);
            patch_ids[k] = ids[k];
            patch_src[k] = pose_index.at(pt.source_frame);
            std::memcpy(patch_x + k * pp, pt.x.data(), sizeof(double) * pp);
            std::memcpy(patch_y + k * pp, pt.y.data(), sizeof(double) * pp);
            depth[k] = pt.inverse_depth;
        }
        const double margin = 2.0 * kMaxObservableMarginPx;
        for (size_t e = 0; e < active.size(); ++e) {
            const auto& [key, revision] = active[e];
            const Patch& pt = graph.patch(key.first);
            const PatchReprojection reproj = reproject_patch(graph.frame(pt.source_frame).pose,
                                                             graph.frame(key.second).pose, graph.intrinsics(), pt);
            const Vec2 center = reproj.center(pt);
            const bool observable = !reproj.behind_camera && center.x() > -margin && center.y() > -margin &&
                                    center.x() < graph.image_width() - 1 + margin &&
                                    center.y() < graph.image_height() - 1 + margin;
            e_patch[e] = patch_index.at(key.first);
            e_pose[e] = pose_index.at(key.second);
            const Vec2 target = center + revision->delta;
            e_target[2 * e] = target.x();
            e_target[2 * e + 1] = target.y();
            e_weight[2 * e] = observable ? revision->weight.x() : 0.0;
            e_weight[2 * e + 1] = observable ? revision->weight.y() : 0.0;
        }
    });
}

// optimize_window on the reference graph (mutates it; bundle_adjust.cpp:225-375).
int orc_optimize_window(void* g, int window, int iterations, int structure_only, double damping,
                        double* residual_norms, int* n_norms, int* num_edges) {
    return guard([&] {
        WindowOptions opt;
        opt.window = window;
        opt.iterations = iterations;
        opt.structure_only_iterations = structure_only;
        opt.damping = damping;
        const BASolution s = optimize_window(G(g), opt);
        *n_norms = static_cast<int>(s.residual_norms.size());
        for (size_t i = 0; i < s.residual_norms.size(); ++i) residual_norms[i] = s.residual_norms[i];
        *num_edges = s.num_edges;
    });
}

// optimize_window's loop (bundle_adjust.cpp:309-366) on a flat problem with
// frozen targets, every step the reference's gauss_newton_step.
int orc_ba_window(int n_poses, const double* poses, const uint8_t* fixed, int n_patches, int p, const int* src,
                  const double* px, const double* py, const double* depth, int n_edges, const int* e_patch,
                  const int* e_pose, const double* e_target, const double* e_weight, const double* K,
                  double damping, int iterations, int structure_only, double* out_poses, double* out_depth,
                  double* residual_norms, int* n_norms) {
    return guard([&] {
        BAProblem problem = load_problem(n_poses, poses, fixed, n_patches, p, src, px, py, depth, nullptr, n_edges,
                                         e_patch, e_pose, e_target, e_weight, K, damping);
        BASolution combined;
        combined.poses = problem.poses;
        for (const Patch& pt : problem.patches) combined.inverse_depths.push_back(pt.inverse_depth);
        for (int it = 0; it < structure_only; ++it) {
            BAProblem st = problem;
            st.pose_fixed.assign(st.poses.size(), true);
            const BASolution step = gauss_newton_step(st);
            for (size_t k = 0; k < problem.patches.size(); ++k) problem.patches[k].inverse_depth = step.inverse_depths[k];
            combined.inverse_depths = step.inverse_depths;
        }
        for (int it = 0; it < iterations; ++it) {
            BASolution step = gauss_newton_step(problem);
            if (step.residual_norms.back() > 1.5 * step.residual_norms.front() + 1e-9) {
                bool accepted = false;
                for (double extra = 1e3; extra <= 1e9; extra *= 1e3) {
                    problem.damping = damping * extra;
                    BASolution damped = gauss_newton_step(problem);
                    if (damped.residual_norms.back() <= 1.5 * damped.residual_norms.front() + 1e-9) {
                        step = damped;
                        accepted = true;
                        break;
                    }
                }
                problem.damping = damping;
                if (!accepted) {
                    if (combined.residual_norms.empty()) combined.residual_norms.push_back(step.residual_norms.front());
                    combined.residual_norms.push_back(step.residual_norms.front());
                    continue;
                }
            }
            if (combined.residual_norms.empty()) combined.residual_norms.push_back(step.residual_norms.front());
            combined.residual_norms.push_back(step.residual_norms.back());
            combined.poses = step.poses;
            combined.inverse_depths = step.inverse_depths;
            problem.poses = step.poses;
            for (size_t k = 0; k < problem.patches.size(); ++k) problem.patches[k].inverse_depth = step.inverse_depths[k];
        }
        for (int i = 0; i < n_poses; ++i) store_pose(combined.poses[i], out_poses + 7 * i);
        for (int k = 0; k < n_patches; ++k) out_depth[k] = combined.inverse_depths[k];
        *n_norms = static_cast<int>(combined.residual_norms.size());
        for (size_t i = 0; i < combined.residual_norms.size(); ++i) residual_norms[i] = combined.residual_norms[i];
    });
}

// gauss_newton_step (bundle_adjust.cpp:117-223) with NormalEquations capture.
int orc_gauss_newton_step(int n_poses, const double* poses, const uint8_t* fixed, int n_patches, int p,
                          const int* src, const double* px, const double* py, const double* depth,
                          const uint8_t* depth_free, int n_edges, const int* e_patch, const int* e_pose,
                          const double* e_target, const double* e_weight, const double* K, double damping,
                          double* out_poses, double* out_depth, double* residual_norms, double* debug_h,
                          double* debug_b, int* n_free_poses, int* n_free_depths) {
    return guard([&] {
        const BAProblem pr = load_problem(n_poses, poses, fixed, n_patches, p, src, px, py, depth, depth_free,
                                          n_edges, e_patch, e_pose, e_target, e_weight, K, damping);
        NormalEquations ne;
        const BASolution s = gauss_newton_step(pr, &ne);
        for (int i = 0; i < n_poses; ++i) store_pose(s.poses[i], out_poses + 7 * i);
        for (int k = 0; k < n_patches; ++k) out_depth[k] = s.inverse_depths[k];
        residual_norms[0] = s.residual_norms[0];
        residual_norms[1] = s.residual_norms[1];
        if (n_free_poses) *n_free_poses = ne.num_free_poses;
        if (n_free_depths) *n_free_depths = ne.num_free_depths;
        const Eigen::Index n = ne.h.rows();
        if (debug_h)
            for (Eigen::Index r = 0; r < n; ++r)
                for (Eigen::Index c = 0; c < n; ++c) debug_h[r * n + c] = ne.h(r, c);
        if (debug_b)
            for (Eigen::Index r = 0; r < n; ++r) debug_b[r] = ne.b(r);
    });
}

// schur_solve (bundle_adjust.cpp:62-94) on dense row-major inputs.
int orc_schur_solve(int np, int nd, const double* hpp, const double* hpd, const double* hdd, const double* bp,
                    const double* bd, double* dp, double* dd) {
    return guard([&] {
        Eigen::MatrixXd a(np, np), b(np, nd);
        Eigen::VectorXd d(nd), vp(np), vd(nd);
        for (int r = 0; r < np; ++r) {
            for (int c = 0; c < np; ++c) a(r, c) = hpp[r * np + c];
            for (int c = 0; c < nd; ++c) b(r, c) = hpd[r * nd + c];
            vp(r) = bp[r];
        }
        for (int k = 0; k < nd; ++k) {
            d(k) = hdd[k];
            vd(k) = bd[k];
        }
        const SchurResult res = schur_solve(a, b, d, vp, vd);
        for (int r = 0; r < np; ++r) dp[r] = res.pose_delta(r);
        for (int k = 0; k < nd; ++k) dd[k] = res.depth_delta(k);
    });
}

// Eigen::LDLT solve as the reference calls it (bundle_adjust.cpp:76).
int orc_ldlt_solve(int n, const double* a, const double* rhs, double* x, int* ok) {
    return guard([&] {
        Eigen::MatrixXd m(n, n);
        Eigen::VectorXd b(n);
        for (int r = 0; r < n; ++r) {
            for (int c = 0; c < n; ++c) m(r, c) = a[r * n + c];
            b(r) = rhs[r];
        }
        const Eigen::LDLT<Eigen::MatrixXd> ldlt(m);
        *ok = ldlt.info() == Eigen::Success ? 1 : 0;
        const Eigen::VectorXd s = ldlt.solve(b);
        for (int r = 0; r < n; ++r) x[r] = s(r);
    });
}

// ---- timing entries for bench.py's CPU legs (the reference's own code) ----
// Per-iteration correlation work of the reference pipeline over a flat window:
// for every edge reproject_patch (camera.cpp:47-71) then correlate
// (correlation.cpp:37-71), edges split over `threads` host threads (the
// reference itself is single-threaded; edges are independent).  Patches,
// PatchFeatures and FeaturePyramids are staged before the clock starts, as the
// pipeline keeps them resident (flow_provider.hpp:108-112).
int orc_bench_corr(int n_poses, const double* poses, int n_patches, int p, const int* src, const double* px,
                   const double* py, const double* depth, int n_edges, const int* e_patch, const int* e_pose,
                   const int* e_frame, const double* K, int channels, const float* patch_feats,
                   const float* frames0, int w0, int h0, const float* frames1, int w1, int h1, int threads,
                   double* seconds) {
    return guard([&] {
        std::vector<Pose> P;
        for (int i = 0; i < n_poses; ++i) P.push_back(load_pose(poses + 7 * i));
        std::vector<Patch> pt;
        std::vector<PatchFeatures> pf;
        const size_t pp = static_cast<size_t>(p) * p;
        for (int k = 0; k < n_patches; ++k) {
            pt.push_back(load_patch(p, px + k * p * p, py + k * p * p, depth[k], src[k]));
            const float* g = patch_feats + static_cast<size_t>(k) * 2 * pp * channels;
            pf.push_back(load_feats(p, channels, g, g + pp * channels));
        }
        const Intrinsics Kc = load_K(K);
        FrameCache cache{frames0, frames1, w0, h0, w1, h1, channels, {}};
        for (int e = 0; e < n_edges; ++e) cache.at(e_frame[e]);
        std::vector<CorrelationGrid> out(static_cast<size_t>(n_edges));
        const int nt = threads > 0 ? threads : 1;
        const auto t0 = std::chrono::steady_clock::now();
        auto work = [&](int t) {
            for (int e = t; e < n_edges; e += nt) {
                const Patch& patch = pt[e_patch[e]];
                const PatchReprojection r = reproject_patch(P[patch.source_frame], P[e_pose[e]], Kc, patch);
                out[e] = correlate(pf[e_patch[e]], cache.at(e_frame[e]), r.points);
            }
        };
        std::vector<std::thread> pool;
        for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
        work(0);
        for (auto& th : pool) th.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}
// optimize_window (bundle_adjust.cpp:225-375) on a copy of the graph; *seconds
// = the call alone (the copy is made before the clock starts).
int orc_bench_optimize_window(void* g, int window, int iterations, double damping, double* seconds) {
    return guard([&] {
        PatchGraph copy = G(g);
        WindowOptions opt;
        opt.window = window;
        opt.iterations = iterations;
        opt.damping = damping;
        const auto t0 = std::chrono::steady_clock::now();
        optimize_window(copy, opt);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

}  // extern "C"

