// pvo_b200.hpp — header-only C++ layer over include/pvo_capi.h.
//
// Restores the reference's C++ conventions on top of the C-ABI: RAII handles,
// std::vector-owned outputs returned by value, and the reference's exception
// types (std::invalid_argument, pvo::DegenerateProblem : std::runtime_error,
// std::domain_error, std::out_of_range — bundle_adjust.hpp:54-56, se3.cpp:58-60)
// rethrown from the status codes.  Poses are 7 doubles in Eigen coefficient
// order (qx, qy, qz, qw, tx, ty, tz); INTEGRATION.md shows the Eigen-typed
// shims a maintainer adds to proj/src/*.cpp on top of this.
#pragma once

#include <array>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../pvo_capi.h"

namespace pvo {
namespace b200 {

// pvo::DegenerateProblem of bundle_adjust.hpp:54-56.
struct DegenerateProblem : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int status) {
    if (status == PVO_OK) return;
    const std::string msg = pvo_last_error();
    switch (status) {
        case PVO_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case PVO_DEGENERATE: throw DegenerateProblem(msg);
        case PVO_DOMAIN_ERROR: throw std::domain_error(msg);
        case PVO_OUT_OF_RANGE: throw std::out_of_range(msg);
        case PVO_UNSUPPORTED: throw std::logic_error("unsupported: " + msg);
        default: throw CudaError(msg);
    }
}

using Pose = std::array<double, 7>;
using Tangent = std::array<double, 6>;

// ---- SE(3) (se3.hpp:63-77) ----
inline Pose exp(const Tangent& xi) {
    Pose p;
    check(pvo_se3_exp(xi.data(), p.data()));
    return p;
}
inline Tangent log(const Pose& p) {
    Tangent xi;
    check(pvo_se3_log(p.data(), xi.data()));
    return xi;
}
inline Pose compose(const Pose& a, const Pose& b) {
    Pose p;
    check(pvo_se3_compose(a.data(), b.data(), p.data()));
    return p;
}
inline Pose inverse(const Pose& a) {
    Pose p;
    check(pvo_se3_inverse(a.data(), p.data()));
    return p;
}
inline Pose retract(const Pose& a, const Tangent& xi) {
    Pose p;
    check(pvo_se3_retract(a.data(), xi.data(), p.data()));
    return p;
}

// ---- device context (one per host thread) ----
class Context {
  public:
    explicit Context(int device = 0) { check(pvo_ctx_create(device, &ctx_)); }
    ~Context() {
        if (ctx_) pvo_ctx_destroy(ctx_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    pvo_ctx* get() const { return ctx_; }

  private:
    pvo_ctx* ctx_ = nullptr;
};

// ---- correlate (correlation.hpp:33-34): out [2][p*p][7][7] ----
inline std::array<std::vector<float>, 2> correlate(Context& ctx, int p, int channels, const std::vector<float>& feats0,
                                                   const std::vector<float>& feats1, const std::vector<float>& level0,
                                                   int w0, int h0, const std::vector<float>& level1, int w1, int h1,
                                                   const std::vector<double>& coords) {
    if (static_cast<int>(coords.size()) != 2 * p * p) throw std::invalid_argument("correlate: reprojection size mismatch");
    std::vector<float> out(static_cast<size_t>(2) * p * p * 49);
    check(pvo_correlate(ctx.get(), p, channels, feats0.data(), feats1.data(), level0.data(), w0, h0, level1.data(), w1,
                        h1, coords.data(), out.data()));
    std::array<std::vector<float>, 2> grid;
    grid[0].assign(out.begin(), out.begin() + p * p * 49);
    grid[1].assign(out.begin() + p * p * 49, out.end());
    return grid;
}

// ---- schur_solve (bundle_adjust.hpp:89-91), row-major dense inputs ----
inline std::pair<std::vector<double>, std::vector<double>> schur_solve(Context& ctx, int np, int nd,
                                                                       const std::vector<double>& h_pp,
                                                                       const std::vector<double>& h_pd,
                                                                       const std::vector<double>& h_dd,
                                                                       const std::vector<double>& b_p,
                                                                       const std::vector<double>& b_d) {
    std::vector<double> dp(np), dd(nd);
    check(pvo_schur_solve(ctx.get(), np, nd, h_pp.data(), h_pd.data(), h_dd.data(), b_p.data(), b_d.data(), dp.data(),
                          dd.data()));
    return {std::move(dp), std::move(dd)};
}

// ---- PatchGraph (patch_graph.hpp:66-136) ----
class PatchGraph {
  public:
    PatchGraph(const std::array<double, 4>& K, int w, int h, int patch_width = 3) {
        check(pvo_graph_create(K.data(), w, h, patch_width, &g_));
    }
    ~PatchGraph() {
        if (g_) pvo_graph_destroy(g_);
    }
    PatchGraph(const PatchGraph&) = delete;
    PatchGraph& operator=(const PatchGraph&) = delete;

    int add_frame(double timestamp, const Pose& pose) {
        int idx = -1;
        check(pvo_graph_add_frame(g_, timestamp, pose.data(), &idx));
        return idx;
    }
    std::vector<int> add_patches(int frame, const std::vector<double>& centroids_xy,
                                 const std::vector<double>& inverse_depths) {
        if (centroids_xy.size() != 2 * inverse_depths.size()) {
            throw std::invalid_argument("patch graph: centroid/depth count mismatch");
        }
        std::vector<int> ids(inverse_depths.size());
        check(pvo_graph_add_patches(g_, frame, static_cast<int>(inverse_depths.size()), centroids_xy.data(),
                                    inverse_depths.data(), ids.data()));
        return ids;
    }
    int connect(int radius) {
        int n = 0;
        check(pvo_graph_connect(g_, radius, &n));
        return n;
    }
    void remove_frame(int frame) { check(pvo_graph_remove_frame(g_, frame)); }
    void set_revision(int patch_id, int frame, const std::array<double, 2>& delta,
                      const std::array<double, 2>& weight) {
        check(pvo_graph_set_revision(g_, patch_id, frame, delta.data(), weight.data()));
    }
    std::array<double, 2> build_target(int patch_id, int frame) const {
        std::array<double, 2> t;
        check(pvo_graph_build_target(g_, patch_id, frame, t.data()));
        return t;
    }
    // Edges in reference key order (patch id, frame index).
    std::vector<std::pair<int, int>> edges() const {
        const int n = pvo_graph_num_edges(g_);
        std::vector<int> kk(n), jj(n);
        check(pvo_graph_edges(g_, kk.data(), jj.data(), nullptr, nullptr));
        std::vector<std::pair<int, int>> out(n);
        for (int i = 0; i < n; ++i) out[i] = {kk[i], jj[i]};
        return out;
    }
    pvo_graph* get() const { return g_; }

  private:
    pvo_graph* g_ = nullptr;
};

struct WindowResult {
    std::vector<double> residual_norms;
    int num_edges = 0;
};

// optimize_window (bundle_adjust.hpp:111): mutates the graph.
inline WindowResult optimize_window(Context& ctx, PatchGraph& graph, int window = 10, int iterations = 2,
                                    int structure_only_iterations = 0, double damping = 1e-4) {
    WindowResult r;
    r.residual_norms.resize(iterations + 2);
    int n = 0;
    check(pvo_optimize_window(ctx.get(), graph.get(), window, iterations, structure_only_iterations, damping,
                              r.residual_norms.data(), &n, &r.num_edges));
    r.residual_norms.resize(n);
    return r;
}

// CorrelationFlowProvider::measure (flow_provider.cpp:209-287) per edge against the
// context's frame store.  flags: 1 flat, 2 out of range, 4 behind the camera.
struct Measurements {
    std::vector<double> delta, weight;  // [E][2]
    std::vector<uint8_t> flags;         // [E]
};
inline Measurements measure_batch(Context& ctx, const std::vector<int>& e_patch, const std::vector<int>& e_slot,
                                  const std::vector<double>& centers, const std::vector<uint8_t>& behind,
                                  int n_patches, const std::vector<float>& patch_feats) {
    const int E = static_cast<int>(e_patch.size());
    Measurements m;
    m.delta.resize(2 * (size_t)E);
    m.weight.resize(2 * (size_t)E);
    m.flags.resize(E);
    check(pvo_measure_batch(ctx.get(), E, n_patches, 3, e_patch.data(), e_slot.data(), centers.data(),
                            behind.empty() ? nullptr : behind.data(), patch_feats.data(), m.delta.data(),
                            m.weight.data(), m.flags.data()));
    return m;
}

// A batch of independent windows on one device (config 5): concatenated arrays
// with pose / patch / edge offsets, window-local indices (pvo_batch_load).
class Batch {
  public:
    explicit Batch(Context& ctx) : ctx_(ctx) {}
    void load(int n_windows, const int* pose_off, const int* patch_off, const int* edge_off, const double* poses,
              const uint8_t* fixed, const int* pose_slot, const int* src, const double* px, const double* py,
              const double* depth, const float* patch_feats, const int* e_patch, const int* e_pose,
              const double* e_delta, const double* e_weight, const double K[4], int image_w, int image_h) {
        check(pvo_batch_load(ctx_.get(), n_windows, pose_off, patch_off, edge_off, poses, fixed, pose_slot, 3, src, px,
                             py, depth, patch_feats, e_patch, e_pose, e_delta, e_weight, K, image_w, image_h));
    }
    void reset() { check(pvo_batch_reset(ctx_.get())); }
    void iteration(int iterations = 2, double damping = 1e-4) {
        check(pvo_batch_iteration(ctx_.get(), iterations, damping, nullptr, PVO_DEVICE));
    }
    // poses [N][7], depths [P], residual norms [n_windows][pvo_batch_norm_stride()], counts [n_windows]
    void read(double* poses, double* depth, double* norms, int* n_norms) {
        check(pvo_batch_read(ctx_.get(), poses, depth, norms, n_norms));
    }

  private:
    Context& ctx_;
};

}  // namespace b200
}  // namespace pvo
