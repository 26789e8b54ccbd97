// dropin_bundle_adjust.cpp — the operators of proj/include/pvo/bundle_adjust.hpp
// on the GPU.
//
// Replaces proj/src/bundle_adjust.cpp.  Host work is limited to what the
// reference's API shape forces: validating and flattening BAProblem / the
// PatchGraph window into the C-ABI's arrays, and rebuilding the returned
// Eigen / Pose objects.  Every number comes from the sm_100a kernels:
//   gauss_newton_step (bundle_adjust.cpp:117-223) -> pvo_gauss_newton_step
//     (assembly + Schur + LDL^T + retraction + both WRMS norms on the device;
//      NormalEquations captured on the device when asked for);
//   schur_solve (:62-94)                         -> pvo_schur_solve;
//   optimize_window (:225-375)                   -> window flatten here
//     (:231-285, the reference's orders) + pvo_ba_window with device-frozen
//     targets (:288-307), structure-only steps and the divergence guard
//     (:309-366); results written back into the graph (:368-373).
// build_target (:47-60) reprojects through the GPU reproject_patch.
#include <map>
#include <ostream>
#include <stdexcept>

#include "dropin_runtime.hpp"
#include "pvo/bundle_adjust.hpp"

namespace pvo {

namespace {

[[noreturn]] void throw_degenerate(const std::string& msg) { throw DegenerateProblem(msg); }
void check(int status) { dropin::check(status, &throw_degenerate); }

// Patches of one problem share a width (the flat C-ABI arrays are [P][p*p]).
int common_width(const std::vector<Patch>& patches) {
    int p = patches.empty() ? 3 : patches[0].width;
    for (const Patch& patch : patches)
        if (patch.width != p) throw std::logic_error("pvo_b200: unsupported shape: mixed patch widths in one problem");
    return p;
}

struct FlatPatches {
    int p = 3;
    std::vector<int> src;
    std::vector<double> x, y, depth;
    void add(const Patch& patch, int source_slot) {
        src.push_back(source_slot);
        x.insert(x.end(), patch.x.begin(), patch.x.end());
        y.insert(y.end(), patch.y.begin(), patch.y.end());
        depth.push_back(patch.inverse_depth);
    }
};

Eigen::MatrixXd from_row_major(const double* v, int rows, int cols) {
    Eigen::MatrixXd m(rows, cols);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) m(r, c) = v[(size_t)r * cols + c];
    return m;
}

}  // namespace

void BAProblem::validate() const {
    // bundle_adjust.cpp:11-36, same checks and messages
    if (poses.size() != pose_fixed.size()) throw std::invalid_argument("ba: pose/fixed-mask size mismatch");
    if (!depth_free.empty() && depth_free.size() != patches.size())
        throw std::invalid_argument("ba: depth mask size mismatch");
    const int n_patches = (int)patches.size(), n_poses = (int)poses.size();
    for (const BAEdge& e : edges) {
        if (e.patch_id < 0 || e.patch_id >= n_patches || e.target_pose < 0 || e.target_pose >= n_poses)
            throw std::invalid_argument("ba: edge references an unknown patch or pose");
        if (!e.target_point.allFinite()) throw std::invalid_argument("ba: non-finite edge target");
        const bool in_range = e.weight.x() >= 0 && e.weight.x() < 1 && e.weight.y() >= 0 && e.weight.y() < 1;
        if (!in_range) throw std::invalid_argument("ba: edge weights must lie in [0, 1)");
    }
    for (const Patch& patch : patches)
        if (patch.source_frame < 0 || patch.source_frame >= n_poses)
            throw std::invalid_argument("ba: patch source pose out of range");
}

void NormalEquations::dump(std::ostream& out) const {
    // text form: "rows free_poses free_depths", then one row of h per line followed by b(row)
    out << h.rows() << " " << num_free_poses << " " << num_free_depths << "\n";
    out.precision(17);
    for (Eigen::Index r = 0; r < h.rows(); ++r) {
        for (Eigen::Index c = 0; c < h.cols(); ++c) out << h(r, c) << " ";
        out << b(r) << "\n";
    }
}

Vec2 build_target(const PatchGraph& graph, const PatchGraph::EdgeKey& edge) {
    const auto it = graph.edges().find(edge);
    if (it == graph.edges().end()) throw std::invalid_argument("build_target: no such edge");
    if (!it->second) throw std::invalid_argument("build_target: edge has no revision");
    const Patch& patch = graph.patch(edge.first);
    const PatchReprojection reproj = reproject_patch(graph.frame(patch.source_frame).pose,
                                                     graph.frame(edge.second).pose, graph.intrinsics(), patch);
    return reproj.center(patch) + it->second->delta;
}

SchurResult schur_solve(const Eigen::MatrixXd& h_pose_pose, const Eigen::MatrixXd& h_pose_depth,
                        const Eigen::VectorXd& h_depth_depth, const Eigen::VectorXd& b_pose,
                        const Eigen::VectorXd& b_depth) {
    const int np = (int)h_pose_pose.rows(), nd = (int)h_depth_depth.size();
    if (h_pose_pose.cols() != np || b_pose.size() != np || b_depth.size() != nd ||
        (np > 0 && (h_pose_depth.rows() != np || h_pose_depth.cols() != nd)))
        throw std::invalid_argument("schur: block sizes do not match");
    std::vector<double> hpp((size_t)np * np), hpd((size_t)np * nd), hdd(nd), bp(np), bd(nd);
    for (int r = 0; r < np; ++r) {
        for (int c = 0; c < np; ++c) hpp[(size_t)r * np + c] = h_pose_pose(r, c);
        for (int c = 0; c < nd; ++c) hpd[(size_t)r * nd + c] = h_pose_depth(r, c);
        bp[r] = b_pose(r);
    }
    for (int k = 0; k < nd; ++k) {
        hdd[k] = h_depth_depth(k);
        bd[k] = b_depth(k);
    }
    std::vector<double> dp(np), dd(nd);
    check(pvo_schur_solve(dropin::context(), np, nd, hpp.data(), hpd.data(), hdd.data(), bp.data(), bd.data(),
                          dp.data(), dd.data()));
    SchurResult result;
    result.pose_delta.resize(np);
    result.depth_delta.resize(nd);
    for (int r = 0; r < np; ++r) result.pose_delta(r) = dp[r];
    for (int k = 0; k < nd; ++k) result.depth_delta(k) = dd[k];
    return result;
}

BASolution gauss_newton_step(const BAProblem& problem, NormalEquations* debug) {
    problem.validate();
    if (problem.edges.empty()) throw std::invalid_argument("ba: need at least one edge");
    const int n_poses = (int)problem.poses.size(), n_patches = (int)problem.patches.size();
    const int n_edges = (int)problem.edges.size();

    std::vector<double> poses(7 * (size_t)n_poses);
    std::vector<uint8_t> fixed(n_poses), dfree(n_patches, 1);
    int free_poses = 0, free_depths = 0;
    for (int i = 0; i < n_poses; ++i) {
        dropin::flat_into(problem.poses[i], &poses[7 * (size_t)i]);
        fixed[i] = problem.pose_fixed[i] ? 1 : 0;
        free_poses += fixed[i] ? 0 : 1;
    }
    for (int k = 0; k < n_patches; ++k) {
        if (!problem.depth_free.empty()) dfree[k] = problem.depth_free[k] ? 1 : 0;
        free_depths += dfree[k];
    }
    FlatPatches fp;
    fp.p = common_width(problem.patches);
    for (const Patch& patch : problem.patches) fp.add(patch, patch.source_frame);
    std::vector<int> e_patch(n_edges), e_pose(n_edges);
    std::vector<double> target(2 * (size_t)n_edges), weight(2 * (size_t)n_edges);
    for (int e = 0; e < n_edges; ++e) {
        const BAEdge& edge = problem.edges[e];
        e_patch[e] = edge.patch_id;
        e_pose[e] = edge.target_pose;
        target[2 * e] = edge.target_point.x();
        target[2 * e + 1] = edge.target_point.y();
        weight[2 * e] = edge.weight.x();
        weight[2 * e + 1] = edge.weight.y();
    }
    const double K[4] = {problem.intrinsics.fx, problem.intrinsics.fy, problem.intrinsics.cx, problem.intrinsics.cy};
    const int n = 6 * free_poses + free_depths;
    std::vector<double> out_poses(poses.size()), out_depth(n_patches), norms(2);
    std::vector<double> dh(debug ? (size_t)n * n : 0), db(debug ? n : 0);
    int nfp = 0, nfd = 0;
    check(pvo_gauss_newton_step(dropin::context(), n_poses, poses.data(), fixed.data(), n_patches, fp.p, fp.src.data(),
                                fp.x.data(), fp.y.data(), fp.depth.data(), dfree.data(), n_edges, e_patch.data(),
                                e_pose.data(), target.data(), weight.data(), K, problem.damping, out_poses.data(),
                                out_depth.data(), norms.data(), debug ? dh.data() : nullptr,
                                debug ? db.data() : nullptr, &nfp, &nfd));
    if (debug) {
        debug->h = from_row_major(dh.data(), n, n);
        debug->b.resize(n);
        for (int r = 0; r < n; ++r) debug->b(r) = db[r];
        debug->num_free_poses = nfp;
        debug->num_free_depths = nfd;
    }
    BASolution solution;
    solution.num_edges = n_edges;
    solution.residual_norms = {norms[0], norms[1]};
    solution.poses.reserve(n_poses);
    for (int i = 0; i < n_poses; ++i)
        solution.poses.push_back(dropin::unflat(&out_poses[7 * (size_t)i], &problem.poses[i]));
    solution.inverse_depths = out_depth;
    return solution;
}

BASolution optimize_window(PatchGraph& graph, const WindowOptions& options) {
    if (options.window < 1) throw std::invalid_argument("ba: window must be >= 1");
    if (options.iterations < 0 || options.structure_only_iterations < 0)
        throw std::invalid_argument("ba: negative iteration count");

    // ---- the window problem, in the reference's orders (bundle_adjust.cpp:231-285) ----
    const auto& frames = graph.frames();
    std::map<int, int> position;  // keyframe order of the surviving frames
    for (const auto& entry : frames) position.emplace(entry.first, (int)position.size());
    const int n_frames = (int)frames.size();
    const int window_start = std::max(n_frames - options.window, 0);
    const int first_free = std::max(n_frames - options.window, 1);

    std::vector<int> patch_ids;  // included patches, ascending id
    std::vector<std::pair<PatchGraph::EdgeKey, const FlowRevision*>> active;  // revised edges, key order
    for (const auto& [patch_id, patch] : graph.patches()) {
        if (position.at(patch.source_frame) < window_start) continue;
        const size_t before = active.size();
        for (const auto& key : graph.edges_of_patch(patch_id)) {
            const auto& revision = graph.edges().at(key);
            if (revision) active.emplace_back(key, &*revision);
        }
        if (active.size() > before) patch_ids.push_back(patch_id);
    }
    if (active.empty()) return BASolution();

    std::map<int, int> pose_slot;  // frames referenced, ascending index -> slot
    for (int id : patch_ids) pose_slot.emplace(graph.patch(id).source_frame, 0);
    for (const auto& a : active) pose_slot.emplace(a.first.second, 0);
    {
        int slot = 0;
        for (auto& entry : pose_slot) entry.second = slot++;
    }
    const int n_poses = (int)pose_slot.size(), n_patches = (int)patch_ids.size(), n_edges = (int)active.size();
    std::vector<const Pose*> original(n_poses);
    std::vector<double> poses(7 * (size_t)n_poses);
    std::vector<uint8_t> fixed(n_poses);
    for (const auto& [frame, slot] : pose_slot) {
        original[slot] = &graph.frame(frame).pose;
        dropin::flat_into(*original[slot], &poses[7 * (size_t)slot]);
        fixed[slot] = position.at(frame) < first_free ? 1 : 0;
    }
    std::map<int, int> patch_slot;
    std::vector<Patch> included;
    FlatPatches fp;
    for (int id : patch_ids) {
        patch_slot.emplace(id, (int)patch_slot.size());
        included.push_back(graph.patch(id));
    }
    fp.p = common_width(included);
    for (const Patch& patch : included) fp.add(patch, pose_slot.at(patch.source_frame));
    std::vector<int> e_patch(n_edges), e_pose(n_edges);
    std::vector<double> delta(2 * (size_t)n_edges), weight(2 * (size_t)n_edges);
    for (int e = 0; e < n_edges; ++e) {
        const auto& [key, revision] = active[e];
        e_patch[e] = patch_slot.at(key.first);
        e_pose[e] = pose_slot.at(key.second);
        delta[2 * e] = revision->delta.x();
        delta[2 * e + 1] = revision->delta.y();
        weight[2 * e] = revision->weight.x();
        weight[2 * e + 1] = revision->weight.y();
    }

    // ---- frozen targets + iterations on the device ----
    const Intrinsics& Ki = graph.intrinsics();
    const double K[4] = {Ki.fx, Ki.fy, Ki.cx, Ki.cy};
    std::vector<double> out_poses(poses.size()), out_depth(n_patches);
    std::vector<double> norms((size_t)options.iterations + options.structure_only_iterations + 2);
    int n_norms = 0;
    check(pvo_ba_window(dropin::context(), n_poses, poses.data(), fixed.data(), n_patches, fp.p, fp.src.data(),
                        fp.x.data(), fp.y.data(), fp.depth.data(), n_edges, e_patch.data(), e_pose.data(),
                        delta.data(), weight.data(), K, graph.image_width(), graph.image_height(),
                        /*freeze_targets=*/1, options.damping, options.iterations, options.structure_only_iterations,
                        out_poses.data(), out_depth.data(), norms.data(), &n_norms));

    // ---- results (bundle_adjust.cpp:368-373) ----
    BASolution combined;
    combined.num_edges = n_edges;
    combined.residual_norms.assign(norms.begin(), norms.begin() + n_norms);
    combined.inverse_depths = out_depth;
    combined.poses.reserve(n_poses);
    for (int s = 0; s < n_poses; ++s)
        combined.poses.push_back(dropin::unflat(&out_poses[7 * (size_t)s], original[s]));
    for (const auto& [frame, slot] : pose_slot)
        if (!fixed[slot]) graph.set_pose(frame, combined.poses[slot]);
    for (const auto& [id, slot] : patch_slot) graph.set_inverse_depth(id, combined.inverse_depths[slot]);
    return combined;
}

}  // namespace pvo
