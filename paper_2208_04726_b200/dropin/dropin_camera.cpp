// dropin_camera.cpp — the operators of proj/include/pvo/camera.hpp on the GPU.
//
// Replaces proj/src/camera.cpp.  Intrinsics / Patch construction stay host
// data-structure code (camera.cpp:8-45 semantics: same validation, same
// row-major grid arithmetic); reproject_patch (camera.cpp:47-71) and
// reprojection_jacobians (camera.cpp:73-108) run the FP64 sm_100a kernels
// behind pvo_reproject_patches / pvo_reprojection_jacobians (bitwise-equal
// pose shortcut included).  Each call is one small launch + read-back; the
// batched C-ABI entries are the throughput path.
#include <stdexcept>

#include "dropin_runtime.hpp"
#include "pvo/camera.hpp"

namespace pvo {

Intrinsics::Intrinsics(double fx_, double fy_, double cx_, double cy_) : fx(fx_), fy(fy_), cx(cx_), cy(cy_) {
    // the comparison form keeps the reference's NaN behaviour (camera.cpp:10)
    if (fx <= 0 || fy <= 0) throw std::invalid_argument("intrinsics: focal lengths must be positive");
}

Patch Patch::make(int source_frame, const Vec2& centroid, int width, double inverse_depth) {
    if (width < 1) throw std::invalid_argument("patch: width must be >= 1");
    if (inverse_depth < 0) throw std::invalid_argument("patch: inverse depth must be >= 0");
    Patch out;
    out.source_frame = source_frame;
    out.width = width;
    out.inverse_depth = inverse_depth;
    const int n = width * width;
    const double half = 0.5 * (width - 1);
    out.x.resize(n);
    out.y.resize(n);
    for (int k = 0; k < n; ++k) {  // pixel k = (row k / p, col k % p), row-major
        out.x[k] = centroid.x() + (k % width) - half;
        out.y[k] = centroid.y() + (k / width) - half;
    }
    return out;
}

Vec2 Patch::center() const {
    const int n = size();
    if (width % 2 == 1) return Vec2(x[n / 2], y[n / 2]);
    double sx = 0, sy = 0;  // even widths: the mean, summed in pixel order
    for (int k = 0; k < n; ++k) {
        sx += x[k];
        sy += y[k];
    }
    return Vec2(sx / n, sy / n);
}

PatchReprojection reproject_patch(const Pose& pose_i, const Pose& pose_j, const Intrinsics& K, const Patch& patch) {
    const int n = patch.size();
    const auto pi = dropin::flat(pose_i), pj = dropin::flat(pose_j);
    const double k4[4] = {K.fx, K.fy, K.cx, K.cy};
    std::vector<double> xy(2 * (size_t)n);
    uint8_t behind = 0;
    PatchReprojection out;
    if (n > 0) {
        dropin::check(pvo_reproject_patches(dropin::context(), 1, patch.width, pi.data(), pj.data(), k4,
                                            patch.x.data(), patch.y.data(), &patch.inverse_depth, xy.data(), &behind));
    }
    out.points.reserve(n);
    for (int k = 0; k < n; ++k) out.points.emplace_back(xy[2 * k], xy[2 * k + 1]);
    out.behind_camera = behind != 0;
    return out;
}

ReprojectionJacobians reprojection_jacobians(const Pose& pose_i, const Pose& pose_j, const Intrinsics& K,
                                             const Patch& patch) {
    const auto pi = dropin::flat(pose_i), pj = dropin::flat(pose_j);
    const double k4[4] = {K.fx, K.fy, K.cx, K.cy};
    double r[28];
    uint8_t behind = 0;
    dropin::check(pvo_reprojection_jacobians(dropin::context(), 1, patch.width, pi.data(), pj.data(), k4,
                                             patch.x.data(), patch.y.data(), &patch.inverse_depth, r, &behind));
    ReprojectionJacobians jac;
    jac.center = Vec2(r[0], r[1]);
    for (int row = 0; row < 2; ++row)
        for (int col = 0; col < 6; ++col) {
            jac.d_pose_i(row, col) = r[2 + 6 * row + col];
            jac.d_pose_j(row, col) = r[14 + 6 * row + col];
        }
    jac.d_inverse_depth = Vec2(r[26], r[27]);
    jac.behind_camera = behind != 0;
    return jac;
}

}  // namespace pvo
