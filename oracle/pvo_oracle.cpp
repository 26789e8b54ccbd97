// ============================================================================
// pvo_oracle.cpp — CPU RESTATEMENT OF THE REFERENCE HOT PATH.  TEST
// INFRASTRUCTURE ONLY.
//
// This file is the checker, never the product: only tests/, the graft smoke
// check and bench.py's cpu-baseline leg may load the library built from it
// (oracle/liboracle_pvo.so).  The product path (paper_2208_04726_b200/)
// never links or calls it.
//
// It restates, in plain C++20 without Eigen, the reference's per-iteration
// geometric path from /root/reference/proj:
//   se3.cpp:15-105            SE(3) group operations (Eigen formulas restated)
//   camera.cpp:15-108         Patch::make, reproject_patch, reprojection_jacobians
//   features.cpp:9-52         FeatureGrid::sample_zero_padded / sample_cubic
//   correlation.cpp:8-71      correlate_at, correlate
//   features.cpp:55-235      feature pyramid extraction (pool, whiten, lift) and
//                             crop_patch_features
//   flow_provider.cpp:34-93   OracleFlowProvider::propose (simulator revisions)
//   flow_provider.cpp:150-287 CorrelationFlowProvider::measure (parabola_refine,
//                             subpixel_peak) and propose's per-edge part (:289-314)
//   patch_graph.cpp:27-173    PatchGraph (std::map keyed, same iteration order)
//   pipeline.cpp:164-181      Pipeline::active_edges
//   bundle_adjust.cpp:11-375  validate, build_target, schur_solve (Eigen LDLT
//                             restated), weighted_residual_norm,
//                             gauss_newton_step, optimize_window
//
// The reference itself cannot be compiled here (Eigen3, libpng and the
// vendored doctest/CLI11/json are absent: proj/CMakeLists.txt:5,12,29), so
// this restatement is pinned by the reference's own known-answer and
// property tests, ported in tests/test_oracle_*.py.
// Eigen has no pinned version; the quaternion product, q*v, toRotationMatrix
// and the LDLT (left-looking, pivot on the largest remaining |diagonal|) are
// restated from Eigen 3.x's scalar code paths.
//
// Error behaviour: every extern "C" entry returns a status code
//   0 OK, 1 std::invalid_argument, 2 DegenerateProblem, 3 std::domain_error,
//   4 std::out_of_range, 5 other
// and leaves the exception message in orc_last_error().
// ============================================================================
#include <algorithm>
#include <cfloat>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

struct DegenerateProblem : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------------------
// Small fixed-size linear algebra (stand-ins for the Eigen types of se3.hpp:8-14)
// ---------------------------------------------------------------------------
struct V2 {
    double x = 0, y = 0;
};
struct V3 {
    double x = 0, y = 0, z = 0;
};
static inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
static inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
static inline V3 scale(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
static inline V3 cross(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
static inline double sqnorm(V3 a) { return a.x * a.x + a.y * a.y + a.z * a.z; }

struct M3 {
    double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
};
static inline M3 ident() {
    M3 r;
    r.m[0][0] = r.m[1][1] = r.m[2][2] = 1.0;
    return r;
}
static inline M3 mmul(const M3& a, const M3& b) {
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r.m[i][j] = a.m[i][0] * b.m[0][j] + a.m[i][1] * b.m[1][j] + a.m[i][2] * b.m[2][j];
    return r;
}
static inline V3 mvec(const M3& a, V3 v) {
    return {a.m[0][0] * v.x + a.m[0][1] * v.y + a.m[0][2] * v.z,
            a.m[1][0] * v.x + a.m[1][1] * v.y + a.m[1][2] * v.z,
            a.m[2][0] * v.x + a.m[2][1] * v.y + a.m[2][2] * v.z};
}
// skew: se3.cpp:22-26
static inline M3 skew(V3 v) {
    M3 r;
    r.m[0][1] = -v.z;
    r.m[0][2] = v.y;
    r.m[1][0] = v.z;
    r.m[1][2] = -v.x;
    r.m[2][0] = -v.y;
    r.m[2][1] = v.x;
    return r;
}

// Eigen::Quaterniond restated: coeffs stored (x, y, z, w).
struct Q {
    double x = 0, y = 0, z = 0, w = 1;
};
static inline Q qnormalized(Q q) {
    const double n2 = q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w;
    if (n2 > 0) {
        const double n = std::sqrt(n2);
        return {q.x / n, q.y / n, q.z / n, q.w / n};
    }
    return q;
}
// Hamilton product (Eigen quat_product).
static inline Q qmul(Q a, Q b) {
    Q r;
    r.w = a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z;
    r.x = a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y;
    r.y = a.w * b.y + a.y * b.w + a.z * b.x - a.x * b.z;
    r.z = a.w * b.z + a.z * b.w + a.x * b.y - a.y * b.x;
    return r;
}
// q * v (Eigen _transformVector): uv = 2 vec x v; v + w uv + vec x uv.
static inline V3 qrot(Q q, V3 v) {
    const V3 vec{q.x, q.y, q.z};
    V3 uv = cross(vec, v);
    uv = add(uv, uv);
    return add(add(v, scale(q.w, uv)), cross(vec, uv));
}
// toRotationMatrix (Eigen Quaternion::toRotationMatrix).
static inline M3 qmat(Q q) {
    const double tx = 2 * q.x, ty = 2 * q.y, tz = 2 * q.z;
    const double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
    const double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
    const double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
    M3 r;
    r.m[0][0] = 1 - (tyy + tzz);
    r.m[0][1] = txy - twz;
    r.m[0][2] = txz + twy;
    r.m[1][0] = txy + twz;
    r.m[1][1] = 1 - (txx + tzz);
    r.m[1][2] = tyz - twx;
    r.m[2][0] = txz - twy;
    r.m[2][1] = tyz + twx;
    r.m[2][2] = 1 - (txx + tyy);
    return r;
}

// ---------------------------------------------------------------------------
// SE(3): se3.hpp:16-77, se3.cpp:28-105
// ---------------------------------------------------------------------------
struct Pose {
    Q q;
    V3 t;
    Pose() = default;
    // se3.hpp:41 — the constructor always normalizes.
    Pose(Q q_, V3 t_) : q(qnormalized(q_)), t(t_) {}
    static Pose raw(Q q_, V3 t_) {  // exact coefficients (graph state set verbatim)
        Pose p;
        p.q = q_;
        p.t = t_;
        return p;
    }
    // se3.hpp:55-57 (Eigen coefficient-wise ==)
    bool bitwise_equal(const Pose& o) const {
        return q.x == o.q.x && q.y == o.q.y && q.z == o.q.z && q.w == o.q.w && t.x == o.t.x &&
               t.y == o.t.y && t.z == o.t.z;
    }
};

struct Tangent {
    V3 trans, rot;  // se3.hpp:18-32: translation first, then rotation
};

constexpr double kSmallAngle = 1e-8;        // se3.cpp:10
constexpr double kBranchCutMargin = 1e-6;   // se3.cpp:11

// se3.cpp:28-50
Pose exp(const Tangent& xi) {
    const V3 omega = xi.rot;
    const double theta2 = sqnorm(omega);
    const double theta = std::sqrt(theta2);
    Q q;
    M3 v;
    if (theta < kSmallAngle) {
        q = Q{0.5 * omega.x, 0.5 * omega.y, 0.5 * omega.z, 1.0};
        const M3 w = skew(omega);
        const M3 ww = mmul(w, w);
        v = ident();
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) v.m[i][j] = v.m[i][j] + 0.5 * w.m[i][j] + (1.0 / 6.0) * ww.m[i][j];
    } else {
        const double half = 0.5 * theta;
        const double s = std::sin(half) / theta;
        q = Q{s * omega.x, s * omega.y, s * omega.z, std::cos(half)};
        const M3 w = skew(omega);
        const M3 ww = mmul(w, w);
        const double a = (1.0 - std::cos(theta)) / theta2;
        const double b = (theta - std::sin(theta)) / (theta2 * theta);
        v = ident();
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) v.m[i][j] = v.m[i][j] + a * w.m[i][j] + b * ww.m[i][j];
    }
    return Pose(q, mvec(v, xi.trans));
}

// se3.cpp:52-80
Tangent log(const Pose& pose) {
    Q q = pose.q;
    if (q.w < 0.0) q = Q{-q.x, -q.y, -q.z, -q.w};
    const V3 vec{q.x, q.y, q.z};
    const double vec_norm = std::sqrt(sqnorm(vec));
    const double theta = 2.0 * std::atan2(vec_norm, q.w);
    if (theta >= M_PI - kBranchCutMargin) {
        throw std::domain_error("se3 log: rotation angle within 1e-6 of pi");
    }
    V3 omega;
    if (theta < kSmallAngle || vec_norm < kSmallAngle) {
        omega = scale(2.0, vec);
    } else {
        omega = scale(theta / vec_norm, vec);
    }
    const double theta2 = sqnorm(omega);
    const M3 w = skew(omega);
    const M3 ww = mmul(w, w);
    M3 v_inv = ident();
    double c;
    if (theta2 < kSmallAngle * kSmallAngle) {
        c = 1.0 / 12.0;
    } else {
        const double t = std::sqrt(theta2);
        c = (1.0 - t * std::sin(t) / (2.0 * (1.0 - std::cos(t)))) / theta2;
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) v_inv.m[i][j] = v_inv.m[i][j] - 0.5 * w.m[i][j] + c * ww.m[i][j];
    return Tangent{mvec(v_inv, pose.t), omega};
}

// se3.cpp:82-84
Pose compose(const Pose& a, const Pose& b) {
    return Pose(qmul(a.q, b.q), add(qrot(a.q, b.t), a.t));
}
// se3.cpp:86-89
Pose inverse(const Pose& a) {
    const Q qi{-a.q.x, -a.q.y, -a.q.z, a.q.w};
    return Pose(qi, scale(-1.0, qrot(qi, a.t)));
}
// se3.cpp:91-93
Pose retract(const Pose& a, const Tangent& xi) { return compose(exp(xi), a); }

// se3.cpp:95-99
double rotation_angle(const Pose& a) {
    Q q = a.q;
    if (q.w < 0.0) q = Q{-q.x, -q.y, -q.z, -q.w};
    return 2.0 * std::atan2(std::sqrt(q.x * q.x + q.y * q.y + q.z * q.z), q.w);
}
// se3.cpp:101-105
double pose_distance(const Pose& a, const Pose& b, double* angle_out) {
    const Pose delta = compose(a, inverse(b));
    if (angle_out) *angle_out = rotation_angle(delta);
    return std::sqrt(sqnorm(delta.t));
}

// ---------------------------------------------------------------------------
// Camera: camera.hpp:10-72, camera.cpp:15-108
// ---------------------------------------------------------------------------
struct Intrinsics {
    double fx = 0, fy = 0, cx = 0, cy = 0;
    V3 unproject(double px, double py) const { return {(px - cx) / fx, (py - cy) / fy, 1.0}; }
};

struct Patch {
    int source_frame = -1;
    int width = 0;
    std::vector<double> x, y;
    double inverse_depth = 0.0;
    int size() const { return width * width; }
    // camera.cpp:34-45
    V2 center() const {
        if (width % 2 == 1) {
            const int mid = size() / 2;
            return {x[mid], y[mid]};
        }
        double sx = 0, sy = 0;
        for (int k = 0; k < size(); ++k) {
            sx += x[k];
            sy += y[k];
        }
        return {sx / size(), sy / size()};
    }
};

// camera.cpp:15-32
Patch make_patch(int source_frame, V2 centroid, int width, double inverse_depth) {
    if (width < 1) throw std::invalid_argument("patch: width must be >= 1");
    if (inverse_depth < 0) throw std::invalid_argument("patch: inverse depth must be >= 0");
    Patch p;
    p.source_frame = source_frame;
    p.width = width;
    p.inverse_depth = inverse_depth;
    const double half = 0.5 * (width - 1);
    for (int row = 0; row < width; ++row) {
        for (int col = 0; col < width; ++col) {
            p.x.push_back(centroid.x + col - half);
            p.y.push_back(centroid.y + row - half);
        }
    }
    return p;
}

constexpr double kDepthEpsilon = 1e-6;  // camera.hpp:43

struct PatchReprojection {
    std::vector<V2> points;
    bool behind_camera = false;
};

// camera.cpp:47-71
PatchReprojection reproject_patch(const Pose& pi, const Pose& pj, const Intrinsics& K,
                                  const Patch& patch) {
    PatchReprojection out;
    out.points.reserve(patch.size());
    if (pi.bitwise_equal(pj)) {
        for (int k = 0; k < patch.size(); ++k) out.points.push_back({patch.x[k], patch.y[k]});
        return out;
    }
    const Pose rel = compose(pj, inverse(pi));
    const M3 r = qmat(rel.q);
    const V3 ts = scale(patch.inverse_depth, rel.t);
    for (int k = 0; k < patch.size(); ++k) {
        const V3 ray = K.unproject(patch.x[k], patch.y[k]);
        const V3 q = add(mvec(r, ray), ts);
        if (q.z <= kDepthEpsilon) out.behind_camera = true;
        const double z = std::max(q.z, kDepthEpsilon);
        out.points.push_back({K.fx * q.x / z + K.cx, K.fy * q.y / z + K.cy});
    }
    return out;
}

struct Jacobians {
    V2 center;
    double di[2][6];
    double dj[2][6];
    double dd[2];
    bool behind = false;
};

// camera.cpp:73-108 (no bitwise shortcut here)
Jacobians reprojection_jacobians(const Pose& pi, const Pose& pj, const Intrinsics& K,
                                 const Patch& patch) {
    const Pose rel = compose(pj, inverse(pi));
    const M3 r = qmat(rel.q);
    const V3 t = rel.t;
    const double d = patch.inverse_depth;
    const V2 c = patch.center();
    const V3 ray = K.unproject(c.x, c.y);
    const V3 q = add(mvec(r, ray), scale(d, t));
    Jacobians jac;
    jac.behind = q.z <= kDepthEpsilon;
    const double z = std::max(q.z, kDepthEpsilon);
    jac.center = {K.fx * q.x / z + K.cx, K.fy * q.y / z + K.cy};
    const double P[2][3] = {{K.fx / z, 0, -K.fx * q.x / (z * z)},
                            {0, K.fy / z, -K.fy * q.y / (z * z)}};
    // d q / d xi_j = [d I | -[q]x];  d q / d xi_i = [-d R | R [ray]x]
    double Aj[3][6], Ai[3][6];
    const M3 sq = skew(q);
    const M3 rs = mmul(r, skew(ray));
    for (int m = 0; m < 3; ++m) {
        for (int c3 = 0; c3 < 3; ++c3) {
            Aj[m][c3] = (m == c3) ? d : 0.0;
            Aj[m][3 + c3] = -sq.m[m][c3];
            Ai[m][c3] = -d * r.m[m][c3];
            Ai[m][3 + c3] = rs.m[m][c3];
        }
    }
    for (int row = 0; row < 2; ++row) {
        for (int col = 0; col < 6; ++col) {
            jac.dj[row][col] = P[row][0] * Aj[0][col] + P[row][1] * Aj[1][col] + P[row][2] * Aj[2][col];
            jac.di[row][col] = P[row][0] * Ai[0][col] + P[row][1] * Ai[1][col] + P[row][2] * Ai[2][col];
        }
        jac.dd[row] = P[row][0] * t.x + P[row][1] * t.y + P[row][2] * t.z;
    }
    return jac;
}

// ---------------------------------------------------------------------------
// Features + correlation: features.hpp:14-64, features.cpp:9-52,
// correlation.hpp:11-44, correlation.cpp:8-71
// ---------------------------------------------------------------------------
struct GridView {
    const float* data = nullptr;
    int width = 0, height = 0, channels = 0;
    float at(int x, int y, int c) const {
        return data[(static_cast<size_t>(y) * width + x) * channels + c];
    }
    // features.cpp:9-21
    double sample_zero_padded(double x, double y, int c) const {
        const int x0 = static_cast<int>(std::floor(x));
        const int y0 = static_cast<int>(std::floor(y));
        const double ax = x - x0;
        const double ay = y - y0;
        auto value = [this, c](int xi, int yi) -> double {
            if (xi < 0 || yi < 0 || xi >= width || yi >= height) return 0.0;
            return at(xi, yi, c);
        };
        return (1 - ax) * (1 - ay) * value(x0, y0) + ax * (1 - ay) * value(x0 + 1, y0) +
               (1 - ax) * ay * value(x0, y0 + 1) + ax * ay * value(x0 + 1, y0 + 1);
    }
    // features.cpp:23-52
    double sample_cubic(double x, double y, int c) const {
        const int x0 = static_cast<int>(std::floor(x));
        const int y0 = static_cast<int>(std::floor(y));
        const double tx = x - x0, ty = y - y0;
        auto weights = [](double t, double w[4]) {
            w[0] = ((-0.5 * t + 1.0) * t - 0.5) * t;
            w[1] = (1.5 * t - 2.5) * t * t + 1.0;
            w[2] = ((-1.5 * t + 2.0) * t + 0.5) * t;
            w[3] = (0.5 * t - 0.5) * t * t;
        };
        double wx[4], wy[4];
        weights(tx, wx);
        weights(ty, wy);
        double v = 0;
        for (int j = 0; j < 4; ++j) {
            const int yi = y0 - 1 + j;
            if (yi < 0 || yi >= height) continue;
            double row = 0;
            for (int i = 0; i < 4; ++i) {
                const int xi = x0 - 1 + i;
                if (xi < 0 || xi >= width) continue;
                row += wx[i] * at(xi, yi, c);
            }
            v += wy[j] * row;
        }
        return v;
    }
};

constexpr int kCorrRadius = 3;                     // correlation.hpp:11
constexpr int kCorrSize = 2 * kCorrRadius + 1;     // correlation.hpp:12
constexpr double kFeatureStride = 4.0;             // features.hpp:46

// correlation.cpp:8-23
double correlate_at(const float* feature, int channels, const GridView& grid, double x, double y) {
    double dot = 0, norm_sq = 0;
    for (int c = 0; c < channels; ++c) {
        const double v = grid.sample_zero_padded(x, y, c);
        dot += feature[c] * v;
        norm_sq += v * v;
    }
    return norm_sq > 1e-12 ? dot / std::sqrt(norm_sq) : 0.0;
}

// correlation.cpp:25-35
double correlate_at_cubic(const float* feature, int channels, const GridView& grid, double x,
                          double y) {
    double dot = 0, norm_sq = 0;
    for (int c = 0; c < channels; ++c) {
        const double v = grid.sample_cubic(x, y, c);
        dot += feature[c] * v;
        norm_sq += v * v;
    }
    return norm_sq > 1e-12 ? dot / std::sqrt(norm_sq) : 0.0;
}

// correlation.cpp:37-71.  feats[l] = p*p*channels descriptors of level l;
// out = [2][p*p][7][7] in the reference's index order.
void correlate(int p, int channels, const float* feats0, const float* feats1, const GridView& l0,
               const GridView& l1, const double* coords /* p*p x 2 */, float* out) {
    for (int k = 0; k < p * p; ++k) {
        if (!std::isfinite(coords[2 * k]) || !std::isfinite(coords[2 * k + 1])) {
            throw std::invalid_argument("correlate: non-finite reprojection");
        }
    }
    const GridView* levels[2] = {&l0, &l1};
    const float* feats[2] = {feats0, feats1};
    const size_t per_level = static_cast<size_t>(p) * p * kCorrSize * kCorrSize;
    for (int level = 0; level < 2; ++level) {
        const double s = kFeatureStride * (level == 0 ? 1.0 : kFeatureStride);
        size_t idx = 0;
        for (int v = 0; v < p; ++v) {
            for (int u = 0; u < p; ++u) {
                const float* g = feats[level] + static_cast<size_t>(v * p + u) * channels;
                const double bx = coords[2 * (v * p + u)] / s;
                const double by = coords[2 * (v * p + u) + 1] / s;
                for (int alpha = 0; alpha < kCorrSize; ++alpha) {
                    for (int beta = 0; beta < kCorrSize; ++beta) {
                        out[level * per_level + idx++] = static_cast<float>(correlate_at(
                            g, channels, *levels[level], bx + (beta - kCorrRadius),
                            by + (alpha - kCorrRadius)));
                    }
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// CorrelationFlowProvider::measure (flow_provider.cpp:150-287)
// ---------------------------------------------------------------------------
struct Measurement {
    V2 delta{0, 0};
    V2 weight{0.01, 0.01};
    bool flat = false, out_of_range = false;
};

// flow_provider.cpp:152-162
double parabola_refine(const float* feature, int channels, const GridView& grid, double x, double y, bool along_x,
                       double h) {
    const double f0 = correlate_at_cubic(feature, channels, grid, x - (along_x ? h : 0), y - (along_x ? 0 : h));
    const double f1 = correlate_at_cubic(feature, channels, grid, x, y);
    const double f2 = correlate_at_cubic(feature, channels, grid, x + (along_x ? h : 0), y + (along_x ? 0 : h));
    const double denom = f0 - 2 * f1 + f2;
    if (std::abs(denom) < 1e-12 || denom > 0) return 0.0;  // not a local max
    return std::clamp(0.5 * h * (f0 - f2) / denom, -h, h);
}

// flow_provider.cpp:167-205
V2 subpixel_peak(const float* feature, int channels, const GridView& grid, V2 base, bool* on_border) {
    int best_a = kCorrRadius, best_b = kCorrRadius;
    double best = -std::numeric_limits<double>::infinity();
    for (int alpha = 0; alpha < kCorrSize; ++alpha) {
        for (int beta = 0; beta < kCorrSize; ++beta) {
            const double v =
                correlate_at(feature, channels, grid, base.x + beta - kCorrRadius, base.y + alpha - kCorrRadius);
            if (v > best) {
                best = v;
                best_a = alpha;
                best_b = beta;
            }
        }
    }
    if (on_border) *on_border = best_a == 0 || best_a == kCorrSize - 1 || best_b == 0 || best_b == kCorrSize - 1;
    double dx = best_b - kCorrRadius, dy = best_a - kCorrRadius;
    double current = correlate_at_cubic(feature, channels, grid, base.x + dx, base.y + dy);
    for (const double h : {0.5, 0.25, 0.125, 0.0625, 0.03125, 0.015625}) {
        for (const bool along_x : {true, false}) {
            const double step = parabola_refine(feature, channels, grid, base.x + dx, base.y + dy, along_x, h);
            if (step == 0.0) continue;
            const double nx = dx + (along_x ? step : 0);
            const double ny = dy + (along_x ? 0 : step);
            const double value = correlate_at_cubic(feature, channels, grid, base.x + nx, base.y + ny);
            if (value >= current) {  // hill climb only
                dx = nx;
                dy = ny;
                current = value;
            }
        }
    }
    return {dx, dy};
}

// flow_provider.cpp:209-287; g0 / g1 = the centre pixel's level-0 / level-1 descriptors
Measurement measure(const float* g0, const float* g1, int channels, const GridView& l0, const GridView& l1,
                    V2 center) {
    Measurement m;
    const V2 base0{center.x / kFeatureStride, center.y / kFeatureStride};
    double values[kCorrSize * kCorrSize];
    double peak = -std::numeric_limits<double>::infinity();
    double minimum = std::numeric_limits<double>::infinity();
    double mean = 0;
    int peak_a = 0, peak_b = 0;
    for (int alpha = 0; alpha < kCorrSize; ++alpha) {
        for (int beta = 0; beta < kCorrSize; ++beta) {
            const double v = correlate_at(g0, channels, l0, base0.x + beta - kCorrRadius, base0.y + alpha - kCorrRadius);
            values[alpha * kCorrSize + beta] = v;
            mean += v;
            minimum = std::min(minimum, v);
            if (v > peak) {
                peak = v;
                peak_a = alpha;
                peak_b = beta;
            }
        }
    }
    mean /= kCorrSize * kCorrSize;
    const double peak_to_mean = (peak - minimum) / (mean - minimum + 1e-9);
    if (!(peak_to_mean >= 1.05)) {
        m.flat = true;
        return m;
    }
    double second = -std::numeric_limits<double>::infinity();
    for (int alpha = 0; alpha < kCorrSize; ++alpha) {
        for (int beta = 0; beta < kCorrSize; ++beta) {
            if (std::max(std::abs(alpha - peak_a), std::abs(beta - peak_b)) <= 1) continue;
            second = std::max(second, values[alpha * kCorrSize + beta]);
        }
    }
    const double score = 2.0 * (peak - 0.75) + (peak - second - 0.08);
    double confidence = std::clamp(1.0 / (1.0 + std::exp(-12.0 * score)), 0.01, 0.99);
    bool border0 = false, border1 = false;
    const V2 peak0 = subpixel_peak(g0, channels, l0, base0, &border0);
    const double s1 = kFeatureStride * kFeatureStride;
    const V2 peak1 = subpixel_peak(g1, channels, l1, {center.x / s1, center.y / s1}, &border1);
    const V2 e0{kFeatureStride * peak0.x, kFeatureStride * peak0.y};
    const V2 e1{s1 * peak1.x, s1 * peak1.y};
    if (border0 && border1) {
        m.out_of_range = true;
        return m;
    }
    if (border0) {
        m.delta = e1;
        confidence = std::min(confidence, 0.25);
    } else {
        m.delta = e0;
        const double dx = e1.x - e0.x, dy = e1.y - e0.y;
        if (!border1 && std::sqrt(dx * dx + dy * dy) > 2.0 * kFeatureStride * kFeatureStride) {
            confidence = std::min(confidence, 0.25);
        }
    }
    m.weight = {confidence, confidence};
    return m;
}

// ---------------------------------------------------------------------------
// PatchGraph: patch_graph.hpp:15-136, patch_graph.cpp:27-173
// ---------------------------------------------------------------------------
struct FlowRevision {
    V2 delta, weight;
};
struct FrameNode {
    int frame_index = -1;
    double timestamp = 0;
    Pose pose;
};
struct LogEntry {
    int removed_frame = -1, anchor_frame = -1;
    Pose relative;
    double timestamp = 0;
};

class PatchGraph {
  public:
    using EdgeKey = std::pair<int, int>;
    PatchGraph(const Intrinsics& K, int w, int h, int p) : K_(K), w_(w), h_(h), p_(p) {
        if (p < 1) throw std::invalid_argument("patch graph: patch width must be >= 1");
    }
    // patch_graph.cpp:27-34
    int add_frame(double ts, const Pose& pose) {
        if (!frames_.empty() && ts <= frames_.rbegin()->second.timestamp) {
            throw std::invalid_argument("patch graph: timestamp must exceed the last frame's");
        }
        const int index = frames_.empty() ? 0 : frames_.rbegin()->first + 1;
        frames_[index] = FrameNode{index, ts, pose};
        return index;
    }
    // patch_graph.cpp:36-60
    std::vector<int> add_patches(int frame, const std::vector<V2>& centroids,
                                 const std::vector<double>& depths) {
        if (!frames_.count(frame)) {
            throw std::invalid_argument("patch graph: no frame " + std::to_string(frame));
        }
        if (centroids.size() != depths.size()) {
            throw std::invalid_argument("patch graph: centroid/depth count mismatch");
        }
        const double half = 0.5 * (p_ - 1);
        std::vector<int> ids;
        for (size_t k = 0; k < centroids.size(); ++k) {
            const V2 c = centroids[k];
            if (c.x - half < 0 || c.y - half < 0 || c.x + half > w_ - 1 || c.y + half > h_ - 1) {
                throw std::invalid_argument("patch graph: centroid leaves the image bounds");
            }
            const int id = next_patch_id_++;
            patches_.emplace(id, make_patch(frame, c, p_, depths[k]));
            ids.push_back(id);
        }
        return ids;
    }
    std::map<int, int> positions() const {
        std::map<int, int> pos;
        int i = 0;
        for (const auto& kv : frames_) pos[kv.first] = i++;
        return pos;
    }
    // patch_graph.cpp:62-85
    std::vector<EdgeKey> connect(int radius) {
        if (radius < 1) throw std::invalid_argument("patch graph: radius must be >= 1");
        const std::map<int, int> position = positions();
        std::vector<EdgeKey> added;
        for (const auto& [patch_id, patch] : patches_) {
            const int src = position.at(patch.source_frame);
            for (const auto& [frame_index, node] : frames_) {
                if (std::abs(position.at(frame_index) - src) > radius - 1) continue;
                const EdgeKey key{patch_id, frame_index};
                if (edges_.emplace(key, std::nullopt).second) added.push_back(key);
            }
        }
        return added;
    }
    // patch_graph.cpp:87-128
    void remove_frame(int frame_index) {
        auto it = frames_.find(frame_index);
        if (it == frames_.end()) {
            throw std::invalid_argument("patch graph: no frame " + std::to_string(frame_index));
        }
        int newer = 0;
        for (auto r = frames_.rbegin(); r != frames_.rend() && newer < 3; ++r) {
            if (r->first == frame_index) {
                throw std::invalid_argument("patch graph: frame is among the most recent 3 keyframes");
            }
            ++newer;
        }
        if (it == frames_.begin()) {
            throw std::invalid_argument("patch graph: the oldest frame has no predecessor to anchor");
        }
        auto pred = std::prev(it);
        log_.push_back({frame_index, pred->first, compose(it->second.pose, inverse(pred->second.pose)),
                        it->second.timestamp});
        for (auto e = edges_.begin(); e != edges_.end();) {
            if (e->first.second == frame_index) e = edges_.erase(e);
            else ++e;
        }
        for (auto p = patches_.begin(); p != patches_.end();) {
            if (p->second.source_frame == frame_index) {
                const int id = p->first;
                edges_.erase(edges_.lower_bound({id, std::numeric_limits<int>::min()}),
                             edges_.upper_bound({id, std::numeric_limits<int>::max()}));
                p = patches_.erase(p);
            } else {
                ++p;
            }
        }
        frames_.erase(it);
    }
    // patch_graph.cpp:153-164
    void set_revision(const EdgeKey& key, const FlowRevision& rev) {
        auto it = edges_.find(key);
        if (it == edges_.end()) throw std::invalid_argument("patch graph: no edge");
        if (rev.weight.x <= 0 || rev.weight.x >= 1 || rev.weight.y <= 0 || rev.weight.y >= 1) {
            throw std::invalid_argument("patch graph: revision weights must lie in (0, 1)");
        }
        it->second = rev;
    }
    // patch_graph.cpp:166-173
    std::vector<EdgeKey> edges_of_patch(int patch_id) const {
        std::vector<EdgeKey> keys;
        for (auto it = edges_.lower_bound({patch_id, std::numeric_limits<int>::min()});
             it != edges_.end() && it->first.first == patch_id; ++it) {
            keys.push_back(it->first);
        }
        return keys;
    }

    const Intrinsics& intrinsics() const { return K_; }
    int image_width() const { return w_; }
    int image_height() const { return h_; }
    int patch_width() const { return p_; }
    const std::map<int, FrameNode>& frames() const { return frames_; }
    const std::map<int, Patch>& patches() const { return patches_; }
    const std::map<EdgeKey, std::optional<FlowRevision>>& edges() const { return edges_; }
    const FrameNode& frame(int i) const { return frames_.at(i); }
    const Patch& patch(int i) const { return patches_.at(i); }
    void set_pose(int i, const Pose& p) { frames_.at(i).pose = p; }
    void set_inverse_depth(int i, double d) { patches_.at(i).inverse_depth = d; }
    const std::vector<LogEntry>& log() const { return log_; }

  private:
    Intrinsics K_;
    int w_, h_, p_;
    int next_patch_id_ = 0;
    std::map<int, FrameNode> frames_;
    std::map<int, Patch> patches_;
    std::map<EdgeKey, std::optional<FlowRevision>> edges_;
    std::vector<LogEntry> log_;
};

// pipeline.cpp:164-181
std::vector<PatchGraph::EdgeKey> active_edges(const PatchGraph& graph, int window) {
    std::vector<int> recent;
    for (auto it = graph.frames().rbegin();
         it != graph.frames().rend() && static_cast<int>(recent.size()) < window; ++it) {
        recent.push_back(it->first);
    }
    const int oldest = recent.empty() ? 0 : recent.back();
    std::vector<PatchGraph::EdgeKey> edges;
    for (const auto& [key, rev] : graph.edges()) {
        if (graph.patch(key.first).source_frame >= oldest) edges.push_back(key);
    }
    return edges;
}

// ---------------------------------------------------------------------------
// Bundle adjustment: bundle_adjust.hpp:15-111, bundle_adjust.cpp:11-375
// ---------------------------------------------------------------------------
constexpr double kDefaultDamping = 1e-4;        // bundle_adjust.hpp:15
constexpr double kMaxObservableMarginPx = 32.0; // bundle_adjust.hpp:18

struct BAEdge {
    int patch_id = -1, target_pose = -1;
    V2 target_point, weight;
};
struct BAProblem {
    std::vector<Pose> poses;
    std::vector<bool> pose_fixed;
    std::vector<Patch> patches;
    std::vector<bool> depth_free;
    std::vector<BAEdge> edges;
    Intrinsics intrinsics;
    double damping = kDefaultDamping;

    // bundle_adjust.cpp:11-36
    void validate() const {
        if (poses.size() != pose_fixed.size()) {
            throw std::invalid_argument("ba: pose/fixed-mask size mismatch");
        }
        if (!depth_free.empty() && depth_free.size() != patches.size()) {
            throw std::invalid_argument("ba: depth mask size mismatch");
        }
        for (const BAEdge& e : edges) {
            if (e.patch_id < 0 || e.patch_id >= static_cast<int>(patches.size()) || e.target_pose < 0 ||
                e.target_pose >= static_cast<int>(poses.size())) {
                throw std::invalid_argument("ba: edge references an unknown patch or pose");
            }
            if (!std::isfinite(e.target_point.x) || !std::isfinite(e.target_point.y)) {
                throw std::invalid_argument("ba: non-finite edge target");
            }
            if (e.weight.x < 0 || e.weight.x >= 1 || e.weight.y < 0 || e.weight.y >= 1) {
                throw std::invalid_argument("ba: edge weights must lie in [0, 1)");
            }
        }
        for (const Patch& p : patches) {
            if (p.source_frame < 0 || p.source_frame >= static_cast<int>(poses.size())) {
                throw std::invalid_argument("ba: patch source pose out of range");
            }
        }
    }
};

struct BASolution {
    std::vector<Pose> poses;
    std::vector<double> inverse_depths;
    std::vector<double> residual_norms;
    int num_edges = 0;
};

struct Dense {
    int rows = 0, cols = 0;
    std::vector<double> a;
    Dense() = default;
    Dense(int r, int c) : rows(r), cols(c), a(static_cast<size_t>(r) * c, 0.0) {}
    double& operator()(int r, int c) { return a[static_cast<size_t>(r) * cols + c]; }
    double operator()(int r, int c) const { return a[static_cast<size_t>(r) * cols + c]; }
};

struct NormalEquations {
    Dense h;
    std::vector<double> b;
    int num_free_poses = 0, num_free_depths = 0;
};

// bundle_adjust.cpp:47-60
V2 build_target(const PatchGraph& graph, const PatchGraph::EdgeKey& edge) {
    const auto it = graph.edges().find(edge);
    if (it == graph.edges().end()) throw std::invalid_argument("build_target: no such edge");
    if (!it->second.has_value()) throw std::invalid_argument("build_target: edge has no revision");
    const Patch& patch = graph.patch(edge.first);
    const PatchReprojection r = reproject_patch(graph.frame(patch.source_frame).pose,
                                                graph.frame(edge.second).pose, graph.intrinsics(), patch);
    const V2 c = r.points[patch.size() / 2];
    return {c.x + it->second->delta.x, c.y + it->second->delta.y};
}

// Eigen::LDLT<MatrixXd> (Lower) restated: ldlt_inplace<Lower>::unblocked + _solve_impl.
// Returns false when Eigen's info() would report NumericalIssue.
bool ldlt_solve(Dense mat, const std::vector<double>& rhs, std::vector<double>& x) {
    const int n = mat.rows;
    std::vector<int> transp(n);
    std::vector<double> temp(n);
    bool ret = true;
    for (int k = 0; k < n; ++k) {
        int big = k;
        double bigv = std::abs(mat(k, k));
        for (int i = k + 1; i < n; ++i) {
            if (std::abs(mat(i, i)) > bigv) {
                bigv = std::abs(mat(i, i));
                big = i;
            }
        }
        transp[k] = big;
        if (k != big) {
            for (int j = 0; j < k; ++j) std::swap(mat(k, j), mat(big, j));
            for (int i = big + 1; i < n; ++i) std::swap(mat(i, k), mat(i, big));
            std::swap(mat(k, k), mat(big, big));
            for (int i = k + 1; i < big; ++i) {
                const double tmp = mat(i, k);
                mat(i, k) = mat(big, i);
                mat(big, i) = tmp;
            }
        }
        const int rs = n - k - 1;
        if (k > 0) {
            for (int j = 0; j < k; ++j) temp[j] = mat(j, j) * mat(k, j);
            double s = 0;
            for (int j = 0; j < k; ++j) s += mat(k, j) * temp[j];
            mat(k, k) -= s;
            for (int i = k + 1; i < n; ++i) {
                double si = 0;
                for (int j = 0; j < k; ++j) si += mat(i, j) * temp[j];
                mat(i, k) -= si;
            }
        }
        const double akk = mat(k, k);
        const bool valid = std::abs(akk) > 0.0;
        if (k == 0 && !valid) {
            for (int j = 0; j < n; ++j) {
                transp[j] = j;
                mat(j, j) = 0;
            }
            break;
        }
        if (rs > 0 && valid) {
            for (int i = k + 1; i < n; ++i) mat(i, k) /= akk;
        } else if (rs > 0) {
            for (int i = k + 1; i < n; ++i) ret = ret && mat(i, k) == 0.0;
        }
    }
    x = rhs;
    for (int k = 0; k < n; ++k) std::swap(x[k], x[transp[k]]);
    for (int i = 0; i < n; ++i) {
        double s = 0;
        for (int j = 0; j < i; ++j) s += mat(i, j) * x[j];
        x[i] -= s;
    }
    for (int i = 0; i < n; ++i) {
        const double d = mat(i, i);
        if (std::abs(d) > DBL_MIN) x[i] /= d;
        else x[i] = 0;
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = 0;
        for (int j = i + 1; j < n; ++j) s += mat(j, i) * x[j];
        x[i] -= s;
    }
    for (int k = n - 1; k >= 0; --k) std::swap(x[k], x[transp[k]]);
    return ret;
}

struct SchurResult {
    std::vector<double> pose_delta, depth_delta;
};

static bool all_finite(const std::vector<double>& v) {
    for (double x : v)
        if (!std::isfinite(x)) return false;
    return true;
}

// bundle_adjust.cpp:62-94.  h_pd is np x nd.
SchurResult schur_solve(const Dense& h_pp, const Dense& h_pd, const std::vector<double>& h_dd,
                        const std::vector<double>& b_p, const std::vector<double>& b_d) {
    for (double v : h_dd)
        if (v <= 0) throw DegenerateProblem("schur: non-positive damped depth-block entry");
    const int np = h_pp.rows, nd = static_cast<int>(h_dd.size());
    std::vector<double> d_inv(nd);
    for (int k = 0; k < nd; ++k) d_inv[k] = 1.0 / h_dd[k];
    SchurResult res;
    if (np > 0) {
        Dense reduced = h_pp;
        // H_pd * diag(d_inv) * H_pd^T, blocked over depths (Eigen GEMM stand-in).
        std::vector<double> row_i(nd);
        for (int i = 0; i < np; ++i) {
            for (int k = 0; k < nd; ++k) row_i[k] = h_pd(i, k) * d_inv[k];
            for (int j = 0; j < np; ++j) {
                double s = 0;
                const double* hj = &h_pd.a[static_cast<size_t>(j) * nd];
                for (int k = 0; k < nd; ++k) s += row_i[k] * hj[k];
                reduced(i, j) -= s;
            }
        }
        std::vector<double> rhs(np);
        for (int i = 0; i < np; ++i) {
            double s = 0;
            for (int k = 0; k < nd; ++k) s += h_pd(i, k) * (d_inv[k] * b_d[k]);
            rhs[i] = b_p[i] - s;
        }
        if (!ldlt_solve(reduced, rhs, res.pose_delta)) {
            throw DegenerateProblem("schur: reduced camera system factorization failed");
        }
        if (!all_finite(res.pose_delta)) throw DegenerateProblem("schur: non-finite pose update");
    }
    res.depth_delta.resize(nd);
    for (int k = 0; k < nd; ++k) {
        double s = 0;
        for (int i = 0; i < np; ++i) s += h_pd(i, k) * res.pose_delta[i];
        res.depth_delta[k] = d_inv[k] * (b_d[k] - s);
    }
    if (!all_finite(res.depth_delta)) throw DegenerateProblem("schur: non-finite depth update");
    return res;
}

// bundle_adjust.cpp:99-113
double weighted_residual_norm(const BAProblem& pr) {
    double sum = 0, wsum = 0;
    for (const BAEdge& e : pr.edges) {
        const Patch& patch = pr.patches[e.patch_id];
        const PatchReprojection r =
            reproject_patch(pr.poses[patch.source_frame], pr.poses[e.target_pose], pr.intrinsics, patch);
        const V2 c = r.points[patch.size() / 2];
        const double rx = c.x - e.target_point.x, ry = c.y - e.target_point.y;
        const double wx = r.behind_camera ? 0.0 : e.weight.x;
        const double wy = r.behind_camera ? 0.0 : e.weight.y;
        sum += wx * rx * rx + wy * ry * ry;
        wsum += wx + wy;
    }
    return wsum > 0 ? std::sqrt(sum / wsum) : 0.0;
}

// bundle_adjust.cpp:117-223
BASolution gauss_newton_step(const BAProblem& pr, NormalEquations* debug) {
    pr.validate();
    if (pr.edges.empty()) throw std::invalid_argument("ba: need at least one edge");
    std::vector<int> pose_slot(pr.poses.size(), -1);
    int nfp = 0;
    for (size_t i = 0; i < pr.poses.size(); ++i)
        if (!pr.pose_fixed[i]) pose_slot[i] = nfp++;
    std::vector<int> depth_slot(pr.patches.size(), -1);
    int nfd = 0;
    for (size_t k = 0; k < pr.patches.size(); ++k)
        if (pr.depth_free.empty() || pr.depth_free[k]) depth_slot[k] = nfd++;
    const int np = 6 * nfp, nd = nfd, n = np + nd;
    Dense h(n, n);
    std::vector<double> b(n, 0.0);

    for (const BAEdge& e : pr.edges) {
        const Patch& patch = pr.patches[e.patch_id];
        const Jacobians jac =
            reprojection_jacobians(pr.poses[patch.source_frame], pr.poses[e.target_pose], pr.intrinsics, patch);
        const double r[2] = {jac.center.x - e.target_point.x, jac.center.y - e.target_point.y};
        if (!std::isfinite(r[0]) || !std::isfinite(r[1])) throw DegenerateProblem("ba: non-finite residual");
        const double w[2] = {jac.behind ? 0.0 : e.weight.x, jac.behind ? 0.0 : e.weight.y};
        if (w[0] == 0.0 && w[1] == 0.0) continue;
        struct Block {
            int off, cols;
            double j[2][6];
        } blocks[3];
        int nb = 0;
        const int si = pose_slot[patch.source_frame], sj = pose_slot[e.target_pose], sd = depth_slot[e.patch_id];
        if (si >= 0) {
            blocks[nb].off = 6 * si;
            blocks[nb].cols = 6;
            std::memcpy(blocks[nb].j, jac.di, sizeof(jac.di));
            ++nb;
        }
        if (sj >= 0) {
            blocks[nb].off = 6 * sj;
            blocks[nb].cols = 6;
            std::memcpy(blocks[nb].j, jac.dj, sizeof(jac.dj));
            ++nb;
        }
        if (sd >= 0) {
            blocks[nb].off = np + sd;
            blocks[nb].cols = 1;
            std::memset(blocks[nb].j, 0, sizeof(blocks[nb].j));
            blocks[nb].j[0][0] = jac.dd[0];
            blocks[nb].j[1][0] = jac.dd[1];
            ++nb;
        }
        for (int a = 0; a < nb; ++a) {
            for (int ra = 0; ra < blocks[a].cols; ++ra) {
                const double t0 = blocks[a].j[0][ra] * w[0];
                const double t1 = blocks[a].j[1][ra] * w[1];
                b[blocks[a].off + ra] -= t0 * r[0] + t1 * r[1];
                for (int c = 0; c < nb; ++c) {
                    for (int rc = 0; rc < blocks[c].cols; ++rc) {
                        h(blocks[a].off + ra, blocks[c].off + rc) += t0 * blocks[c].j[0][rc] + t1 * blocks[c].j[1][rc];
                    }
                }
            }
        }
    }
    for (int i = 0; i < n; ++i) h(i, i) += pr.damping;
    if (debug) {
        debug->h = h;
        debug->b = b;
        debug->num_free_poses = nfp;
        debug->num_free_depths = nfd;
    }
    Dense hpp(np, np), hpd(np, nd);
    for (int i = 0; i < np; ++i) {
        for (int j = 0; j < np; ++j) hpp(i, j) = h(i, j);
        for (int k = 0; k < nd; ++k) hpd(i, k) = h(i, np + k);
    }
    std::vector<double> hdd(nd), bp(b.begin(), b.begin() + np), bd(b.begin() + np, b.end());
    for (int k = 0; k < nd; ++k) hdd[k] = h(np + k, np + k);
    const SchurResult delta = schur_solve(hpp, hpd, hdd, bp, bd);

    BASolution sol;
    sol.num_edges = static_cast<int>(pr.edges.size());
    sol.residual_norms.push_back(weighted_residual_norm(pr));
    sol.poses = pr.poses;
    for (size_t i = 0; i < pr.poses.size(); ++i) {
        if (pose_slot[i] >= 0) {
            const double* d = &delta.pose_delta[6 * pose_slot[i]];
            sol.poses[i] = retract(pr.poses[i], Tangent{{d[0], d[1], d[2]}, {d[3], d[4], d[5]}});
        }
    }
    sol.inverse_depths.resize(pr.patches.size());
    for (size_t k = 0; k < pr.patches.size(); ++k) {
        double d = pr.patches[k].inverse_depth;
        if (depth_slot[k] >= 0) d = std::max(0.0, d + delta.depth_delta[depth_slot[k]]);
        sol.inverse_depths[k] = d;
    }
    BAProblem upd = pr;
    upd.poses = sol.poses;
    for (size_t k = 0; k < upd.patches.size(); ++k) upd.patches[k].inverse_depth = sol.inverse_depths[k];
    sol.residual_norms.push_back(weighted_residual_norm(upd));
    return sol;
}

struct WindowOptions {
    int window = 10, iterations = 2, structure_only_iterations = 0;
    double damping = kDefaultDamping;
};

// Problem build of bundle_adjust.cpp:225-307, factored out so tests can
// compare the flattened problem (slot maps, edge order, frozen targets).
struct WindowProblem {
    BAProblem problem;
    std::vector<int> pose_frames;  // slot -> frame index
    std::vector<int> patch_ids;    // slot -> patch id
};

bool build_window_problem(const PatchGraph& graph, const WindowOptions& options, WindowProblem& out) {
    if (options.window < 1) throw std::invalid_argument("ba: window must be >= 1");
    const auto& frames = graph.frames();
    const int num_frames = static_cast<int>(frames.size());
    const std::map<int, int> position = graph.positions();
    const int window_start = std::max(num_frames - options.window, 0);
    const int first_free = std::max(num_frames - options.window, 1);

    std::vector<int> patch_ids;
    std::vector<std::pair<PatchGraph::EdgeKey, const FlowRevision*>> active;
    for (const auto& [pid, patch] : graph.patches()) {
        if (position.at(patch.source_frame) < window_start) continue;
        bool any = false;
        for (const auto& key : graph.edges_of_patch(pid)) {
            const auto& rev = graph.edges().at(key);
            if (!rev.has_value()) continue;
            active.emplace_back(key, &*rev);
            any = true;
        }
        if (any) patch_ids.push_back(pid);
    }
    if (active.empty()) return false;

    std::map<int, int> pose_index;
    for (int pid : patch_ids) pose_index.emplace(graph.patch(pid).source_frame, 0);
    for (const auto& [key, rev] : active) pose_index.emplace(key.second, 0);
    {
        int slot = 0;
        for (auto& kv : pose_index) kv.second = slot++;
    }
    BAProblem& pr = out.problem;
    pr = BAProblem{};
    pr.intrinsics = graph.intrinsics();
    pr.damping = options.damping;
    out.pose_frames.clear();
    for (const auto& [fi, slot] : pose_index) {
        pr.poses.push_back(graph.frame(fi).pose);
        pr.pose_fixed.push_back(position.at(fi) < first_free);
        out.pose_frames.push_back(fi);
    }
    std::map<int, int> patch_index;
    for (int pid : patch_ids) {
        patch_index[pid] = static_cast<int>(pr.patches.size());
        Patch patch = graph.patch(pid);
        patch.source_frame = pose_index.at(patch.source_frame);
        pr.patches.push_back(std::move(patch));
    }
    out.patch_ids = patch_ids;
    const double margin = 2.0 * kMaxObservableMarginPx;
    for (const auto& [key, rev] : active) {
        const Patch& patch = graph.patch(key.first);
        const PatchReprojection r = reproject_patch(graph.frame(patch.source_frame).pose,
                                                    graph.frame(key.second).pose, graph.intrinsics(), patch);
        const V2 c = r.points[patch.size() / 2];
        const bool observable = !r.behind_camera && c.x > -margin && c.y > -margin &&
                                c.x < graph.image_width() - 1 + margin &&
                                c.y < graph.image_height() - 1 + margin;
        BAEdge e;
        e.patch_id = patch_index.at(key.first);
        e.target_pose = pose_index.at(key.second);
        e.target_point = {c.x + rev->delta.x, c.y + rev->delta.y};
        e.weight = observable ? rev->weight : V2{0, 0};
        pr.edges.push_back(e);
    }
    return true;
}

// bundle_adjust.cpp:225-375
BASolution optimize_window(PatchGraph& graph, const WindowOptions& options) {
    WindowProblem wp;
    if (!build_window_problem(graph, options, wp)) return BASolution{};
    BAProblem& problem = wp.problem;
    BASolution combined;
    combined.num_edges = static_cast<int>(problem.edges.size());
    combined.poses = problem.poses;
    for (const Patch& p : problem.patches) combined.inverse_depths.push_back(p.inverse_depth);

    for (int it = 0; it < options.structure_only_iterations; ++it) {
        BAProblem st = problem;
        st.pose_fixed.assign(st.poses.size(), true);
        const BASolution step = gauss_newton_step(st, nullptr);
        for (size_t k = 0; k < problem.patches.size(); ++k) problem.patches[k].inverse_depth = step.inverse_depths[k];
        combined.inverse_depths = step.inverse_depths;
    }
    for (int it = 0; it < options.iterations; ++it) {
        BASolution step = gauss_newton_step(problem, nullptr);
        if (step.residual_norms.back() > 1.5 * step.residual_norms.front() + 1e-9) {
            bool accepted = false;
            for (double extra = 1e3; extra <= 1e9; extra *= 1e3) {
                problem.damping = options.damping * extra;
                BASolution damped = gauss_newton_step(problem, nullptr);
                if (damped.residual_norms.back() <= 1.5 * damped.residual_norms.front() + 1e-9) {
                    step = damped;
                    accepted = true;
                    break;
                }
            }
            problem.damping = options.damping;
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
    for (size_t slot = 0; slot < wp.pose_frames.size(); ++slot) {
        if (!problem.pose_fixed[slot]) graph.set_pose(wp.pose_frames[slot], combined.poses[slot]);
    }
    for (size_t slot = 0; slot < wp.patch_ids.size(); ++slot) {
        graph.set_inverse_depth(wp.patch_ids[slot], combined.inverse_depths[slot]);
    }
    return combined;
}

}  // namespace orc

// ============================================================================
// extern "C" surface (ctypes), flat arrays.  Pose = 7 doubles (qx qy qz qw tx ty tz).
// ============================================================================
using namespace orc;

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

Pose load_pose(const double* p) { return Pose::raw(Q{p[0], p[1], p[2], p[3]}, V3{p[4], p[5], p[6]}); }
void store_pose(const Pose& p, double* o) {
    o[0] = p.q.x;
    o[1] = p.q.y;
    o[2] = p.q.z;
    o[3] = p.q.w;
    o[4] = p.t.x;
    o[5] = p.t.y;
    o[6] = p.t.z;
}
Intrinsics load_K(const double* k) { return Intrinsics{k[0], k[1], k[2], k[3]}; }
Patch load_patch(int p, const double* x, const double* y, double d, int src) {
    Patch pt;
    pt.width = p;
    pt.source_frame = src;
    pt.inverse_depth = d;
    pt.x.assign(x, x + p * p);
    pt.y.assign(y, y + p * p);
    return pt;
}

// Flat BA problem (same layout as the product C-ABI pvo_ba_problem).
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
        ed.target_point = {e_target[2 * e], e_target[2 * e + 1]};
        ed.weight = {e_weight[2 * e], e_weight[2 * e + 1]};
        pr.edges.push_back(ed);
    }
    pr.intrinsics = load_K(K);
    pr.damping = damping;
    return pr;
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// ---- se3 ----
int orc_se3_exp(const double* xi, double* pose) {
    return guard([&] { store_pose(orc::exp(Tangent{{xi[0], xi[1], xi[2]}, {xi[3], xi[4], xi[5]}}), pose); });
}
int orc_se3_log(const double* pose, double* xi) {
    return guard([&] {
        const Tangent t = orc::log(load_pose(pose));
        const double v[6] = {t.trans.x, t.trans.y, t.trans.z, t.rot.x, t.rot.y, t.rot.z};
        std::memcpy(xi, v, sizeof(v));
    });
}
int orc_se3_compose(const double* a, const double* b, double* out) {
    return guard([&] { store_pose(compose(load_pose(a), load_pose(b)), out); });
}
int orc_se3_inverse(const double* a, double* out) {
    return guard([&] { store_pose(inverse(load_pose(a)), out); });
}
int orc_se3_retract(const double* a, const double* xi, double* out) {
    return guard([&] {
        store_pose(retract(load_pose(a), Tangent{{xi[0], xi[1], xi[2]}, {xi[3], xi[4], xi[5]}}), out);
    });
}
int orc_se3_pose_distance(const double* a, const double* b, double* dist, double* angle) {
    return guard([&] { *dist = pose_distance(load_pose(a), load_pose(b), angle); });
}
// Pose(q, t) constructor: normalizes q (se3.hpp:41).
int orc_se3_make_pose(const double* q_xyzw, const double* t, double* out) {
    return guard([&] {
        store_pose(Pose(Q{q_xyzw[0], q_xyzw[1], q_xyzw[2], q_xyzw[3]}, V3{t[0], t[1], t[2]}), out);
    });
}

// ---- camera ----
int orc_patch_make(double cx, double cy, int width, double inverse_depth, double* x, double* y) {
    return guard([&] {
        const Patch p = make_patch(0, V2{cx, cy}, width, inverse_depth);
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
            out_xy[2 * k] = r.points[k].x;
            out_xy[2 * k + 1] = r.points[k].y;
        }
        *behind = r.behind_camera ? 1 : 0;
    });
}
// out: center(2), d_pose_i(12, row-major 2x6), d_pose_j(12), d_inverse_depth(2)
int orc_reprojection_jacobians(const double* pi, const double* pj, const double* K, int p, const double* x,
                               const double* y, double inv_depth, double* out, int* behind) {
    return guard([&] {
        const Jacobians j =
            reprojection_jacobians(load_pose(pi), load_pose(pj), load_K(K), load_patch(p, x, y, inv_depth, 0));
        out[0] = j.center.x;
        out[1] = j.center.y;
        std::memcpy(out + 2, j.di, sizeof(j.di));
        std::memcpy(out + 14, j.dj, sizeof(j.dj));
        out[26] = j.dd[0];
        out[27] = j.dd[1];
        *behind = j.behind ? 1 : 0;
    });
}

// ---- features / correlation ----
int orc_sample_zero_padded(const float* grid, int w, int h, int c, double x, double y, int ch, double* out) {
    return guard([&] { *out = GridView{grid, w, h, c}.sample_zero_padded(x, y, ch); });
}
int orc_sample_cubic(const float* grid, int w, int h, int c, double x, double y, int ch, double* out) {
    return guard([&] { *out = GridView{grid, w, h, c}.sample_cubic(x, y, ch); });
}
int orc_correlate_at(const float* feature, int channels, const float* grid, int w, int h, double x, double y,
                     double* out) {
    return guard([&] { *out = correlate_at(feature, channels, GridView{grid, w, h, channels}, x, y); });
}
int orc_correlate_at_cubic(const float* feature, int channels, const float* grid, int w, int h, double x,
                           double y, double* out) {
    return guard([&] { *out = correlate_at_cubic(feature, channels, GridView{grid, w, h, channels}, x, y); });
}
int orc_correlate(int p, int channels, const float* feats0, const float* feats1, const float* lvl0, int w0,
                  int h0, const float* lvl1, int w1, int h1, const double* coords, float* out) {
    return guard([&] {
        correlate(p, channels, feats0, feats1, GridView{lvl0, w0, h0, channels}, GridView{lvl1, w1, h1, channels},
                  coords, out);
    });
}
// Batched correlate over edges (host threads).  frames0/frames1: [F][H][W][C];
// patch_feats: [P][2][p*p][C]; coords: [E][p*p][2]; out: [E][2][p*p][49].
int orc_correlate_batch(int n_edges, const int* e_patch, const int* e_frame, const double* coords, int p,
                        int channels, const float* patch_feats, const float* frames0, int w0, int h0,
                        const float* frames1, int w1, int h1, float* out, int threads) {
    return guard([&] {
        const size_t pp = static_cast<size_t>(p) * p;
        const size_t f0 = static_cast<size_t>(w0) * h0 * channels, f1 = static_cast<size_t>(w1) * h1 * channels;
        const size_t out_stride = 2 * pp * kCorrSize * kCorrSize;
        std::vector<std::string> errs(threads > 0 ? threads : 1);
        const int nt = threads > 0 ? threads : 1;
        auto work = [&](int t) {
            try {
                for (int e = t; e < n_edges; e += nt) {
                    const float* g = patch_feats + static_cast<size_t>(e_patch[e]) * 2 * pp * channels;
                    correlate(p, channels, g, g + pp * channels,
                              GridView{frames0 + e_frame[e] * f0, w0, h0, channels},
                              GridView{frames1 + e_frame[e] * f1, w1, h1, channels}, coords + e * pp * 2,
                              out + e * out_stride);
                }
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
    });
}

// CorrelationFlowProvider::propose's per-edge part (flow_provider.cpp:297-312)
// on flattened inputs: centers [E][2] = reproject_patch(...).points[centre],
// behind [E]; patch_feats [P][2][p*p][C]; frames [F][H][W][C].
// Out: delta [E][2], weight [E][2], flags [E] (bit 0 flat, bit 1 out_of_range,
// bit 2 behind the camera).
int orc_measure_batch(int n_edges, const int* e_patch, const int* e_frame, const double* centers,
                      const uint8_t* behind, int p, int channels, const float* patch_feats, const float* frames0,
                      int w0, int h0, const float* frames1, int w1, int h1, double* delta, double* weight,
                      uint8_t* flags, int threads) {
    return guard([&] {
        const size_t pp = static_cast<size_t>(p) * p;
        const size_t f0 = static_cast<size_t>(w0) * h0 * channels, f1 = static_cast<size_t>(w1) * h1 * channels;
        const int nt = threads > 0 ? threads : 1;
        auto work = [&](int t) {
            for (int e = t; e < n_edges; e += nt) {
                Measurement m;
                uint8_t fl = 0;
                if (behind && behind[e]) {
                    fl = 4;  // weight (0.01, 0.01), delta 0 (flow_provider.cpp:301-302)
                } else {
                    const float* g = patch_feats + static_cast<size_t>(e_patch[e]) * 2 * pp * channels;
                    const size_t cp = pp / 2;  // centre pixel (patch.size() / 2)
                    m = measure(g + cp * channels, g + (pp + cp) * channels, channels,
                                GridView{frames0 + e_frame[e] * f0, w0, h0, channels},
                                GridView{frames1 + e_frame[e] * f1, w1, h1, channels},
                                {centers[2 * e], centers[2 * e + 1]});
                    fl = (m.flat ? 1 : 0) | (m.out_of_range ? 2 : 0);
                }
                delta[2 * e] = m.delta.x;
                delta[2 * e + 1] = m.delta.y;
                weight[2 * e] = m.weight.x;
                weight[2 * e + 1] = m.weight.y;
                flags[e] = fl;
            }
        };
        std::vector<std::thread> pool;
        for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
        work(0);
        for (auto& th : pool) th.join();
    });
}

// ---- OracleFlowProvider::propose (flow_provider.cpp:34-93) on a flattened window ----
// gt_poses [N][7] (scene poses of the window's pose slots), gt_d [P] (scene inverse
// depth at each patch centre, flow_provider.cpp:24), the RNG a mt19937_64 seeded
// once per call.  Out: delta [E][2], weight [E][2].
namespace {
struct OracleV2 {  // two-argument construction: the same argument evaluation order as Vec2(a(), b())
    double x, y;
    OracleV2(double a, double b) : x(a), y(b) {}
};
}  // namespace
int orc_oracle_propose(int n_poses, const double* poses, const double* gt_poses, int n_patches, const int* src,
                       const double* px, const double* py, const double* depth, const double* gt_d, int n_edges,
                       const int* e_patch, const int* e_pose, const double* K, double flow_sigma,
                       double outlier_fraction, uint64_t seed, double* delta, double* weight) {
    return guard([&] {
        (void)n_poses;
        (void)n_patches;
        const Intrinsics Kc = load_K(K);
        std::mt19937_64 rng(seed);
        std::normal_distribution<double> gauss(0.0, flow_sigma);
        std::uniform_real_distribution<double> uniform(-32.0, 32.0);
        const double sigma2 = flow_sigma * flow_sigma;
        const double w = std::clamp(1.0 / (1.0 + sigma2), 0.01, 0.99);
        constexpr double kMaxRevisionPx = 64.0;  // flow_provider.hpp:47
        for (int e = 0; e < n_edges; ++e) {
            const int k = e_patch[e], i = src[k], j = e_pose[e];
            Patch cur;
            cur.x.assign(px + 9 * (size_t)k, px + 9 * (size_t)k + 9);
            cur.y.assign(py + 9 * (size_t)k, py + 9 * (size_t)k + 9);
            cur.width = 3;
            cur.inverse_depth = depth[k];
            // ground-truth reprojection of the patch centre (flow_provider.cpp:52-55)
            const Patch probe = make_patch(0, cur.center(), 1, gt_d[k]);
            const PatchReprojection gt =
                reproject_patch(load_pose(gt_poses + 7 * i), load_pose(gt_poses + 7 * j), Kc, probe);
            const PatchReprojection now = reproject_patch(load_pose(poses + 7 * i), load_pose(poses + 7 * j), Kc, cur);
            double dx = 0, dy = 0, wx = 0.01, wy = 0.01;
            if (!(gt.behind_camera || now.behind_camera)) {
                dx = gt.points[0].x - now.points[4].x;
                dy = gt.points[0].y - now.points[4].y;
                if (flow_sigma > 0) {
                    const OracleV2 n(gauss(rng), gauss(rng));
                    dx += n.x;
                    dy += n.y;
                }
                const bool in_range = std::abs(dx) <= kMaxRevisionPx && std::abs(dy) <= kMaxRevisionPx;
                dx = std::clamp(dx, -kMaxRevisionPx, kMaxRevisionPx);
                dy = std::clamp(dy, -kMaxRevisionPx, kMaxRevisionPx);
                wx = wy = in_range ? w : 0.01;
            }
            delta[2 * e] = dx;
            delta[2 * e + 1] = dy;
            weight[2 * e] = wx;
            weight[2 * e + 1] = wy;
        }
        const size_t num_outliers = static_cast<size_t>(outlier_fraction * static_cast<double>(n_edges));
        if (num_outliers > 0) {
            std::vector<size_t> index(n_edges);
            for (size_t i = 0; i < index.size(); ++i) index[i] = i;
            std::shuffle(index.begin(), index.end(), rng);
            for (size_t i = 0; i < num_outliers; ++i) {
                const OracleV2 u(uniform(rng), uniform(rng));
                delta[2 * index[i]] = u.x;
                delta[2 * index[i] + 1] = u.y;
                weight[2 * index[i]] = 0.01;
                weight[2 * index[i] + 1] = 0.01;
            }
        }
    });
}

// ---- feature extraction (features.cpp:55-235) ----
// image [ih][iw] float; level0 [ih/4][iw/4][25 bc], level1 [ih/16][iw/16][25 bc]
int orc_extract_features(const float* image, int iw, int ih, int bc, float* level0, float* level1) {
    return guard([&] {
        if (bc != 1 && bc != 3) throw std::invalid_argument("features: base channel count must be 1 or 3");
        if (iw < 12 || ih < 12) throw std::invalid_argument("features: image too small");
        const int w = iw / 4, h = ih / 4;
        std::vector<float> raw((size_t)w * h), rough((size_t)w * h), res((size_t)w * h), base((size_t)w * h * bc);
        // pool_image: float sums over 4x4 blocks (features.cpp:55-71)
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                float sum = 0;
                for (int dy = 0; dy < 4; ++dy)
                    for (int dx = 0; dx < 4; ++dx) sum += image[(size_t)(4 * y + dy) * iw + 4 * x + dx];
                raw[(size_t)y * w + x] = sum / 16.0f;
            }
        auto clipped = [&](int x, int y, int r, auto&& f) {
            for (int dy = -r; dy <= r; ++dy)
                for (int dx = -r; dx <= r; ++dx) {
                    const int xi = x + dx, yi = y + dy;
                    if (xi < 0 || yi < 0 || xi >= w || yi >= h) continue;
                    f(xi, yi, dx, dy);
                }
        };
        // residual against the clipped 5x5 mean (features.cpp:105-121)
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                double sum = 0;
                int count = 0;
                clipped(x, y, 2, [&](int xi, int yi, int, int) {
                    sum += raw[(size_t)yi * w + xi];
                    ++count;
                });
                rough[(size_t)y * w + x] = raw[(size_t)y * w + x] - static_cast<float>(sum / count);
            }
        // 3x3 binomial smoothing (features.cpp:123-141)
        const double kern[3] = {1, 2, 1};
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                double sum = 0, wt = 0;
                clipped(x, y, 1, [&](int xi, int yi, int dx, int dy) {
                    const double k = kern[dx + 1] * kern[dy + 1];
                    sum += k * rough[(size_t)yi * w + xi];
                    wt += k;
                });
                res[(size_t)y * w + x] = static_cast<float>(sum / wt);
            }
        // local-RMS normalisation (features.cpp:143-160)
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                double sum_sq = 0;
                int count = 0;
                clipped(x, y, 2, [&](int xi, int yi, int, int) {
                    const float r = res[(size_t)yi * w + xi];
                    sum_sq += r * r;
                    ++count;
                });
                const double rms = std::sqrt(sum_sq / count);
                base[((size_t)y * w + x) * bc] = rms > 1e-6 ? res[(size_t)y * w + x] / static_cast<float>(rms) : 0.0f;
            }
        if (bc == 3) {  // central-difference gradients (features.cpp:162-173)
            auto g0 = [&](int x, int y) { return base[((size_t)y * w + x) * 3]; };
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x) {
                    base[((size_t)y * w + x) * 3 + 1] = 0.5f * (g0(std::min(x + 1, w - 1), y) - g0(std::max(x - 1, 0), y));
                    base[((size_t)y * w + x) * 3 + 2] = 0.5f * (g0(x, std::min(y + 1, h - 1)) - g0(x, std::max(y - 1, 0)));
                }
        }
        // lift_neighborhood (features.cpp:177-200)
        auto lift = [&](const std::vector<float>& g, int gw, int gh, float* out) {
            const int C = 25 * bc;
            for (int y = 0; y < gh; ++y)
                for (int x = 0; x < gw; ++x) {
                    float* o = out + ((size_t)y * gw + x) * C;
                    int ch = 0;
                    for (int dy = -2; dy <= 2; ++dy)
                        for (int dx = -2; dx <= 2; ++dx) {
                            const int xi = x + dx, yi = y + dy;
                            const bool in = xi >= 0 && yi >= 0 && xi < gw && yi < gh;
                            for (int c = 0; c < bc; ++c) o[ch++] = in ? g[((size_t)yi * gw + xi) * bc + c] : 0.0f;
                        }
                    double nsq = 0;
                    for (int c = 0; c < C; ++c) nsq += o[c] * o[c];
                    if (nsq > 1e-12) {
                        const float inv = static_cast<float>(1.0 / std::sqrt(nsq));
                        for (int c = 0; c < C; ++c) o[c] *= inv;
                    }
                }
        };
        lift(base, w, h, level0);
        // level 1: pool_features of the base grid, lifted (features.cpp:73-89, :226-231)
        const int w1 = w / 4, h1 = h / 4;
        std::vector<float> pooled((size_t)w1 * h1 * bc);
        for (int y = 0; y < h1; ++y)
            for (int x = 0; x < w1; ++x)
                for (int c = 0; c < bc; ++c) {
                    float sum = 0;
                    for (int dy = 0; dy < 4; ++dy)
                        for (int dx = 0; dx < 4; ++dx) sum += base[((size_t)(4 * y + dy) * w + 4 * x + dx) * bc + c];
                    pooled[((size_t)y * w1 + x) * bc + c] = sum / 16.0f;
                }
        lift(pooled, w1, h1, level1);
    });
}

// crop_patch_features (features.cpp:204-224): out [n][2][9][C]
int orc_crop_patches(int n, const double* px, const double* py, const float* l0, int w0, int h0, const float* l1,
                     int w1, int h1, int C, float* out) {
    return guard([&] {
        const GridView grids[2] = {GridView{l0, w0, h0, C}, GridView{l1, w1, h1, C}};
        for (int p = 0; p < n; ++p)
            for (int level = 0; level < 2; ++level) {
                const double stride = level == 0 ? kFeatureStride : kFeatureStride * kFeatureStride;
                for (int k = 0; k < 9; ++k)
                    for (int c = 0; c < C; ++c)
                        out[(((size_t)p * 2 + level) * 9 + k) * C + c] = static_cast<float>(
                            grids[level].sample_cubic(px[9 * (size_t)p + k] / stride, py[9 * (size_t)p + k] / stride, c));
            }
    });
}

// ---- patch graph ----
void* orc_graph_create(const double* K, int w, int h, int p) {
    try {
        return new PatchGraph(load_K(K), w, h, p);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void orc_graph_destroy(void* g) { delete static_cast<PatchGraph*>(g); }
int orc_graph_add_frame(void* g, double ts, const double* pose, int* out_index) {
    return guard([&] { *out_index = static_cast<PatchGraph*>(g)->add_frame(ts, load_pose(pose)); });
}
int orc_graph_add_patches(void* g, int frame, int n, const double* centroids, const double* depths, int* out_ids) {
    return guard([&] {
        std::vector<V2> c(n);
        for (int i = 0; i < n; ++i) c[i] = {centroids[2 * i], centroids[2 * i + 1]};
        const auto ids = static_cast<PatchGraph*>(g)->add_patches(frame, c, std::vector<double>(depths, depths + n));
        if (out_ids) std::memcpy(out_ids, ids.data(), sizeof(int) * ids.size());
    });
}
int orc_graph_connect(void* g, int radius, int* n_added) {
    return guard([&] { *n_added = static_cast<int>(static_cast<PatchGraph*>(g)->connect(radius).size()); });
}
int orc_graph_remove_frame(void* g, int frame) {
    return guard([&] { static_cast<PatchGraph*>(g)->remove_frame(frame); });
}
int orc_graph_set_revision(void* g, int patch, int frame, const double* delta, const double* weight) {
    return guard([&] {
        static_cast<PatchGraph*>(g)->set_revision({patch, frame},
                                                  FlowRevision{{delta[0], delta[1]}, {weight[0], weight[1]}});
    });
}
int orc_graph_num_edges(void* g) { return static_cast<int>(static_cast<PatchGraph*>(g)->edges().size()); }
int orc_graph_num_frames(void* g) { return static_cast<int>(static_cast<PatchGraph*>(g)->frames().size()); }
int orc_graph_num_patches(void* g) { return static_cast<int>(static_cast<PatchGraph*>(g)->patches().size()); }
// Edges in key order; rev = [E][4] (dx dy wx wy) zeros when unset (dump_edges, patch_graph.cpp:144-151).
int orc_graph_edges(void* g, int* kk, int* jj, double* rev, uint8_t* has_rev) {
    return guard([&] {
        size_t i = 0;
        for (const auto& [key, r] : static_cast<PatchGraph*>(g)->edges()) {
            kk[i] = key.first;
            jj[i] = key.second;
            if (rev) {
                rev[4 * i] = r ? r->delta.x : 0.0;
                rev[4 * i + 1] = r ? r->delta.y : 0.0;
                rev[4 * i + 2] = r ? r->weight.x : 0.0;
                rev[4 * i + 3] = r ? r->weight.y : 0.0;
            }
            if (has_rev) has_rev[i] = r.has_value() ? 1 : 0;
            ++i;
        }
    });
}
int orc_graph_frames(void* g, int* indices, double* poses) {
    return guard([&] {
        size_t i = 0;
        for (const auto& [idx, node] : static_cast<PatchGraph*>(g)->frames()) {
            indices[i] = idx;
            if (poses) store_pose(node.pose, poses + 7 * i);
            ++i;
        }
    });
}
int orc_graph_patches(void* g, int* ids, int* src, double* depth) {
    return guard([&] {
        size_t i = 0;
        for (const auto& [id, p] : static_cast<PatchGraph*>(g)->patches()) {
            ids[i] = id;
            if (src) src[i] = p.source_frame;
            if (depth) depth[i] = p.inverse_depth;
            ++i;
        }
    });
}
int orc_graph_set_pose(void* g, int frame, const double* pose) {
    return guard([&] { static_cast<PatchGraph*>(g)->set_pose(frame, load_pose(pose)); });
}
int orc_graph_set_inverse_depth(void* g, int patch, double d) {
    return guard([&] { static_cast<PatchGraph*>(g)->set_inverse_depth(patch, d); });
}
int orc_graph_active_edges(void* g, int window, int* kk, int* jj, int* n) {
    return guard([&] {
        const auto e = active_edges(*static_cast<PatchGraph*>(g), window);
        *n = static_cast<int>(e.size());
        if (kk)
            for (size_t i = 0; i < e.size(); ++i) {
                kk[i] = e[i].first;
                jj[i] = e[i].second;
            }
    });
}
int orc_graph_build_target(void* g, int patch, int frame, double* out) {
    return guard([&] {
        const V2 t = build_target(*static_cast<PatchGraph*>(g), {patch, frame});
        out[0] = t.x;
        out[1] = t.y;
    });
}

// Flattened window problem (sizes first with null arrays).
int orc_window_problem(void* g, int window, double damping, int* n_poses, int* n_patches, int* n_edges,
                       int* pose_frames, double* poses, uint8_t* fixed, int* patch_ids, int* patch_src,
                       double* patch_x, double* patch_y, double* depth, int* e_patch, int* e_pose,
                       double* e_target, double* e_weight) {
    return guard([&] {
        WindowOptions opt;
        opt.window = window;
        opt.damping = damping;
        WindowProblem wp;
        if (!build_window_problem(*static_cast<PatchGraph*>(g), opt, wp)) {
            *n_poses = *n_patches = *n_edges = 0;
            return;
        }
        const BAProblem& pr = wp.problem;
        *n_poses = static_cast<int>(pr.poses.size());
        *n_patches = static_cast<int>(pr.patches.size());
        *n_edges = static_cast<int>(pr.edges.size());
        if (!pose_frames) return;
        const int pp = pr.patches.empty() ? 0 : pr.patches[0].size();
        for (size_t i = 0; i < pr.poses.size(); ++i) {
            pose_frames[i] = wp.pose_frames[i];
            store_pose(pr.poses[i], poses + 7 * i);
            fixed[i] = pr.pose_fixed[i] ? 1 : 0;
        }
        for (size_t k = 0; k < pr.patches.size(); ++k) {
            patch_ids[k] = wp.patch_ids[k];
            patch_src[k] = pr.patches[k].source_frame;
            std::memcpy(patch_x + k * pp, pr.patches[k].x.data(), sizeof(double) * pp);
            std::memcpy(patch_y + k * pp, pr.patches[k].y.data(), sizeof(double) * pp);
            depth[k] = pr.patches[k].inverse_depth;
        }
        for (size_t e = 0; e < pr.edges.size(); ++e) {
            e_patch[e] = pr.edges[e].patch_id;
            e_pose[e] = pr.edges[e].target_pose;
            e_target[2 * e] = pr.edges[e].target_point.x;
            e_target[2 * e + 1] = pr.edges[e].target_point.y;
            e_weight[2 * e] = pr.edges[e].weight.x;
            e_weight[2 * e + 1] = pr.edges[e].weight.y;
        }
    });
}

// optimize_window on the oracle graph (mutates it).  residual_norms needs
// room for 1 + iterations entries.
int orc_optimize_window(void* g, int window, int iterations, int structure_only, double damping,
                        double* residual_norms, int* n_norms, int* num_edges) {
    return guard([&] {
        WindowOptions opt;
        opt.window = window;
        opt.iterations = iterations;
        opt.structure_only_iterations = structure_only;
        opt.damping = damping;
        const BASolution s = optimize_window(*static_cast<PatchGraph*>(g), opt);
        *n_norms = static_cast<int>(s.residual_norms.size());
        for (size_t i = 0; i < s.residual_norms.size(); ++i) residual_norms[i] = s.residual_norms[i];
        *num_edges = s.num_edges;
    });
}

// optimize_window on a flattened problem (the graph-free core of
// bundle_adjust.cpp:309-366), for direct parity with the product's
// pvo_ba_window entry.  Outputs poses/depths after the iterations.
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
            const BASolution step = gauss_newton_step(st, nullptr);
            for (size_t k = 0; k < problem.patches.size(); ++k) problem.patches[k].inverse_depth = step.inverse_depths[k];
            combined.inverse_depths = step.inverse_depths;
        }
        for (int it = 0; it < iterations; ++it) {
            BASolution step = gauss_newton_step(problem, nullptr);
            if (step.residual_norms.back() > 1.5 * step.residual_norms.front() + 1e-9) {
                bool accepted = false;
                for (double extra = 1e3; extra <= 1e9; extra *= 1e3) {
                    problem.damping = damping * extra;
                    BASolution damped = gauss_newton_step(problem, nullptr);
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

// gauss_newton_step on a flattened problem; optional dense H ((np+nd)^2) and b capture.
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
        if (debug_h) std::memcpy(debug_h, ne.h.a.data(), sizeof(double) * ne.h.a.size());
        if (debug_b) std::memcpy(debug_b, ne.b.data(), sizeof(double) * ne.b.size());
    });
}

// schur_solve on dense row-major inputs.
int orc_schur_solve(int np, int nd, const double* hpp, const double* hpd, const double* hdd, const double* bp,
                    const double* bd, double* dp, double* dd) {
    return guard([&] {
        Dense a(np, np), b(np, nd);
        std::memcpy(a.a.data(), hpp, sizeof(double) * np * np);
        std::memcpy(b.a.data(), hpd, sizeof(double) * np * nd);
        const SchurResult r = schur_solve(a, b, std::vector<double>(hdd, hdd + nd), std::vector<double>(bp, bp + np),
                                          std::vector<double>(bd, bd + nd));
        if (np > 0) std::memcpy(dp, r.pose_delta.data(), sizeof(double) * np);
        std::memcpy(dd, r.depth_delta.data(), sizeof(double) * nd);
    });
}

// Eigen LDLT solve on its own (for pinning the restatement against scipy).
int orc_ldlt_solve(int n, const double* a, const double* rhs, double* x, int* ok) {
    return guard([&] {
        Dense m(n, n);
        std::memcpy(m.a.data(), a, sizeof(double) * n * n);
        std::vector<double> out;
        *ok = ldlt_solve(m, std::vector<double>(rhs, rhs + n), out) ? 1 : 0;
        std::memcpy(x, out.data(), sizeof(double) * n);
    });
}

// ---- timing entries for bench.py's CPU legs (test infrastructure) ----
// The per-iteration correlation work of the reference's pipeline over a flat
// window: for every edge reproject_patch (camera.cpp:47-71) then correlate
// (correlation.cpp:37-71), edges split over `threads` host threads.  Inputs are
// staged before the clock starts (the pipeline keeps patches, descriptors and
// pyramids resident); *seconds = wall time of the edge loop only.
int orc_bench_corr(int n_poses, const double* poses, int n_patches, int p, const int* src, const double* px,
                   const double* py, const double* depth, int n_edges, const int* e_patch, const int* e_pose,
                   const int* e_frame, const double* K, int channels, const float* patch_feats,
                   const float* frames0, int w0, int h0, const float* frames1, int w1, int h1, int threads,
                   double* seconds) {
    return guard([&] {
        std::vector<Pose> P;
        for (int i = 0; i < n_poses; ++i) P.push_back(load_pose(poses + 7 * i));
        std::vector<Patch> pt;
        for (int k = 0; k < n_patches; ++k) pt.push_back(load_patch(p, px + k * p * p, py + k * p * p, depth[k], src[k]));
        const Intrinsics Kc = load_K(K);
        const size_t pp = static_cast<size_t>(p) * p;
        const size_t f0 = static_cast<size_t>(w0) * h0 * channels, f1 = static_cast<size_t>(w1) * h1 * channels;
        std::vector<float> out(static_cast<size_t>(n_edges) * 2 * pp * kCorrSize * kCorrSize);
        const int nt = threads > 0 ? threads : 1;
        const auto t0 = std::chrono::steady_clock::now();
        auto work = [&](int t) {
            for (int e = t; e < n_edges; e += nt) {
                const Patch& patch = pt[e_patch[e]];
                const PatchReprojection r = reproject_patch(P[patch.source_frame], P[e_pose[e]], Kc, patch);
                std::vector<double> c(2 * pp);
                for (size_t k = 0; k < pp; ++k) c[2 * k] = r.points[k].x, c[2 * k + 1] = r.points[k].y;
                const float* g = patch_feats + static_cast<size_t>(e_patch[e]) * 2 * pp * channels;
                correlate(p, channels, g, g + pp * channels, GridView{frames0 + e_frame[e] * f0, w0, h0, channels},
                          GridView{frames1 + e_frame[e] * f1, w1, h1, channels}, c.data(),
                          out.data() + static_cast<size_t>(e) * 2 * pp * kCorrSize * kCorrSize);
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
        PatchGraph copy = *static_cast<PatchGraph*>(g);
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

