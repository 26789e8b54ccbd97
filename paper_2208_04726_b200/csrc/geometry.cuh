// geometry.cuh — FP64 SE(3) + pinhole geometry shared by host and device.
//
// One definition compiled twice (host C++ and sm_100a device code) so the
// host-side window flattening and every kernel evaluate the same formulas.
// Follows the reference's conventions:
//   pose = world->camera, quaternion coefficients (x, y, z, w) + t
//       (se3.hpp:38-61, Eigen coeff order)
//   compose(a, b) = (qa qb, qa tb + ta), normalized in the Pose ctor
//       (se3.cpp:82-84, se3.hpp:41)
//   inverse(a) = (conj qa, -(conj qa) ta)                    (se3.cpp:86-89)
//   exp with the theta < 1e-8 branch                         (se3.cpp:28-50)
//   retract(a, xi) = exp(xi) a, xi = (trans, rot)            (se3.cpp:91-93)
//   reproject_patch with the bitwise-equal-pose shortcut     (camera.cpp:47-71)
//   reprojection_jacobians, no shortcut                      (camera.cpp:73-108)
// Quaternion arithmetic follows Eigen's scalar formulas.
#pragma once

#include <cmath>
#include <cstdint>

#if defined(__CUDACC__)
#define PVO_HD __host__ __device__ __forceinline__
#if defined(__CUDA_ARCH__)
#define PVO_UNROLL _Pragma("unroll")
#else
#define PVO_UNROLL
#endif
#else
#define PVO_HD inline
#define PVO_UNROLL
#endif

namespace pvo_dev {

constexpr double kDepthEpsilon = 1e-6;   // camera.hpp:43
constexpr double kSmallAngle = 1e-8;     // se3.cpp:10

struct Quat {
    double x, y, z, w;
};
struct Vec3 {
    double x, y, z;
};
struct SE3 {
    Quat q;
    Vec3 t;
};
struct Cam {
    double fx, fy, cx, cy;
};

PVO_HD Vec3 v_add(Vec3 a, Vec3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
PVO_HD Vec3 v_scale(double s, Vec3 a) { return {s * a.x, s * a.y, s * a.z}; }
PVO_HD Vec3 v_cross(Vec3 a, Vec3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

PVO_HD Quat q_normalized(Quat q) {
    const double n2 = q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w;
    if (n2 > 0) {
        const double n = sqrt(n2);
        return {q.x / n, q.y / n, q.z / n, q.w / n};
    }
    return q;
}
PVO_HD Quat q_mul(Quat a, Quat b) {
    return {a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
            a.w * b.y + a.y * b.w + a.z * b.x - a.x * b.z,
            a.w * b.z + a.z * b.w + a.x * b.y - a.y * b.x,
            a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z};
}
// q * v: uv = 2 (vec x v); v + w uv + vec x uv
PVO_HD Vec3 q_rotate(Quat q, Vec3 v) {
    const Vec3 vec{q.x, q.y, q.z};
    Vec3 uv = v_cross(vec, v);
    uv = v_add(uv, uv);
    return v_add(v_add(v, v_scale(q.w, uv)), v_cross(vec, uv));
}
// Row-major 3x3 rotation matrix (Quaternion::toRotationMatrix).
PVO_HD void q_matrix(Quat q, double r[9]) {
    const double tx = 2 * q.x, ty = 2 * q.y, tz = 2 * q.z;
    const double twx = tx * q.w, twy = ty * q.w, twz = tz * q.w;
    const double txx = tx * q.x, txy = ty * q.x, txz = tz * q.x;
    const double tyy = ty * q.y, tyz = tz * q.y, tzz = tz * q.z;
    r[0] = 1 - (tyy + tzz);
    r[1] = txy - twz;
    r[2] = txz + twy;
    r[3] = txy + twz;
    r[4] = 1 - (txx + tzz);
    r[5] = tyz - twx;
    r[6] = txz - twy;
    r[7] = tyz + twx;
    r[8] = 1 - (txx + tyy);
}

PVO_HD SE3 se3_load(const double* p) { return {{p[0], p[1], p[2], p[3]}, {p[4], p[5], p[6]}}; }
PVO_HD void se3_store(const SE3& a, double* p) {
    p[0] = a.q.x;
    p[1] = a.q.y;
    p[2] = a.q.z;
    p[3] = a.q.w;
    p[4] = a.t.x;
    p[5] = a.t.y;
    p[6] = a.t.z;
}
// Pose(q, t) constructor semantics: q is normalized.
PVO_HD SE3 se3_make(Quat q, Vec3 t) { return {q_normalized(q), t}; }
PVO_HD SE3 se3_compose(const SE3& a, const SE3& b) {
    return se3_make(q_mul(a.q, b.q), v_add(q_rotate(a.q, b.t), a.t));
}
PVO_HD SE3 se3_inverse(const SE3& a) {
    const Quat qi{-a.q.x, -a.q.y, -a.q.z, a.q.w};
    return se3_make(qi, v_scale(-1.0, q_rotate(qi, a.t)));
}
PVO_HD bool se3_equal(const SE3& a, const SE3& b) {
    return a.q.x == b.q.x && a.q.y == b.q.y && a.q.z == b.q.z && a.q.w == b.q.w && a.t.x == b.t.x &&
           a.t.y == b.t.y && a.t.z == b.t.z;
}

// exp of xi = (tx, ty, tz, wx, wy, wz).  V = I + a W + b W^2 applied to the
// translation without forming W^2 explicitly would change rounding; we form
// the 3x3 like the reference.
PVO_HD SE3 se3_exp(const double xi[6]) {
    const double ox = xi[3], oy = xi[4], oz = xi[5];
    const double theta2 = ox * ox + oy * oy + oz * oz;
    const double theta = sqrt(theta2);
    Quat q;
    double a, b;
    if (theta < kSmallAngle) {
        q = {0.5 * ox, 0.5 * oy, 0.5 * oz, 1.0};
        a = 0.5;
        b = 1.0 / 6.0;
    } else {
        const double half = 0.5 * theta;
        double sh, ch, st, ct;
#if defined(__CUDA_ARCH__)
        sincos(half, &sh, &ch);  // one argument reduction per angle (same values as sin / cos)
        sincos(theta, &st, &ct);
#else
        sh = sin(half);
        ch = cos(half);
        st = sin(theta);
        ct = cos(theta);
#endif
        const double s = sh / theta;
        q = {s * ox, s * oy, s * oz, ch};
        a = (1.0 - ct) / theta2;
        b = (theta - st) / (theta2 * theta);
    }
    // W = skew(omega); W^2 entries
    const double w[9] = {0, -oz, oy, oz, 0, -ox, -oy, ox, 0};
    double v[9];
PVO_UNROLL
    for (int i = 0; i < 3; ++i) {
PVO_UNROLL
        for (int j = 0; j < 3; ++j) {
            const double ww = w[3 * i] * w[j] + w[3 * i + 1] * w[3 + j] + w[3 * i + 2] * w[6 + j];
            v[3 * i + j] = (i == j ? 1.0 : 0.0) + a * w[3 * i + j] + b * ww;
        }
    }
    const Vec3 t{v[0] * xi[0] + v[1] * xi[1] + v[2] * xi[2], v[3] * xi[0] + v[4] * xi[1] + v[5] * xi[2],
                 v[6] * xi[0] + v[7] * xi[1] + v[8] * xi[2]};
    return se3_make(q, t);
}
PVO_HD SE3 se3_retract(const SE3& a, const double xi[6]) { return se3_compose(se3_exp(xi), a); }

// Relative pose T_j T_i^-1 as rotation matrix + translation (camera.cpp:59-61).
struct Relative {
    double r[9];
    Vec3 t;
};
PVO_HD Relative relative_pose(const SE3& pi, const SE3& pj) {
    const SE3 rel = se3_compose(pj, se3_inverse(pi));
    Relative out;
    q_matrix(rel.q, out.r);
    out.t = rel.t;
    return out;
}

// Reprojection of one point with a precomputed relative pose.  Returns q.z
// (for the behind-camera test) and writes the pixel.
PVO_HD double reproject_point(const Relative& rel, const Cam& K, double inv_depth, double px, double py,
                              double* u, double* v) {
    const double rx = (px - K.cx) / K.fx, ry = (py - K.cy) / K.fy;
    const double qx = rel.r[0] * rx + rel.r[1] * ry + rel.r[2] + rel.t.x * inv_depth;
    const double qy = rel.r[3] * rx + rel.r[4] * ry + rel.r[5] + rel.t.y * inv_depth;
    const double qz = rel.r[6] * rx + rel.r[7] * ry + rel.r[8] + rel.t.z * inv_depth;
    const double z = qz > kDepthEpsilon ? qz : kDepthEpsilon;
    *u = K.fx * qx / z + K.cx;
    *v = K.fy * qy / z + K.cy;
    return qz;
}

// Analytic Jacobians of the dehomogenized patch center (camera.cpp:73-108).
// di/dj are row-major 2x6, dd is 2x1.
struct CenterJac {
    double cu, cv;
    double di[12], dj[12], dd[2];
    bool behind;
};
PVO_HD CenterJac center_jacobians(const Relative& rel, const Cam& K, double d, double cxp, double cyp) {
    const double* r = rel.r;
    const Vec3 ray{(cxp - K.cx) / K.fx, (cyp - K.cy) / K.fy, 1.0};
    const double qx = r[0] * ray.x + r[1] * ray.y + r[2] * ray.z + rel.t.x * d;
    const double qy = r[3] * ray.x + r[4] * ray.y + r[5] * ray.z + rel.t.y * d;
    const double qz = r[6] * ray.x + r[7] * ray.y + r[8] * ray.z + rel.t.z * d;
    CenterJac j;
    j.behind = qz <= kDepthEpsilon;
    const double z = qz > kDepthEpsilon ? qz : kDepthEpsilon;
    j.cu = K.fx * qx / z + K.cx;
    j.cv = K.fy * qy / z + K.cy;
    const double P[2][3] = {{K.fx / z, 0.0, -K.fx * qx / (z * z)}, {0.0, K.fy / z, -K.fy * qy / (z * z)}};
    // dq/dxi_j = [d I | -[q]x]
    const double Aj[3][6] = {{d, 0, 0, 0, qz, -qy}, {0, d, 0, -qz, 0, qx}, {0, 0, d, qy, -qx, 0}};
    // dq/dxi_i = [-d R | R [ray]x]
    const double sr[9] = {0, -ray.z, ray.y, ray.z, 0, -ray.x, -ray.y, ray.x, 0};
    double Ai[3][6];
PVO_UNROLL
    for (int m = 0; m < 3; ++m) {
PVO_UNROLL
        for (int c = 0; c < 3; ++c) {
            Ai[m][c] = -d * r[3 * m + c];
            Ai[m][3 + c] = r[3 * m] * sr[c] + r[3 * m + 1] * sr[3 + c] + r[3 * m + 2] * sr[6 + c];
        }
    }
PVO_UNROLL
    for (int row = 0; row < 2; ++row) {
PVO_UNROLL
        for (int c = 0; c < 6; ++c) {
            j.dj[6 * row + c] = P[row][0] * Aj[0][c] + P[row][1] * Aj[1][c] + P[row][2] * Aj[2][c];
            j.di[6 * row + c] = P[row][0] * Ai[0][c] + P[row][1] * Ai[1][c] + P[row][2] * Ai[2][c];
        }
        j.dd[row] = P[row][0] * rel.t.x + P[row][1] * rel.t.y + P[row][2] * rel.t.z;
    }
    return j;
}

}  // namespace pvo_dev
