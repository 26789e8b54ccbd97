// ba_common.cuh — device helpers shared by the window BA kernels (ba.cu:
// the persistent single-kernel path, ba_large.cu: the multi-kernel path for
// large pose systems).
#pragma once

#include "geometry.cuh"
#include "kernels.cuh"

namespace pvo_dev {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

__device__ inline void set_status(int* status, int code) { atomicOr(status, 1 << code); }

// Reprojected center + behind flag with reproject_patch semantics
// (camera.cpp:47-71): bitwise-equal shortcut, behind if ANY pixel's q_z <= eps.
__device__ inline void reproject_center(const SE3& pi, const SE3& pj, const Cam& K, const double* px,
                                        const double* py, double d, double* cu, double* cv, bool* behind) {
    if (se3_equal(pi, pj)) {
        *cu = px[4];
        *cv = py[4];
        *behind = false;
        return;
    }
    const Relative rel = relative_pose(pi, pj);
    bool b = false;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        double u, v;
        const double qz = reproject_point(rel, K, d, px[k], py[k], &u, &v);
        if (qz <= kDepthEpsilon) b = true;
        if (k == 4) {
            *cu = u;
            *cv = v;
        }
    }
    *behind = b;
}

// reproject_patch of a 1x1 patch at (cx, cy) with inverse depth d (the oracle
// provider's probe, flow_provider.cpp:52-55): the bitwise-equal shortcut, else
// the pixel's reprojection and its own behind flag
__device__ inline void reproject_center_probe(const SE3& pi, const SE3& pj, const Cam& K, double cx, double cy,
                                              double d, double* cu, double* cv, bool* behind) {
    if (se3_equal(pi, pj)) {
        *cu = cx;
        *cv = cy;
        *behind = false;
        return;
    }
    const Relative rel = relative_pose(pi, pj);
    const double qz = reproject_point(rel, K, d, cx, cy, cu, cv);
    *behind = qz <= kDepthEpsilon;
}

// Per-pose rotation matrix + translation, so that a relative pose is a 3x3
// product instead of two quaternion normalisations per edge:
//   T_j T_i^-1 = (R_j R_i^T, t_j - R_j R_i^T t_i)   (camera.cpp:59-61)
__device__ inline void pose_mats(const double* poses, double* mats, int n) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const SE3 p = se3_load(poses + 7 * i);
        q_matrix(p.q, mats + 12 * i);
        mats[12 * i + 9] = p.t.x;
        mats[12 * i + 10] = p.t.y;
        mats[12 * i + 11] = p.t.z;
    }
}
__device__ __forceinline__ Relative rel_from_mats(const double* Mi, const double* Mj) {
    Relative r;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
            r.r[3 * a + b] = Mj[3 * a] * Mi[3 * b] + Mj[3 * a + 1] * Mi[3 * b + 1] + Mj[3 * a + 2] * Mi[3 * b + 2];
    const double ti0 = Mi[9], ti1 = Mi[10], ti2 = Mi[11];
    r.t.x = Mj[9] - (r.r[0] * ti0 + r.r[1] * ti1 + r.r[2] * ti2);
    r.t.y = Mj[10] - (r.r[3] * ti0 + r.r[4] * ti1 + r.r[5] * ti2);
    r.t.z = Mj[11] - (r.r[6] * ti0 + r.r[7] * ti1 + r.r[8] * ti2);
    return r;
}
// reproject_patch center + behind flag (camera.cpp:47-71) from a relative
// pose: the shortcut when the two poses are bitwise equal, otherwise behind
// if ANY of the 9 pixels has q_z <= eps (no division except the centre's).
__device__ __forceinline__ void center_behind(bool equal, const Relative& rel, const Cam& K, const double* px,
                                              const double* py, double d, double* cu, double* cv, bool* behind) {
    if (equal) {
        *cu = px[4];
        *cv = py[4];
        *behind = false;
        return;
    }
    bool b = false;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        if (k == 4) {
            double u, v;
            const double qz = reproject_point(rel, K, d, px[k], py[k], &u, &v);
            *cu = u;
            *cv = v;
            b = b || qz <= kDepthEpsilon;
        } else {
            const double rx = (px[k] - K.cx) / K.fx, ry = (py[k] - K.cy) / K.fy;
            const double qz = rel.r[6] * rx + rel.r[7] * ry + rel.r[8] + rel.t.z * d;
            b = b || qz <= kDepthEpsilon;
        }
    }
    *behind = b;
}

// ---------------------------------------------------------------------------
// Frozen target + effective weight of edge e (bundle_adjust.cpp:288-307):
// target = center(reproject_patch) + delta; weight 0 if behind the camera or
// the centre is outside the image +- 2 * kMaxObservableMarginPx.
// ---------------------------------------------------------------------------
__device__ inline void freeze_edge(const BAParams& a, const double* poses, int e) {
    const Cam K{a.K[0], a.K[1], a.K[2], a.K[3]};
    const double margin = 2.0 * 32.0;  // 2 * kMaxObservableMarginPx (bundle_adjust.hpp:18)
    {
        if (!a.freeze_targets) {
            a.e_target[2 * e] = a.e_in[2 * e];
            a.e_target[2 * e + 1] = a.e_in[2 * e + 1];
            a.e_weight[2 * e] = a.e_weight_in[2 * e];
            a.e_weight[2 * e + 1] = a.e_weight_in[2 * e + 1];
            return;
        }
        const int k = a.e_patch[e];
        const SE3 pi = se3_load(poses + 7 * a.patch_src[k]);
        const SE3 pj = se3_load(poses + 7 * a.e_pose[e]);
        double cu, cv;
        bool behind;
        reproject_center(pi, pj, K, a.patch_x + 9 * (size_t)k, a.patch_y + 9 * (size_t)k, a.depth[k], &cu, &cv,
                         &behind);
        const bool observable = !behind && cu > -margin && cv > -margin && cu < a.image_w - 1 + margin &&
                                cv < a.image_h - 1 + margin;
        a.e_target[2 * e] = cu + a.e_in[2 * e];
        a.e_target[2 * e + 1] = cv + a.e_in[2 * e + 1];
        a.e_weight[2 * e] = observable ? a.e_weight_in[2 * e] : 0.0;
        a.e_weight[2 * e + 1] = observable ? a.e_weight_in[2 * e + 1] : 0.0;
    }
}


}  // namespace pvo_dev
