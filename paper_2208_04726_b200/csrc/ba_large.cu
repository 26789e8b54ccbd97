// ba_large.cu — bundle adjustment of a window whose pose system is too large
// for the single persistent kernel of ba.cu (more than 16 free poses or 128
// poses: BASELINE config 4, 63 free poses -> a 378 x 378 reduced system,
// 32,768 patches, 404,480 edges), sm_100a, FP64.
//
// Same mathematics as ba.cu / the reference (bundle_adjust.cpp:62-375):
// frozen targets, per-edge Jacobians (camera.cpp:73-108), Schur elimination of
// the depth block, LDL^T of the reduced pose system, retraction, clamped depth
// back-substitution, weighted residual norms and the divergence guard.  The
// organisation changes with the scale:
//
//  * patches are cut into GROUPS: runs of consecutive patches with the same
//    source pose, <= 64 patches each.  All edges of a run touch a contiguous
//    band of free pose slots (the patch graph only connects frames within the
//    graph radius, patch_graph.cpp:79), so each group accumulates its part of
//    the reduced system S = sum_e J~^T W J~ - v_k v_k^T / h_k into a small
//    LOCAL block (<= 25 poses = 150 dims) in shared memory, entry-owned by the
//    CTA's threads in patch order (deterministic, no atomics);
//  * an entry-parallel kernel sums the group blocks into the dense S (fixed
//    group order) and adds the damping;
//  * one CTA factors S with a blocked (32) right-looking LDL^T restricted to
//    the band (half-bandwidth = widest group window - 1; without pivoting
//    there is no fill-in outside the band: 5x fewer flops than dense at
//    config 4), the rhs carried as an extra row (forward substitution for
//    free), 4x4 register-tiled trailing updates, then a blocked banded
//    back-substitution and the retraction.  Unlike ba.cu it keeps the natural
//    order instead of Eigen's diagonal pivoting: a symmetric permutation of an
//    SPD system, the same solution up to rounding (tested against the oracle,
//    which follows Eigen), and pivoting would destroy the band;
//  * depth back-substitution + residual at the candidate state, then a
//    one-CTA guard kernel that accepts / retries with heavier damping / skips,
//    exactly as bundle_adjust.cpp:327-366.  Later attempts of an iteration
//    are enqueued up front and exit at once when the guard is settled
//    (control word on the device): no host synchronisation in the loop.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "ba_common.cuh"
#include "kernels.cuh"

namespace pvo_dev {

namespace {

constexpr int kT = 256;  // assemble / update CTA size
constexpr int kW = kT / 32;
constexpr int kMaxE = 32;       // edges per patch (lane per edge)
constexpr int kRec = 30;        // doubles per edge record: Gs[12] Jt[12] Jd[2] r[2] w[2]
constexpr int kGs = 0, kJt = 12, kJd = 24, kR = 26, kWt = 28;
constexpr int kScal = 40;       // per-warp scalars: h, bd, 1/h, pad, 6x6 source block
constexpr int kST = 256;        // solver CTA size (255 registers: the panel row lives in registers)
constexpr int kB = 32;          // solver block size

__host__ __device__ inline int nent(int n) { return n * (n + 1) / 2; }
__host__ __device__ inline int a16(int x) { return (x + 15) & ~15; }

struct ALayout {
    int S, rhs, tab, rec, vb, sc, wi, wr, total;
};
__host__ __device__ inline ALayout assemble_layout(int nl) {
    ALayout L;
    int o = 0;
    L.S = o;
    o = a16(o + 8 * nent(nl));
    L.rhs = o;
    o = a16(o + 8 * (nl > 0 ? nl : 1));
    L.rec = o;
    o = a16(o + 8 * kW * kMaxE * kRec);
    L.vb = o;
    o = a16(o + 8 * kW * 2 * (nl > 0 ? nl : 1));
    L.sc = o;
    o = a16(o + 8 * kW * kScal);
    L.wr = o;
    o = a16(o + 8 * kW * 2);
    L.tab = o;
    o = a16(o + 4 * nent(nl));
    L.wi = o;
    o = a16(o + 4 * kW * (4 + kMaxLocalPoses + kMaxE));
    L.total = o;
    return L;
}

__device__ __forceinline__ double damping_of(double base, int attempt) {
    return attempt == 0 ? base : base * (attempt == 1 ? 1e3 : attempt == 2 ? 1e6 : 1e9);
}

// ---------------------------------------------------------------------------
// init: frozen targets of every edge + rotation matrices of the current poses
// ---------------------------------------------------------------------------
__global__ void bal_init_kernel(BALargeParams P) {
    const BAParams& a = P.a;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < a.n_edges; e += gridDim.x * blockDim.x)
        freeze_edge(a, a.poses, e);
    if (blockIdx.x == 0) pose_mats(a.poses, P.mats, a.n_poses);
}

// ---------------------------------------------------------------------------
// assemble: one CTA per group -> local Schur block, local rhs, residual sums
// at the current state, per-patch (v_k, h_k, b_dk) for the back-substitution.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kT) bal_assemble_kernel(BALargeParams P, int structure) {
    if (P.ctrl[0] || P.ctrl[2]) return;
    extern __shared__ __align__(16) unsigned char smem[];
    const BAParams& a = P.a;
    const double lambda = damping_of(a.damping, P.ctrl[1]);
    const int g = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int k0 = P.g_begin[g], k1 = P.g_begin[g + 1];
    const int lo = P.g_lo[g];
    const int nl = structure ? 0 : P.g_nl[g];
    const int ne_l = nent(nl);
    const ALayout L = assemble_layout(nl);
    double* S = reinterpret_cast<double*>(smem + L.S);
    double* rhs = reinterpret_cast<double*>(smem + L.rhs);
    unsigned* tab = reinterpret_cast<unsigned*>(smem + L.tab);
    const Cam K{a.K[0], a.K[1], a.K[2], a.K[3]};
    for (int i = tid; i < ne_l; i += kT) {
        S[i] = 0.0;
        int ia = 0, rowlen = nl, base = 0;
        while (i >= base + rowlen) {
            base += rowlen;
            --rowlen;
            ++ia;
        }
        const int ib = ia + i - base;
        tab[i] = (unsigned)ia | ((unsigned)ib << 8) | ((unsigned)(ia / 6) << 16) | ((unsigned)(ib / 6) << 24);
    }
    for (int i = tid; i < nl; i += kT) rhs[i] = 0.0;
    double wr_sum = 0.0, wr_w = 0.0;
    __syncthreads();

    for (int batch = k0; batch < k1; batch += kW) {
        const int k = batch + warp;
        int* wi = reinterpret_cast<int*>(smem + L.wi) + warp * (4 + kMaxLocalPoses + kMaxE);
        double* rec = reinterpret_cast<double*>(smem + L.rec) + (size_t)warp * kMaxE * kRec;
        double* v = reinterpret_cast<double*>(smem + L.vb) + (size_t)warp * 2 * (nl > 0 ? nl : 1);
        double* bvec = v + nl;
        double* sc = reinterpret_cast<double*>(smem + L.sc) + warp * kScal;
        if (k < k1) {
            const int eb = a.patch_edge_begin[k], ne = a.patch_edge_begin[k + 1] - eb;
            const int src = a.patch_src[k];
            const int fsrc = a.pose_free_slot[src];
            const int si = (structure || fsrc < 0) ? -1 : fsrc - lo;
            const int dslot = a.depth_slot[k];
            const double d = a.depth[k];
            const double* px = a.patch_x + 9 * (size_t)k;
            const double* py = a.patch_y + 9 * (size_t)k;
            for (int i = lane; i < 2 * nl; i += 32) v[i] = 0.0;
            double h = 0, bd = 0, vs[6] = {0, 0, 0, 0, 0, 0}, bs[6] = {0, 0, 0, 0, 0, 0};
            int sj = -1;
            double wrs = 0, wrw = 0;
            if (lane < ne) {
                const int e = eb + lane;
                const int tgt = a.e_pose[e];
                const int ft = a.pose_free_slot[tgt];
                sj = (structure || ft < 0) ? -1 : ft - lo;
                const SE3 pi = se3_load(a.poses + 7 * src);
                const SE3 pj = se3_load(a.poses + 7 * tgt);
                const Relative rel = rel_from_mats(P.mats + 12 * src, P.mats + 12 * tgt);
                const CenterJac J = center_jacobians(rel, K, d, px[4], py[4]);
                const double r0 = J.cu - a.e_target[2 * e], r1 = J.cv - a.e_target[2 * e + 1];
                if (!isfinite(r0) || !isfinite(r1)) set_status(a.status, kDevNonFiniteResidual);
                double w0 = J.behind ? 0.0 : a.e_weight[2 * e];
                double w1 = J.behind ? 0.0 : a.e_weight[2 * e + 1];
                const bool active = !(w0 == 0.0 && w1 == 0.0);  // bundle_adjust.cpp:151
                if (!active) {
                    w0 = 0.0;
                    w1 = 0.0;
                }
                double* R = rec + lane * kRec;
#pragma unroll
                for (int c = 0; c < 12; ++c) {
                    const double gs = J.di[c] + ((sj >= 0 && sj == si) ? J.dj[c] : 0.0);
                    R[kGs + c] = active ? gs : 0.0;
                    R[kJt + c] = active ? J.dj[c] : 0.0;
                }
                R[kJd] = active ? J.dd[0] : 0.0;
                R[kJd + 1] = active ? J.dd[1] : 0.0;
                R[kR] = active ? r0 : 0.0;
                R[kR + 1] = active ? r1 : 0.0;
                R[kWt] = w0;
                R[kWt + 1] = w1;
                if (active) {
                    const double t0 = J.dd[0] * w0, t1 = J.dd[1] * w1;
                    h = t0 * J.dd[0] + t1 * J.dd[1];
                    bd = -(t0 * r0 + t1 * r1);
#pragma unroll
                    for (int c = 0; c < 6; ++c) {
                        const double g0 = R[kGs + c] * w0, g1 = R[kGs + 6 + c] * w1;
                        vs[c] = g0 * J.dd[0] + g1 * J.dd[1];
                        bs[c] = -(g0 * r0 + g1 * r1);
                    }
                }
                if (!active || sj == si) sj = -1;  // no separate target block
                // weighted_residual_norm term at the current state (bundle_adjust.cpp:99-113)
                double cu, cv;
                bool behind;
                center_behind(se3_equal(pi, pj), rel, K, px, py, d, &cu, &cv, &behind);
                const double rx = cu - a.e_target[2 * e], ry = cv - a.e_target[2 * e + 1];
                const double wx = behind ? 0.0 : a.e_weight[2 * e];
                const double wy = behind ? 0.0 : a.e_weight[2 * e + 1];
                wrs = wx * rx * rx + wy * ry * ry;
                wrw = wx + wy;
            }
            __syncwarp();
            if (si >= 0 && lane < 21) {  // 6x6 source block sum_e Gs^T W Gs (upper, mirrored)
                int ra = 0, rem = lane;
                while (rem >= 6 - ra) {
                    rem -= 6 - ra;
                    ++ra;
                }
                const int rb = ra + rem;
                double val = 0.0;
                for (int l = 0; l < ne; ++l) {
                    const double* R = rec + l * kRec;
                    val += (R[kGs + ra] * R[kWt]) * R[kGs + rb] + (R[kGs + 6 + ra] * R[kWt + 1]) * R[kGs + 6 + rb];
                }
                sc[4 + 6 * ra + rb] = val;
                sc[4 + 6 * rb + ra] = val;
            }
            h = warp_sum(h);
            bd = warp_sum(bd);
            wrs = warp_sum(wrs);
            wrw = warp_sum(wrw);
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                vs[c] = warp_sum(vs[c]);
                bs[c] = warp_sum(bs[c]);
            }
            __syncwarp();
            for (int l = 0; l < ne; ++l) {  // per-edge target blocks (each target pose at most once)
                const int sjl = __shfl_sync(0xffffffffu, sj, l);
                if (sjl >= 0 && lane < 6) {
                    const double* R = rec + l * kRec;
                    const double g0 = R[kJt + lane] * R[kWt], g1 = R[kJt + 6 + lane] * R[kWt + 1];
                    v[6 * sjl + lane] += g0 * R[kJd] + g1 * R[kJd + 1];
                    bvec[6 * sjl + lane] += -(g0 * R[kR] + g1 * R[kR + 1]);
                }
                __syncwarp();
            }
            if (si >= 0 && lane < 6) {
                v[6 * si + lane] += vs[lane];
                bvec[6 * si + lane] += bs[lane];
            }
            int* p2e = wi + 4;  // local target pose -> edge (or -1)
            for (int i = lane; i < kMaxLocalPoses; i += 32) p2e[i] = -1;
            __syncwarp();
            if (sj >= 0) p2e[sj] = lane;
            if (lane == 0) {
                wi[0] = si;
                wi[1] = ne;
                wi[2] = dslot;
                wi[3] = k;
                const double hd = h + lambda;  // h_dd + damping (bundle_adjust.cpp:185)
                sc[0] = hd;
                sc[1] = bd;
                sc[2] = 1.0 / hd;
                if (dslot >= 0 && !(hd > 0)) set_status(a.status, kDevNonPositiveDepth);
                wr_sum += wrs;
                wr_w += wrw;
            }
        } else if (lane == 0) {
            wi[1] = -1;
        }
        __syncthreads();
        // ---- ordered accumulation of the batch into the group block ----
        for (int w = 0; w < kW; ++w) {
            const int* wiw = reinterpret_cast<const int*>(smem + L.wi) + w * (4 + kMaxLocalPoses + kMaxE);
            if (wiw[1] < 0) break;
            const int si = wiw[0];
            const bool dfree = wiw[2] >= 0;
            const double* recw = reinterpret_cast<const double*>(smem + L.rec) + (size_t)w * kMaxE * kRec;
            const double* vw = reinterpret_cast<const double*>(smem + L.vb) + (size_t)w * 2 * (nl > 0 ? nl : 1);
            const double* bw = vw + nl;
            const double* scw = reinterpret_cast<const double*>(smem + L.sc) + w * kScal;
            const double inv_h = scw[2];
            const int* p2e = wiw + 4;
            for (int ent = tid; ent < ne_l; ent += kT) {
                const unsigned ab = tab[ent];
                const int ia = ab & 0xff, ib = (ab >> 8) & 0xff, A = (ab >> 16) & 0xff, B = ab >> 24;
                const int ra = ia - 6 * A, rb = ib - 6 * B;
                double val = 0.0;
                if (A == si && B == si) {
                    val = scw[4 + 6 * ra + rb];
                } else if (A == si) {
                    const int l = p2e[B];
                    if (l >= 0) {
                        const double* R = recw + l * kRec;
                        val = (R[kGs + ra] * R[kWt]) * R[kJt + rb] + (R[kGs + 6 + ra] * R[kWt + 1]) * R[kJt + 6 + rb];
                    }
                } else if (B == si) {
                    const int l = p2e[A];
                    if (l >= 0) {
                        const double* R = recw + l * kRec;
                        val = (R[kJt + ra] * R[kWt]) * R[kGs + rb] + (R[kJt + 6 + ra] * R[kWt + 1]) * R[kGs + 6 + rb];
                    }
                } else if (A == B) {
                    const int l = p2e[A];
                    if (l >= 0) {
                        const double* R = recw + l * kRec;
                        val = (R[kJt + ra] * R[kWt]) * R[kJt + rb] + (R[kJt + 6 + ra] * R[kWt + 1]) * R[kJt + 6 + rb];
                    }
                }
                if (dfree) val -= (vw[ia] * inv_h) * vw[ib];
                S[ent] += val;
            }
            for (int i = tid; i < nl; i += kT) {
                double r = bw[i];
                if (dfree) r -= vw[i] * (inv_h * scw[1]);
                rhs[i] += r;
            }
            const int kw = wiw[3];
            for (int i = tid; i < nl; i += kT) P.patch_vl[(size_t)kw * P.max_nl + i] = vw[i];
            if (tid == 0) {
                a.patch_h[kw] = scw[0];
                a.patch_bd[kw] = scw[1];
            }
        }
        __syncthreads();
    }
    double* wr = reinterpret_cast<double*>(smem + L.wr);
    if (lane == 0) {
        wr[2 * warp] = wr_sum;
        wr[2 * warp + 1] = wr_w;
    }
    __syncthreads();
    double* part = P.g_part + P.g_off[g];
    for (int i = tid; i < ne_l; i += kT) part[i] = S[i];
    for (int i = tid; i < nl; i += kT) part[ne_l + i] = rhs[i];
    if (tid == 0) {
        double ws = 0, ww = 0;
        for (int w = 0; w < kW; ++w) {
            ws += wr[2 * w];
            ww += wr[2 * w + 1];
        }
        P.g_res[2 * g] = ws;
        P.g_res[2 * g + 1] = ww;
    }
}

// ---------------------------------------------------------------------------
// reduce: dense reduced system (lower triangle, row np = rhs) from the group
// blocks in group order, damping on the diagonal.
// ---------------------------------------------------------------------------
__global__ void bal_reduce_kernel(BALargeParams P) {
    if (P.ctrl[0] || P.ctrl[2]) return;
    const int np = 6 * P.a.n_free_poses;
    const int ld = np + 1;
    const double lambda = damping_of(P.a.damping, P.ctrl[1]);
    const long long total = (long long)ld * (ld + 1) / 2 - 1;  // lower triangle of rows 0..np, without (np, np)
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        int i = (int)((sqrt(8.0 * (double)idx + 1.0) - 1.0) * 0.5);
        while ((long long)i * (i + 1) / 2 > idx) --i;
        while ((long long)(i + 1) * (i + 2) / 2 <= idx) ++i;
        const int j = (int)(idx - (long long)i * (i + 1) / 2);
        double acc = 0.0;
        if (i == np) {  // rhs entry j
            const int pj = j / 6;
            for (int g = 0; g < P.n_groups; ++g) {
                const int lo = P.g_lo[g], nl = P.g_nl[g];
                if (pj >= lo && 6 * (pj - lo) < nl) acc += P.g_part[P.g_off[g] + nent(nl) + (j - 6 * lo)];
            }
        } else if (i - j <= P.bw) {
            const int pi = i / 6, pj = j / 6;
            for (int g = 0; g < P.n_groups; ++g) {
                const int lo = P.g_lo[g], nl = P.g_nl[g];
                if (pj >= lo && 6 * (pi - lo) < nl) {
                    const int la = j - 6 * lo, lb = i - 6 * lo;  // la <= lb
                    acc += P.g_part[P.g_off[g] + la * nl - la * (la - 1) / 2 + (lb - la)];
                }
            }
            if (i == j) acc += lambda;
        }
        P.A[(size_t)i * ld + j] = acc;
    }
}

// ---------------------------------------------------------------------------
// solve: banded blocked LDL^T + back-substitution + retraction (one CTA)
// ---------------------------------------------------------------------------
// A/B knob: the diagonal block factored by one warp (1) or four (4)
#ifndef PVO_BAL_DIAG_WARPS
#define PVO_BAL_DIAG_WARPS 4
#endif
__global__ void __launch_bounds__(kST, 1) bal_solve_kernel(BALargeParams P) {
    if (P.ctrl[0] || P.ctrl[2]) return;
    extern __shared__ __align__(16) unsigned char smem[];
    const BAParams& a = P.a;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int np = P.structure ? 0 : 6 * a.n_free_poses;
    const int ld = 6 * a.n_free_poses + 1;
    double* A = P.A;  // reduced system from the reduce kernel, factorised in place
    const int bw = min(P.bw, np > 0 ? np - 1 : 0);
    const int pr_cap = ((bw + 2 + 3) / 4) * 4;              // panel rows (band) + the rhs row, 4-row tiles
    double* Dg = reinterpret_cast<double*>(smem);          // [32][33] diagonal block
    double* Wp = Dg + kB * (kB + 1);                        // [32][pr_cap] unscaled panel (L D), column-major
    double* x = Wp + (size_t)pr_cap * kB;                   // [np] solution
    double* cc = x + (np > 0 ? np : 1);                     // [33] unscaled pivot column + d_kk
    double* xb = cc + kB + 1;                               // [32]
    double* dinv = xb + kB;                                 // [32]
    __shared__ int s_fail, s_zero;
    if (tid == 0) {
        s_fail = 0;
        s_zero = 0;
    }
    // optional phase clocks (pvo_ctx_set_tracing): [0] start, [1] begin, [2] diag, [3] panel,
    // [4] trailing (accumulated over blocks), [5] factorised, [6] solved, [7] end
    long long* pc = (a.phase_clocks && tid == 0) ? a.phase_clocks + 8 * 14 : nullptr;
    long long tk = 0;
    if (pc) {
        pc[0] = clock64();
        pc[2] = pc[3] = pc[4] = 0;
    }
    __syncthreads();
    if (pc) pc[1] = tk = clock64();
    for (int k0 = 0; k0 < np; k0 += kB) {
        const int kb = min(kB, np - k0);
        const int r0 = k0 + kb;                        // first panel row
        const int r1 = min(np, k0 + kb + bw);           // panel rows [r0, r1) + the rhs row
        const int nr = r1 - r0 + 1;
        // (1) diagonal block, warp 0: lane = row, the row in registers (loads issued
        //     together), the unscaled pivot column broadcast through shared memory
#if PVO_BAL_DIAG_WARPS == 4
        // (A/B variant) four warps: lane = row, warp w holds columns 8w .. 8w+7 of
        // it; per pivot the owner warp publishes d_kk, 1/d_kk and the column into
        // a double-buffered slot, one 128-thread named barrier, then every warp
        // updates its columns (the same expressions as the one-warp form)
        if (warp < 4) {
            constexpr int kCW = kB / 4;
            __shared__ double ccw[2][kB + 1];
            double r[kCW];
#pragma unroll
            for (int c = 0; c < kCW; ++c) {
                const int j = kCW * warp + c;
                r[c] = (lane < kb && j <= lane) ? A[(size_t)(k0 + lane) * ld + k0 + j] : 0.0;
            }
            bool fail = false, zero = false;
#pragma unroll 1
            for (int kk = 0; kk < kb; ++kk) {
                const int ow = kk / kCW, oc = kk - kCW * ow;
                double* cb = ccw[kk & 1];
                const bool below = lane > kk && lane < kb;
                bool vk = true;  // the owner's pivot test (its column kk is written by it alone)
                if (warp == ow) {
                    double rk = 0.0;
#pragma unroll
                    for (int c = 0; c < kCW; ++c)
                        if (c == oc) rk = r[c];
                    const double dk = __shfl_sync(0xffffffffu, rk, kk);
                    const bool valid = fabs(dk) > 0.0;
                    vk = valid;
                    if (k0 + kk == 0 && !valid) zero = true;  // Eigen: all-zero diagonal -> x = 0
                    const double inv = valid ? 1.0 / dk : 0.0;
                    const double ci = below ? rk : 0.0;
                    if (below && !valid && ci != 0.0) fail = true;
                    cb[lane] = ci;
                    if (lane == 0) {
                        cb[kB] = inv;
                        dinv[kk] = inv;
                    }
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                const double inv = cb[kB];
                const double ci = cb[lane];
                const double cs = ci * inv;
#pragma unroll
                for (int c = 0; c < kCW; ++c) {
                    const int j = kCW * warp + c;
                    if (below && j > kk && j <= lane) r[c] -= cs * cb[j];
                    if (below && j == kk) r[c] = vk ? cs : ci;
                }
            }
#pragma unroll
            for (int c = 0; c < kCW; ++c) {
                const int j = kCW * warp + c;
                if (lane < kb && j <= lane) {
                    Dg[lane * (kB + 1) + j] = r[c];
                    A[(size_t)(k0 + lane) * ld + k0 + j] = r[c];
                }
            }
            if (__any_sync(0xffffffffu, fail) && lane == 0) s_fail = 1;
            if (__any_sync(0xffffffffu, zero) && lane == 0) s_zero = 1;
        }
#else
        if (warp == 0) {
            double r[kB];
#pragma unroll
            for (int j = 0; j < kB; ++j) r[j] = (lane < kb && j <= lane) ? A[(size_t)(k0 + lane) * ld + k0 + j] : 0.0;
            bool fail = false, zero = false;
#pragma unroll
            for (int kk = 0; kk < kB; ++kk) {
                if (kk < kb) {
                    if (lane == kk) cc[kB] = r[kk];  // d_kk
                    __syncwarp();
                    const double dk = cc[kB];
                    const bool valid = fabs(dk) > 0.0;
                    if (k0 + kk == 0 && !valid) zero = true;  // Eigen: all-zero diagonal -> x = 0
                    const double inv = valid ? 1.0 / dk : 0.0;
                    if (lane == 0) dinv[kk] = inv;
                    const bool below = lane > kk && lane < kb;
                    const double ci = below ? r[kk] : 0.0;
                    cc[lane] = ci;
                    __syncwarp();
                    if (below && !valid && ci != 0.0) fail = true;
                    const double cs = ci * inv;
#pragma unroll
                    for (int j = kk + 1; j < kB; ++j)
                        if (below && j <= lane) r[j] -= cs * cc[j];
                    if (below) r[kk] = valid ? cs : ci;
                    __syncwarp();
                }
            }
#pragma unroll
            for (int j = 0; j < kB; ++j)
                if (lane < kb && j <= lane) {
                    Dg[lane * (kB + 1) + j] = r[j];
                    A[(size_t)(k0 + lane) * ld + k0 + j] = r[j];
                }
            if (__any_sync(0xffffffffu, fail) && lane == 0) s_fail = 1;
            if (__any_sync(0xffffffffu, zero) && lane == 0) s_zero = 1;
        }
#endif
        __syncthreads();
        if (pc) {
            const long long t = clock64();
            pc[2] += t - tk;
            tk = t;
        }
        if (s_zero) break;
        // (2) panel rows: forward elimination against the diagonal block, one thread per row
        for (int t = tid; t < nr; t += kST) {
            const int i = t < nr - 1 ? r0 + t : np;
            double seg[kB];
#pragma unroll
            for (int j = 0; j < kB; ++j) seg[j] = j < kb ? A[(size_t)i * ld + k0 + j] : 0.0;
            bool fail = false;
#pragma unroll
            for (int kk = 0; kk < kB; ++kk) {
                if (kk < kb) {
                    const double c = seg[kk];
                    // fixed trip count: with j = kk + 1 .. the outer loop stayed rolled
                    // and seg[] went to local memory (STACK 304 B, 600 LDL/STL); columns
                    // j >= kb are never stored, so they need no guard
#pragma unroll
                    for (int j = 0; j < kB; ++j)
                        if (j > kk) seg[j] -= c * Dg[j * (kB + 1) + kk];
                    const double inv = dinv[kk];
                    if (inv == 0.0 && c != 0.0 && i < np) fail = true;
                    Wp[kk * pr_cap + t] = c;
                    seg[kk] = inv != 0.0 ? c * inv : c;
                }
            }
#pragma unroll
            for (int j = 0; j < kB; ++j)
                if (j < kb) A[(size_t)i * ld + k0 + j] = seg[j];
            if (fail) s_fail = 1;
        }
        __syncthreads();
        if (pc) {
            const long long t = clock64();
            pc[3] += t - tk;
            tk = t;
        }
        // (3) trailing update A[i][j] -= sum_kk (L D)_i,kk L_j,kk over the panel rows
        //     (j <= i, j < np; the rhs row is panel row nr - 1), 4 x 4 register tiles:
        //     8 shared loads feed 16 FMAs
        {
            const int TI = (nr + 3) / 4;
            const int ntiles = TI * (TI + 1) / 2;
            for (int t = tid; t < ntiles; t += kST) {
                int I = (int)((sqrtf(8.f * (float)t + 1.f) - 1.f) * 0.5f);
                while (I * (I + 1) / 2 > t) --I;
                while ((I + 1) * (I + 2) / 2 <= t) ++I;
                const int J = t - I * (I + 1) / 2;
                double acc[4][4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
                const double* w0 = Wp + 4 * I;  // rows 4I.. of column kk at w0[kk * pr_cap]
                const double* l0 = Wp + 4 * J;
                double old[4][4];  // the tile's current values: 16 independent loads in flight
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int ti = 4 * I + u;
                    const int i = ti < nr - 1 ? r0 + ti : np;
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const int tj = 4 * J + v;
                        old[u][v] = (ti < nr && tj < nr - 1 && tj <= ti) ? A[(size_t)i * ld + r0 + tj] : 0.0;
                    }
                }
                for (int kk = 0; kk < kb; ++kk) {
                    const double di = dinv[kk];
                    const double2* wq = reinterpret_cast<const double2*>(w0 + kk * pr_cap);
                    const double2* lq = reinterpret_cast<const double2*>(l0 + kk * pr_cap);
                    const double2 wa = wq[0], wb = wq[1], la = lq[0], lb = lq[1];
                    const double wv[4] = {wa.x, wa.y, wb.x, wb.y};
                    const double lr[4] = {la.x, la.y, lb.x, lb.y};
                    double lv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) lv[u] = di != 0.0 ? lr[u] * di : lr[u];  // L_j,kk = W_j,kk / d_kk
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v) acc[u][v] = fma(wv[u], lv[v], acc[u][v]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int ti = 4 * I + u;
                    const int i = ti < nr - 1 ? r0 + ti : np;
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const int tj = 4 * J + v;
                        if (ti < nr && tj < nr - 1 && tj <= ti) A[(size_t)i * ld + r0 + tj] = old[u][v] - acc[u][v];
                    }
                }
            }
        }
        __syncthreads();
        if (pc) {
            const long long t = clock64();
            pc[4] += t - tk;
            tk = t;
        }
    }
    if (pc) pc[5] = clock64();
    if (np > 0 && s_fail) {
        if (tid == 0) set_status(a.status, kDevFactorization);
        P.ctrl[2] = 1;  // factorization failure: stop the window
        return;
    }
    if (np > 0) {
        // z = D^-1 L^-1 b sits in row np (pseudo-inverse of D)
        for (int i = tid; i < np; i += kST)
            x[i] = s_zero ? 0.0 : (fabs(A[(size_t)i * ld + i]) > DBL_MIN ? A[(size_t)np * ld + i] : 0.0);
        __syncthreads();
        if (!s_zero) {
            // banded back-substitution L^T x = z, last block first
            // Band part of each block: lane = column k0 + lane, warp = row stripe, so a
            // warp's loads of a band row are one coalesced 256-byte segment and the
            // stripes' rows are independent loads in flight; warp 0 sums the stripes
            // in stripe order (the one-warp-per-column dot it replaces walked each
            // column's rows with one L2 round trip per 32 rows: 137k -> 82k cycles at C4)
            constexpr int kStripes = kST / 32;
            __shared__ double part[kStripes * 32];
            for (int k0 = ((np - 1) / kB) * kB; k0 >= 0; k0 -= kB) {
                const int kb = min(kB, np - k0);
                const int r1 = min(np, k0 + kb + bw);
                {
                    double s0 = 0.0, s1 = 0.0;
                    if (lane < kb) {
                        const double* col = A + k0 + lane;
                        int j = k0 + kb + warp;
#pragma unroll 4
                        for (; j + kStripes < r1; j += 2 * kStripes) {
                            s0 += col[(size_t)j * ld] * x[j];
                            s1 += col[(size_t)(j + kStripes) * ld] * x[j + kStripes];
                        }
                        if (j < r1) s0 += col[(size_t)j * ld] * x[j];
                    }
                    part[warp * 32 + lane] = s0 + s1;
                }
                __syncthreads();
                if (warp == 0) {
                    double lq[kB];  // L_{k0+q, k0+lane}: loads issued together
#pragma unroll
                    for (int q = 0; q < kB; ++q) lq[q] = (q < kb && lane < q) ? A[(size_t)(k0 + q) * ld + k0 + lane] : 0.0;
                    double sb = 0.0;
#pragma unroll
                    for (int q = 0; q < kStripes; ++q) sb += part[q * 32 + lane];
                    double xc = lane < kb ? x[k0 + lane] - sb : 0.0;
#pragma unroll
                    for (int q = kB - 1; q >= 0; --q) {
                        if (q < kb) {
                            const double xv = __shfl_sync(0xffffffffu, xc, q);
                            if (lane < q) xc -= lq[q] * xv;
                        }
                    }
                    if (lane < kb) x[k0 + lane] = xc;
                }
                __syncthreads();
            }
        }
        if (pc) pc[6] = clock64();
        bool bad = false;
        for (int i = tid; i < np; i += kST) {
            a.delta[i] = x[i];
            bad = bad || !isfinite(x[i]);
        }
        if (__syncthreads_or(bad)) {
            if (tid == 0) set_status(a.status, kDevNonFinitePose);
            P.ctrl[2] = 1;
            return;
        }
    }
    // retraction of the free poses (bundle_adjust.cpp:202-207) + candidate matrices
    for (int i = tid; i < a.n_poses; i += kST) {
        const int slot = np > 0 ? a.pose_free_slot[i] : -1;
        const SE3 p = se3_load(a.poses + 7 * i);
        if (slot >= 0) {
            double xi[6];
#pragma unroll
            for (int c = 0; c < 6; ++c) xi[c] = a.delta[6 * slot + c];
            se3_store(se3_retract(p, xi), a.cand_poses + 7 * i);
        } else {
            se3_store(p, a.cand_poses + 7 * i);
        }
    }
    __syncthreads();
    pose_mats(a.cand_poses, P.cmats, a.n_poses);
    if (pc) pc[7] = clock64();
}

// ---------------------------------------------------------------------------
// update: depth back-substitution (clamped) + residual at the candidate state
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kT) bal_update_kernel(BALargeParams P) {
    if (P.ctrl[0] || P.ctrl[2]) return;  // settled, or failed
    const BAParams& a = P.a;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int G = gridDim.x, b = blockIdx.x;
    const int k0 = (int)((long long)a.n_patches * b / G), k1 = (int)((long long)a.n_patches * (b + 1) / G);
    const Cam K{a.K[0], a.K[1], a.K[2], a.K[3]};
    __shared__ double wr[2 * kW];
    double wr_sum = 0, wr_w = 0;
    for (int k = k0 + warp; k < k1; k += kW) {
        double dnew = a.depth[k];
        if (a.depth_slot[k] >= 0) {
            double dot = 0.0;
            if (!P.structure) {
                const int g = P.patch_group[k];
                const int lo = P.g_lo[g], nl = P.g_nl[g];
                for (int i = lane; i < nl; i += 32) dot += P.patch_vl[(size_t)k * P.max_nl + i] * a.delta[6 * lo + i];
            }
            dot = warp_sum(dot);
            const double dd = (1.0 / a.patch_h[k]) * (a.patch_bd[k] - dot);  // bundle_adjust.cpp:88-89
            if (!isfinite(dd) && lane == 0) set_status(a.status, kDevNonFiniteDepth);
            dnew = fmax(0.0, dnew + dd);  // bundle_adjust.cpp:211
        }
        if (lane == 0) a.cand_depth[k] = dnew;
        const int eb = a.patch_edge_begin[k], ne = a.patch_edge_begin[k + 1] - eb;
        const int src = a.patch_src[k];
        const SE3 pi = se3_load(a.cand_poses + 7 * src);
        double ws = 0, ww = 0;
        for (int l = lane; l < ne; l += 32) {
            const int e = eb + l;
            const int tgt = a.e_pose[e];
            const SE3 pj = se3_load(a.cand_poses + 7 * tgt);
            double cu, cv;
            bool behind;
            const Relative rel = rel_from_mats(P.cmats + 12 * src, P.cmats + 12 * tgt);
            center_behind(se3_equal(pi, pj), rel, K, a.patch_x + 9 * (size_t)k, a.patch_y + 9 * (size_t)k, dnew, &cu,
                          &cv, &behind);
            const double rx = cu - a.e_target[2 * e], ry = cv - a.e_target[2 * e + 1];
            const double wx = behind ? 0.0 : a.e_weight[2 * e];
            const double wy = behind ? 0.0 : a.e_weight[2 * e + 1];
            ws += wx * rx * rx + wy * ry * ry;
            ww += wx + wy;
        }
        ws = warp_sum(ws);
        ww = warp_sum(ww);
        wr_sum += ws;
        wr_w += ww;
    }
    if (lane == 0) {
        wr[2 * warp] = wr_sum;
        wr[2 * warp + 1] = wr_w;
    }
    __syncthreads();
    if (tid == 0) {
        double ws = 0, ww = 0;
        for (int w = 0; w < kW; ++w) {
            ws += wr[2 * w];
            ww += wr[2 * w + 1];
        }
        P.u_res[2 * b] = ws;
        P.u_res[2 * b + 1] = ww;
    }
}

// ---------------------------------------------------------------------------
// decide: the divergence guard (bundle_adjust.cpp:327-366), one CTA
// ---------------------------------------------------------------------------
__global__ void bal_decide_kernel(BALargeParams P, int n_update_ctas) {
    if (P.ctrl[0] || P.ctrl[2]) return;
    const BAParams& a = P.a;
    const int tid = threadIdx.x;
    __shared__ double s_res[4];
    __shared__ int s_commit;
    if (*(volatile int*)a.status) {  // any error of this attempt stops the window (as ba.cu)
        if (tid == 0) P.ctrl[2] = 1;
        return;
    }
    if (tid < 32) {
        double q[4] = {0, 0, 0, 0};
        for (int g = tid; g < P.n_groups; g += 32) {
            q[0] += P.g_res[2 * g];
            q[1] += P.g_res[2 * g + 1];
        }
        for (int c = tid; c < n_update_ctas; c += 32) {
            q[2] += P.u_res[2 * c];
            q[3] += P.u_res[2 * c + 1];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) q[u] = warp_sum(q[u]);
        if (tid == 0)
            for (int u = 0; u < 4; ++u) s_res[u] = q[u];
    }
    __syncthreads();
    if (tid == 0) {
        const double sb = s_res[0], wb = s_res[1], sa = s_res[2], wa = s_res[3];
        const double before = wb > 0 ? sqrt(sb / wb) : 0.0;
        const double after = wa > 0 ? sqrt(sa / wa) : 0.0;
        const double thr = 1.5 * before + 1e-9;
        const int attempt = P.ctrl[1];
        if (a.attempts) *a.attempts += 1;
        bool accept, reject = false;
        if (P.structure) {
            accept = true;
        } else if (attempt == 0) {
            accept = !(after > thr);  // bundle_adjust.cpp:330
        } else {
            accept = after <= thr;  // bundle_adjust.cpp:339-340
        }
        int commit = 0;
        if (!accept && !P.structure) {
            if (attempt < 3) {
                P.ctrl[1] = attempt + 1;
            } else {
                reject = true;  // keep the state put (bundle_adjust.cpp:347-353)
            }
        }
        if (accept || reject) {
            P.ctrl[0] = 1;
            commit = accept;
            if (!P.structure) {
                int n = *a.n_norms;
                if (n == 0) a.residual_norms[n++] = before;
                a.residual_norms[n++] = reject ? before : after;
                *a.n_norms = n;
            }
        }
        s_commit = commit;
    }
    __syncthreads();
    if (s_commit) {
        for (int i = tid; i < 7 * a.n_poses; i += blockDim.x) a.poses[i] = a.cand_poses[i];
        for (int i = tid; i < 12 * a.n_poses; i += blockDim.x) P.mats[i] = P.cmats[i];
        for (int k = tid; k < a.n_patches; k += blockDim.x) a.depth[k] = a.cand_depth[k];
    }
}

}  // namespace

size_t ba_large_solver_smem(int n_free_poses, int bw) {
    const int np = 6 * n_free_poses;
    if (bw > np - 1) bw = np > 0 ? np - 1 : 0;
    const size_t rows = ((size_t)(bw + 2 + 3) / 4) * 4;
    return 8 * ((size_t)kB * (kB + 1) + rows * kB + (np > 0 ? np : 1) + 3 * kB + 1) + 16;
}
int ba_large_assemble_smem(int nl) { return assemble_layout(nl).total; }

cudaError_t launch_ba_large(BALargeParams& p, int num_sms, cudaStream_t stream, int* launches) {
    const BAParams& a = p.a;
    int n = 0;
    cudaError_t err;
    const int asm_bytes = assemble_layout(p.max_nl).total;
    if ((err = cudaFuncSetAttribute(bal_assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, asm_bytes)))
        return err;
    const size_t solve_bytes = ba_large_solver_smem(a.n_free_poses, p.bw);
    if (solve_bytes > 227 * 1024) return cudaErrorNotSupported;
    if ((err = cudaFuncSetAttribute(bal_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)solve_bytes)))
        return err;
    if ((err = cudaMemsetAsync(p.ctrl, 0, 4 * sizeof(int), stream))) return err;
    const int init_grid = min(4 * num_sms, max(1, (a.n_edges + 255) / 256));
    bal_init_kernel<<<init_grid, 256, 0, stream>>>(p);
    ++n;
    const int np = 6 * a.n_free_poses;
    const long long ents = (long long)(np + 1) * (np + 2) / 2;
    long long rg = (ents + 255) / 256;
    if (rg > 4LL * num_sms) rg = 4LL * num_sms;
    const int red_grid = rg < 1 ? 1 : (int)rg;
    const int upd_grid = p.n_update_ctas;
    const int total_iters = a.structure_only + a.iterations;
    for (int it = 0; it < total_iters; ++it) {
        p.structure = it < a.structure_only ? 1 : 0;
        if ((err = cudaMemsetAsync(p.ctrl, 0, 2 * sizeof(int), stream))) return err;  // done, attempt
        const int attempts = p.structure ? 1 : 4;
        for (int att = 0; att < attempts; ++att) {
            bal_assemble_kernel<<<p.n_groups, kT, asm_bytes, stream>>>(p, p.structure);
            ++n;
            if (!p.structure) {
                bal_reduce_kernel<<<red_grid, 256, 0, stream>>>(p);
                ++n;
                if (p.dbg_A && it == 0 && att == 0)
                    cudaMemcpyAsync(p.dbg_A, p.A, sizeof(double) * (size_t)(np + 1) * (np + 1), cudaMemcpyDeviceToDevice, stream);
            }
            bal_solve_kernel<<<1, kST, solve_bytes, stream>>>(p);
            bal_update_kernel<<<upd_grid, kT, 0, stream>>>(p);
            bal_decide_kernel<<<1, 256, 0, stream>>>(p, upd_grid);
            n += 3;
        }
    }
    if (launches) *launches = n;
    return cudaGetLastError();
}

}  // namespace pvo_dev
