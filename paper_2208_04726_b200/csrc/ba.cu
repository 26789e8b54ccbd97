// ba.cu — sparse Gauss-Newton bundle adjustment of one window (K3-K6),
// sm_100a, FP64.
//
// Reference: optimize_window / gauss_newton_step / schur_solve
// (bundle_adjust.cpp:62-375).  The reference builds a dense (6F+P)^2
// Hessian and runs an Eigen LDLT on the Schur complement.  Here the whole
// iteration loop — frozen targets, assembly, Schur elimination of the depth
// block, the pose solve, retraction, the weighted residual norms and the
// divergence guard (damping x1e3, x1e6, x1e9 retries) — runs inside ONE
// persistent cooperative kernel; control never returns to the host.
//
// Phases per Gauss-Newton attempt (3 grid-wide barriers):
//   P1 assemble   warp per patch, lane per edge: Jacobians (camera.cpp:73-108),
//                 residual, weight; per-patch reductions give h_k, b_k, the
//                 patch's H_pd column v_k and gradient; every thread of the CTA
//                 owns fixed entries of the CTA's reduced system
//                     S += sum_e J~_e^T W_e J~_e - v_k v_k^T / h_k
//                     r += b_k - v_k b_dk / h_k
//                 accumulated patch after patch (no atomics, fixed order).
//   --- grid sync
//   P2 reduce     entry-parallel over the grid: S = sum over CTAs (fixed order)
//                 + damping on the diagonal.
//   --- grid sync
//   P3 solve      EVERY CTA solves the small pose system redundantly (identical
//                 inputs and code -> bit-identical results, no broadcast): a
//                 natural-order LDL^T of the SPD reduced system with the
//                 matrix in registers, one barrier per column
//                 (ldlt_solve_cta); retraction of the free poses into the
//                 CTA's own copy of the candidate state.
//   P4 update     warp per patch: depth back-substitution, clamp at 0, weighted
//                 residual at the candidate state (bitwise-equal-pose shortcut).
//   --- grid sync
//   P5 decide     every CTA evaluates the same guard from the same partial sums,
//                 then commits (its pose copy, its depths), retries with heavier
//                 damping, or skips.  Partials and status words are double
//                 buffered by attempt parity, so no barrier is needed here.
// Determinism: every reduction has a fixed order (shuffle trees, per-thread
// entry ownership, ordered cross-CTA sums), so reruns are bit-identical.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "geometry.cuh"
#include "ba_common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace pvo_dev {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxFree = 16;            // free poses  -> np <= 96
constexpr int kMaxNp = 6 * kMaxFree;
constexpr int kMaxEdges = 32;           // edges per patch (lane per edge)
constexpr int kMaxPoses = 128;          // poses held per CTA in shared memory
constexpr int kRec = 30;                // doubles per edge record
// edge record: Gs[12] Jt[12] Jd[2] r[2] w[2]
constexpr int kGs = 0, kJt = 12, kJd = 24, kR = 26, kW = 28;

__host__ __device__ inline int nent_of(int np) { return np * (np + 1) / 2; }
__host__ __device__ inline int align16(int x) { return (x + 15) & ~15; }

// Shared-memory plan (bytes).  Fixed part: entry table, pose copies, delta.
// Union part: assembly scratch | solve workspace.
struct Layout {
    int ab, pose, cand, rmat, rmatc, delta, flags, uni;
    int S, rhs, rec, vb, scal, wr, ints;  // assembly
    int A, x, od, perm, c, l, pw, blk;    // solve
    int total;
};

constexpr int kBlkL = 8;  // LDL^T block size (see ldlt_solve_cta)
// per-warp ints: si, ne, depth slot, patch | p2e[kMaxFree] | nxt[kMaxEdges] | targets[kMaxFree], count
constexpr int kWarpInts = 4 + kMaxFree + kMaxEdges + kMaxFree + 1;
constexpr int kScal = 40;  // per-warp scalars: h, bd, inv_h, pad, then the 6x6 source block

__host__ __device__ inline Layout make_layout(int np_full, int n_poses) {
    Layout L;
    int off = 0;
    L.ab = off;
    off += align16(4 * nent_of(np_full));
    L.pose = off;
    off += align16(8 * 7 * n_poses);
    L.cand = off;
    off += align16(8 * 7 * n_poses);
    L.rmat = off;  // rotation matrix + translation of every pose (current state)
    off += align16(8 * 12 * n_poses);
    L.rmatc = off;  // ... of the candidate state
    off += align16(8 * 12 * n_poses);
    L.delta = off;
    off += align16(8 * (np_full > 0 ? np_full : 1));
    L.flags = off;
    off += 32;
    L.uni = off;
    int a = off;
    L.S = a;
    a += 8 * nent_of(np_full);
    L.rhs = a;
    a += 8 * np_full;
    L.rec = a;
    a += 8 * kWarps * kMaxEdges * kRec;
    L.vb = a;
    a += 8 * kWarps * 2 * np_full;
    L.scal = a;
    a += 8 * kWarps * kScal;
    L.wr = a;
    a += 8 * kWarps * 4;
    L.ints = a;
    a += 4 * kWarps * kWarpInts;
    int s = off;
    L.A = s;
    s += 8 * (np_full + 1) * (np_full + 1);  // + the rhs row
    L.x = s;
    s += 8 * (nent_of(np_full) + np_full);   // staged system, then x
    L.od = s;
    s += 8 * (np_full > kBlkL ? np_full : kBlkL);
    L.c = s;
    s += 8 * np_full;
    L.l = s;
    s += 8 * np_full;
    L.pw = s;
    s += 8 * 16 * (np_full + 1);  // blocked LDL^T panel buffers (L^T panel, L D panel)
    L.perm = s;
    s += 4 * np_full;
    s = align16(s);
    L.blk = s;  // 6-column blocked LDL^T: raw panel [6][112], W and L panels [112][6]
    s += 8 * 3 * 6 * 112;
    L.total = align16(a > s ? a : s);
    return L;
}

template <typename T>
__device__ __forceinline__ T* at(unsigned char* smem, int off) {
    return reinterpret_cast<T*>(smem + off);
}

// ---------------------------------------------------------------------------
// LDL^T solve of the np x np reduced pose system S x = rhs, held as (upper
// triangle row-major, rhs) in global memory; all threads of the CTA.  x_out
// may be shared or global memory.  Returns false (all threads) when a pivot is
// negative / non-finite, or zero with a non-zero column below (LDLT::info()).
//
// The reference factors S with Eigen's pivoted LDLT (bundle_adjust.cpp:76).
// S is symmetric positive definite by construction (the Schur complement of
// the damped, positive definite GN Hessian), so the natural-order LDL^T gives
// the same solution up to rounding; no pivot sequence is simulated.
//
// Register-resident right-looking elimination with one barrier per column:
// [S; rhs^T] (row np carries the right-hand side, so the forward substitution
// comes for free) is distributed block-cyclically over a 16 x 16 thread grid
// and held in registers for the whole factorisation.  Step k broadcasts the
// (final) column k and 1/d_k through a double-buffered shared column; every
// thread applies  A[i][j] -= c_i (c_j / d_k)  (k < j <= i, c = unscaled
// column k; inactive columns get a zero factor, so the update is branch-free)
// and the owners of column k+1 publish it (and the next pivot's reciprocal)
// for step k+1.  The backward substitution L^T x = D^-1 L^-1 rhs runs on
// warp 0 with x in registers, column-oriented, no barriers (|d| <= DBL_MIN ->
// pseudo-inverse 0, LDLT::_solve_impl).  (tools/micro_solve: np = 60 in
// 25.3 us per solve vs 29.0 us for the Eigen-pivot-order blocked version.)
// ---------------------------------------------------------------------------
// 16 x 16 thread grid, block-cyclic: thread (ty, tx) owns rows ty + 16 a and
// columns tx + 16 b of [S; rhs^T]; RPT x CPT entries in registers
constexpr int kGrid = 16;
static_assert(kThreads == kGrid * kGrid, "solve grid");

#ifndef SOLVE_PROBE_BEGIN  // phase clocks for tools/micro_solve.cu
#define SOLVE_PROBE_BEGIN
#define SOLVE_PROBE(i)
#endif
template <int RPT, int CPT>
__device__ bool ldlt_solve_regs(const double* sys, int np, unsigned char* smem, const Layout& L, double* x_out) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ty = tid / kGrid, tx = tid % kGrid;
    SOLVE_PROBE_BEGIN
    const int ld = np + 1;
    double* A = at<double>(smem, L.A);    // [(np+1)][(np+1)]: L (scaled) and z = D^-1 L^-1 rhs in row np
    double* col = at<double>(smem, L.pw);  // [2][np+1] column broadcast, double-buffered by step parity
    double* dinv = at<double>(smem, L.c);  // 1 / d_k
    double* dv = at<double>(smem, L.l);    // d_k
    double v[RPT][CPT];
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
        const int i = ty + kGrid * a;
#pragma unroll
        for (int b = 0; b < CPT; ++b) {
            const int j = tx + kGrid * b;
            // entry (i, j), j <= i: the packed upper triangle's (j, i); row np: the rhs
            double x = 0.0;
            if (j <= i && j < np && i <= np) x = i < np ? sys[j * np - j * (j - 1) / 2 + (i - j)] : sys[nent_of(np) + j];
            v[a][b] = x;
        }
    }
    // column 0 (owned by tx == 0) and the first pivot
    if (tx == 0) {
#pragma unroll
        for (int a = 0; a < RPT; ++a)
            if (ty + kGrid * a <= np) col[ty + kGrid * a] = v[a][0];
        if (ty == 0) {
            dv[0] = v[0][0];
            dinv[0] = v[0][0] != 0.0 ? __drcp_rn(v[0][0]) : 0.0;  // = 1.0 / d (correctly rounded)
        }
    }
    __syncthreads();
    SOLVE_PROBE(0)
    bool fail = false;
    for (int k = 0; k < np; ++k) {
        const double* cur = col + (k & 1) * ld;
        double* nxt = col + ((k + 1) & 1) * ld;
        const double dk = dv[k], inv = dinv[k];
        double ci[RPT], cj[CPT];
#pragma unroll
        for (int a = 0; a < RPT; ++a) {
            const int i = ty + kGrid * a;
            ci[a] = (i > k && i <= np) ? cur[i] : 0.0;
        }
#pragma unroll
        for (int b = 0; b < CPT; ++b) {
            const int j = tx + kGrid * b;
            cj[b] = (j > k && j < np) ? cur[j] * inv : 0.0;  // inactive columns: no update
        }
        // a zero pivot is valid only with a zero column below (LDLT::info()); negative
        // or non-finite pivots do not occur in the SPD system: a failed factorisation
        if (tx == (k & (kGrid - 1)) && dk == 0.0) {
#pragma unroll
            for (int a = 0; a < RPT; ++a) fail = fail || (ci[a] != 0.0 && ty + kGrid * a < np);
        }
        fail = fail || !(dk >= 0.0) || !isfinite(dk);
#pragma unroll
        for (int a = 0; a < RPT; ++a)
#pragma unroll
            for (int b = 0; b < CPT; ++b) v[a][b] -= ci[a] * cj[b];  // A -= c c^T / d_k (unpivoted LDLT)
        // column k+1 is final after step k: its owners publish it and the next pivot
        const int kn = k + 1;
        if (tx == (kn & (kGrid - 1)) && kn < np) {
            const int bn = kn / kGrid;
            double vc[RPT];
#pragma unroll
            for (int a = 0; a < RPT; ++a) {  // v[a][bn] by selects (no dynamic register indexing)
                vc[a] = v[a][0];
#pragma unroll
                for (int b = 1; b < CPT; ++b) vc[a] = b == bn ? v[a][b] : vc[a];
            }
            double dn = 0.0;
#pragma unroll
            for (int a = 0; a < RPT; ++a) {
                const int i = ty + kGrid * a;
                if (i >= kn && i <= np) nxt[i] = vc[a];
                dn = i == kn ? vc[a] : dn;
            }
            if (ty == (kn & (kGrid - 1))) {  // the diagonal entry's owner
                dv[kn] = dn;
                dinv[kn] = dn != 0.0 ? __drcp_rn(dn) : 0.0;
            }
        }
        __syncthreads();
    }
    SOLVE_PROBE(1)
    if (__syncthreads_or(fail)) return false;
    // store L = C D^-1 (strictly lower) and z = D^-1 y (row np); |d| <= DBL_MIN: pseudo-inverse 0
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
        const int i = ty + kGrid * a;
#pragma unroll
        for (int b = 0; b < CPT; ++b) {
            const int j = tx + kGrid * b;
            if (j < i && j < np && i <= np) A[i * ld + j] = fabs(dv[j]) > DBL_MIN ? v[a][b] * dinv[j] : 0.0;
        }
    }
    __syncthreads();
    SOLVE_PROBE(2)
    // backward substitution L^T x = z on warp 0, column-oriented: lane l keeps
    // z_l, z_{l+32}, z_{l+64} in registers; once x_i = z_i is final it is
    // broadcast and every z_r (r < i) takes its L_ir x_i term (no barriers)
    if (warp == 0) {
        __syncwarp();
        const double* z = A + np * ld;
        double z0 = lane < np ? z[lane] : 0.0, z1 = lane + 32 < np ? z[lane + 32] : 0.0;
        double z2 = lane + 64 < np ? z[lane + 64] : 0.0;
        for (int i = np - 1; i >= 0; --i) {
            const int sl = i >> 5;
            const double own = sl == 0 ? z0 : sl == 1 ? z1 : z2;
            const double xi = __shfl_sync(0xffffffffu, own, i & 31);
            const double* Li = A + i * ld;
            if (lane < i) z0 -= Li[lane] * xi;
            if (lane + 32 < i) z1 -= Li[lane + 32] * xi;
            if (lane + 64 < i) z2 -= Li[lane + 64] * xi;
        }
        if (lane < np) x_out[lane] = z0;
        if (lane + 32 < np) x_out[lane + 32] = z1;
        if (lane + 64 < np) x_out[lane + 64] = z2;
    }
    __syncthreads();
    SOLVE_PROBE(3)
    return true;
}

// 1 / d in FP64: the MUFU estimate + two Newton steps (full precision, not the
// correctly rounded __drcp_rn: a shorter dependency chain on the pivot path;
// every thread computes the same value, so CTAs stay bit-identical)
__device__ __forceinline__ double rcp_nr(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}

// Blocked variant: 6 columns (one pose) per step, two barriers per step instead of
// six.  The matrix stays register-resident and block-cyclic as above.  Step K
// (columns k0 .. k0+5): the owners have published the block's raw columns (rows
// >= k0) to a panel; every row thread i >= k0 + 6 (the rhs row np included)
// factors the 6 x 6 diagonal block redundantly in registers (LDL^T, natural order)
// and solves its row, W_i = A_iK L_KK^-T and L_iK = W_i D_K^-1, writing L_iK
// (final) into A and W_i / L_iK into the panels; after a barrier every thread
// applies the block's rank-6 update A_ij -= L_iK . W_jK to its entries and the
// owners of the next block publish it.  The same factorisation as the unblocked
// loop up to the regrouping of each block's six updates.
template <int RPT, int CPT>
__device__ bool ldlt_solve_blk6(const double* sys, int np, unsigned char* smem, const Layout& L, double* x_out) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ty = tid / kGrid, tx = tid % kGrid;
    SOLVE_PROBE_BEGIN
    const int ld = np + 1;
    constexpr int kR = kGrid * RPT;  // rows held (>= np + 1)
    double* A = at<double>(smem, L.A);
    double* dinv = at<double>(smem, L.c);
    double* dv = at<double>(smem, L.l);
    double* P = at<double>(smem, L.blk);  // [6][kR] raw panel columns
    double* Wp = P + 6 * kR;              // [kR][6] W rows
    double* Lp = Wp + 6 * kR;             // [kR][6] L rows
    int* s_fail = at<int>(smem, L.perm);
    double v[RPT][CPT];
#pragma unroll
    for (int a = 0; a < RPT; ++a) {
        const int i = ty + kGrid * a;
#pragma unroll
        for (int b = 0; b < CPT; ++b) {
            const int j = tx + kGrid * b;
            double x = 0.0;
            if (j <= i && j < np && i <= np) x = i < np ? sys[j * np - j * (j - 1) / 2 + (i - j)] : sys[nent_of(np) + j];
            v[a][b] = x;
        }
    }
    if (tid == 0) *s_fail = 0;
    // the first block's raw columns
#pragma unroll
    for (int b = 0; b < CPT; ++b) {
        const int j = tx + kGrid * b;
        if (j < 6 && j < np) {
#pragma unroll
            for (int a = 0; a < RPT; ++a) {
                const int i = ty + kGrid * a;
                if (i >= 0 && i <= np) P[j * kR + i] = v[a][b];
            }
        }
    }
    __syncthreads();
    SOLVE_PROBE(0)
    for (int k0 = 0; k0 < np; k0 += 6) {
        const int kn = k0 + 6;
        // ---- panel: row threads ----
        const int i = k0 + tid;
        if (i <= np) {
            // diagonal block LDL^T in registers: l[r][m] (r > m), d[m]
            double a6[6][6], d[6], id[6];
#pragma unroll
            for (int r = 0; r < 6; ++r)
#pragma unroll
                for (int m = 0; m <= r; ++m) a6[r][m] = P[m * kR + k0 + r];
#pragma unroll
            for (int m = 0; m < 6; ++m) {
                double dm = a6[m][m];
#pragma unroll
                for (int q = 0; q < m; ++q) dm -= a6[m][q] * (a6[m][q] * d[q]);
                d[m] = dm;
                id[m] = dm != 0.0 ? rcp_nr(dm) : 0.0;
#pragma unroll
                for (int r = m + 1; r < 6; ++r) {
                    double s = a6[r][m];
#pragma unroll
                    for (int q = 0; q < m; ++q) s -= a6[r][q] * (a6[m][q] * d[q]);
                    a6[r][m] = s * id[m];  // l_rm
                }
            }
            if (i < kn) {  // a diagonal-block row: its L entries and pivot are final
#pragma unroll
                for (int rr = 0; rr < 6; ++rr) {  // rr == tid (static register indices)
                    if (rr != tid) continue;
#pragma unroll
                    for (int m = 0; m < rr; ++m) A[i * ld + k0 + m] = fabs(d[m]) > DBL_MIN ? a6[rr][m] : 0.0;
                    dv[i] = d[rr];
                    dinv[i] = id[rr];
                    bool bad = !(d[rr] >= 0.0) || !isfinite(d[rr]);
                    // zero pivot: valid only with a zero column below (LDLT::info())
#pragma unroll
                    for (int q = rr + 1; q < 6; ++q) bad = bad || (d[rr] == 0.0 && a6[q][rr] != 0.0);
                    if (bad) *s_fail = 1;
                }
            } else {  // a panel row (or the rhs row): W_i = A_iK L_KK^-T, L_iK = W_i D^-1
                double w[6];
#pragma unroll
                for (int q = 0; q < 6; ++q) {
                    double s = P[q * kR + i];
#pragma unroll
                    for (int m = 0; m < q; ++m) s -= w[m] * a6[q][m];
                    w[q] = s;
                }
                const int r = i - kn;
                bool bad = false;
#pragma unroll
                for (int q = 0; q < 6; ++q) {
                    const double lq = fabs(d[q]) > DBL_MIN ? w[q] * id[q] : 0.0;
                    bad = bad || (d[q] == 0.0 && w[q] != 0.0 && i < np);
                    Wp[r * 6 + q] = w[q];
                    Lp[r * 6 + q] = lq;
                    A[i * ld + k0 + q] = lq;
                }
                if (bad) *s_fail = 1;
            }
        }
        __syncthreads();
        if (kn >= np) break;
        // ---- trailing update A_ij -= L_iK . W_jK for i, j >= k0 + 6 ----
        double lr[RPT][6], wc[CPT][6];
#pragma unroll
        for (int a = 0; a < RPT; ++a) {  // 16-byte loads: a row is 48 B
            const int ia = ty + kGrid * a - kn;
            const bool in = ia >= 0 && ia <= np - kn;
            const double2* src = reinterpret_cast<const double2*>(Lp + (in ? ia : 0) * 6);
#pragma unroll
            for (int h = 0; h < 3; ++h) {
                const double2 t = in ? src[h] : make_double2(0.0, 0.0);
                lr[a][2 * h] = t.x;
                lr[a][2 * h + 1] = t.y;
            }
        }
#pragma unroll
        for (int b = 0; b < CPT; ++b) {
            const int jb = tx + kGrid * b - kn;
            const bool in = jb >= 0 && jb < np - kn;
            const double2* src = reinterpret_cast<const double2*>(Wp + (in ? jb : 0) * 6);
#pragma unroll
            for (int h = 0; h < 3; ++h) {
                const double2 t = in ? src[h] : make_double2(0.0, 0.0);
                wc[b][2 * h] = t.x;
                wc[b][2 * h + 1] = t.y;
            }
        }
#pragma unroll
        for (int a = 0; a < RPT; ++a)
#pragma unroll
            for (int b = 0; b < CPT; ++b) {
                double s = v[a][b];
#pragma unroll
                for (int q = 0; q < 6; ++q) s -= lr[a][q] * wc[b][q];
                v[a][b] = s;
            }
        // the next block's raw columns kn .. kn+5 (rows >= kn)
#pragma unroll
        for (int b = 0; b < CPT; ++b) {
            const int j = tx + kGrid * b;
            if (j >= kn && j < kn + 6 && j < np) {
#pragma unroll
                for (int a = 0; a < RPT; ++a) {
                    const int ii = ty + kGrid * a;
                    if (ii >= kn && ii <= np) P[(j - kn) * kR + ii] = v[a][b];
                }
            }
        }
        __syncthreads();
    }
    SOLVE_PROBE(1)
    if (*((volatile int*)s_fail)) return false;  // uniform: read after the loop's last barrier
    SOLVE_PROBE(2)
    if (warp == 0) {
        __syncwarp();
        const double* z = A + np * ld;
        double z0 = lane < np ? z[lane] : 0.0, z1 = lane + 32 < np ? z[lane + 32] : 0.0;
        double z2 = lane + 64 < np ? z[lane + 64] : 0.0;
        for (int i = np - 1; i >= 0; --i) {
            const int sl = i >> 5;
            const double own = sl == 0 ? z0 : sl == 1 ? z1 : z2;
            const double xi = __shfl_sync(0xffffffffu, own, i & 31);
            const double* Li = A + i * ld;
            if (lane < i) z0 -= Li[lane] * xi;
            if (lane + 32 < i) z1 -= Li[lane + 32] * xi;
            if (lane + 64 < i) z2 -= Li[lane + 64] * xi;
        }
        if (lane < np) x_out[lane] = z0;
        if (lane + 32 < np) x_out[lane + 32] = z1;
        if (lane + 64 < np) x_out[lane + 64] = z2;
    }
    __syncthreads();
    SOLVE_PROBE(3)
    return true;
}

__device__ bool ldlt_solve_cta(const double* sys, int np, unsigned char* smem, const Layout& L, double* x_out) {
#ifndef PVO_LDLT_SCALAR
    if (np % 6 == 0) {  // pose systems: 6 columns per pose
        if (np <= 63) return ldlt_solve_blk6<4, 4>(sys, np, smem, L, x_out);
        return ldlt_solve_blk6<7, 6>(sys, np, smem, L, x_out);
    }
#endif
    if (np <= 63) return ldlt_solve_regs<4, 4>(sys, np, smem, L, x_out);  // rows <= 64, columns <= 64
    return ldlt_solve_regs<7, 6>(sys, np, smem, L, x_out);                // np <= 96: rows <= 112, columns <= 96
}

// ---------------------------------------------------------------------------
// P0: frozen targets (bundle_adjust.cpp:288-307) for the edges of [k0, k1)
// ---------------------------------------------------------------------------
__device__ void phase_freeze(const BAParams& a, const double* poses, int k0, int k1) {
    const int e0 = a.patch_edge_begin[k0], e1 = a.patch_edge_begin[k1];
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) freeze_edge(a, poses, e);
}

// Per-warp int block: [0]=si [1]=ne [2]=dslot [3]=k, [4..4+16)=p2e, then next[32]
__device__ inline int* warp_ints(unsigned char* smem, const Layout& L, int w) {
    return at<int>(smem, L.ints) + w * kWarpInts;
}

// ---------------------------------------------------------------------------
// P1: assembly of the CTA's patches into its partial reduced system.
// ---------------------------------------------------------------------------
__device__ void phase_assemble(const BAParams& a, unsigned char* smem, const Layout& L, const double* poses,
                               const double* mats, int k0, int k1, int np, bool poses_frozen, double lambda,
                               double* part, int* status) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nent = nent_of(np);
    const Cam K{a.K[0], a.K[1], a.K[2], a.K[3]};
    double* S = at<double>(smem, L.S);
    double* rhs = at<double>(smem, L.rhs);
    const unsigned* abt = at<unsigned>(smem, L.ab);
    for (int i = tid; i < nent; i += kThreads) S[i] = 0.0;
    for (int i = tid; i < np; i += kThreads) rhs[i] = 0.0;
    double wr_sum = 0.0, wr_w = 0.0;  // lane 0 of each warp keeps its running sums
    __syncthreads();

    for (int batch = k0; batch < k1; batch += kWarps) {
        const int k = batch + warp;
        int* wi = warp_ints(smem, L, warp);
        double* rec = at<double>(smem, L.rec) + (size_t)warp * kMaxEdges * kRec;
        double* v = at<double>(smem, L.vb) + (size_t)warp * 2 * np;
        double* bvec = v + np;
        double* sc = at<double>(smem, L.scal) + warp * kScal;
        if (k < k1) {
            // global inputs of the patch and of the lane's edge, all issued before
            // the first shared-memory store (which would otherwise order them)
            const int eb = a.patch_edge_begin[k], ne = a.patch_edge_begin[k + 1] - eb;
            const int src = a.patch_src[k];
            const int dslot = a.depth_slot[k];
            const double d = a.depth[k];
            const double* px = a.patch_x + 9 * (size_t)k;
            const double* py = a.patch_y + 9 * (size_t)k;
            const bool has_edge = lane < ne;
            const int e = eb + lane;
            const int tgt = has_edge ? a.e_pose[e] : 0;
            const double et0 = has_edge ? a.e_target[2 * e] : 0.0, et1 = has_edge ? a.e_target[2 * e + 1] : 0.0;
            const double ew0 = has_edge ? a.e_weight[2 * e] : 0.0, ew1 = has_edge ? a.e_weight[2 * e + 1] : 0.0;
            const double px4 = px[4], py4 = py[4];
            const int si = poses_frozen ? -1 : a.pose_free_slot[src];
            int sj = (has_edge && !poses_frozen) ? a.pose_free_slot[tgt] : -1;
            for (int i = lane; i < 2 * np; i += 32) v[i] = 0.0;
            double h = 0, bd = 0, vs[6] = {0, 0, 0, 0, 0, 0}, bs[6] = {0, 0, 0, 0, 0, 0};
            double wrs = 0, wrw = 0;
            if (has_edge) {
                const SE3 pi = se3_load(poses + 7 * src);
                const SE3 pj = se3_load(poses + 7 * tgt);
                const Relative rel = rel_from_mats(mats + 12 * src, mats + 12 * tgt);
                const CenterJac J = center_jacobians(rel, K, d, px4, py4);
                const double r0 = J.cu - et0, r1 = J.cv - et1;
                if (!isfinite(r0) || !isfinite(r1)) set_status(status, kDevNonFiniteResidual);
                double w0 = J.behind ? 0.0 : ew0;
                double w1 = J.behind ? 0.0 : ew1;
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
                R[kW] = w0;
                R[kW + 1] = w1;
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
                const double rx = cu - et0, ry = cv - et1;
                const double wx = behind ? 0.0 : ew0;
                const double wy = behind ? 0.0 : ew1;
                wrs = wx * rx * rx + wy * ry * ry;
                wrw = wx + wy;
            }
            __syncwarp();
            // 6x6 source-pose block sum_e Gs^T W Gs of this patch (upper triangle on
            // lanes 0..20, mirrored), so the CTA accumulation below is O(1) per entry
            if (si >= 0 && lane < 21) {
                int ra = 0, rem = lane;
                while (rem >= 6 - ra) {
                    rem -= 6 - ra;
                    ++ra;
                }
                const int rb = ra + rem;
                double val = 0.0;
                for (int l = 0; l < ne; ++l) {
                    const double* R = rec + l * kRec;
                    val += (R[kGs + ra] * R[kW]) * R[kGs + rb] + (R[kGs + 6 + ra] * R[kW + 1]) * R[kGs + 6 + rb];
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
            // per-edge target blocks: with distinct targets (one edge per (patch, frame):
            // every window problem) each lane adds its own edge's block at once; a
            // repeated target (possible in a flat problem) serialises in edge order
            const bool has_t = sj >= 0;
            const unsigned same = __match_any_sync(0xffffffffu, sj);  // every lane (no short-circuit)
            const unsigned with_t = __ballot_sync(0xffffffffu, has_t);
            const bool dup = has_t && __popc(same & with_t) > 1;
            const bool distinct = !__any_sync(0xffffffffu, dup);
            if (distinct) {
                if (has_t) {
                    const double* R = rec + lane * kRec;
#pragma unroll
                    for (int c = 0; c < 6; ++c) {
                        const double g0 = R[kJt + c] * R[kW], g1 = R[kJt + 6 + c] * R[kW + 1];
                        v[6 * sj + c] += g0 * R[kJd] + g1 * R[kJd + 1];
                        bvec[6 * sj + c] += -(g0 * R[kR] + g1 * R[kR + 1]);
                    }
                }
                __syncwarp();
            } else {
                for (int l = 0; l < ne; ++l) {
                    const int sjl = __shfl_sync(0xffffffffu, sj, l);
                    if (sjl >= 0 && lane < 6) {
                        const double* R = rec + l * kRec;
                        const double g0 = R[kJt + lane] * R[kW], g1 = R[kJt + 6 + lane] * R[kW + 1];
                        v[6 * sjl + lane] += g0 * R[kJd] + g1 * R[kJd + 1];
                        bvec[6 * sjl + lane] += -(g0 * R[kR] + g1 * R[kR + 1]);
                    }
                    __syncwarp();
                }
            }
            if (si >= 0 && lane < 6) {
                v[6 * si + lane] += vs[lane];
                bvec[6 * si + lane] += bs[lane];
            }
            // target-pose -> edge chains (sj >= 0: an active edge with its own free
            // target block; the lanes' slots arrive by shuffle, no global re-reads)
            int* p2e = wi + 4;
            int* nxt = wi + 4 + kMaxFree;
            for (int i = lane; i < kMaxFree; i += 32) p2e[i] = -1;
            __syncwarp();
            if (distinct) {  // one-edge chains: every lane sets its own
                if (lane < ne) nxt[lane] = -1;
                if (has_t) p2e[sj] = lane;
            } else {
                for (int l = ne - 1; l >= 0; --l) {
                    const int sjl = __shfl_sync(0xffffffffu, sj, l);
                    if (lane == 0) {
                        nxt[l] = -1;
                        if (sjl >= 0) {
                            nxt[l] = p2e[sjl];
                            p2e[sjl] = l;
                        }
                    }
                }
            }
            __syncwarp();
            {  // the free target poses with an edge chain, ascending (a ballot compaction)
                int* tl = nxt + kMaxEdges;
                const bool used = lane < kMaxFree && p2e[lane < kMaxFree ? lane : 0] >= 0;
                const unsigned um = __ballot_sync(0xffffffffu, used);
                if (used) tl[__popc(um & ((1u << lane) - 1))] = lane;
                if (lane == 0) tl[kMaxFree] = __popc(um);
            }
            if (lane == 0) {
                wi[0] = si;
                wi[1] = ne;
                wi[2] = dslot;
                wi[3] = k;
                const double hd = h + lambda;  // h_dd + damping (bundle_adjust.cpp:185)
                sc[0] = hd;
                sc[1] = bd;
                sc[2] = 1.0 / hd;  // d_inv (bundle_adjust.cpp:69)
                if (dslot >= 0 && !(hd > 0)) set_status(status, kDevNonPositiveDepth);
                wr_sum += wrs;
                wr_w += wrw;
            }
        } else if (lane == 0) {
            wi[1] = -1;
        }
        __syncthreads();
        if (a.phase_clocks && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0 && batch == k0) a.phase_clocks[15 * 8 + 0] = clock64();

        // ---- ordered accumulation of the batch into the CTA system ----
        // (i) the patches' block terms, patch by patch in order: within a patch
        // every entry of S is touched at most once (the (s,s) block, and per
        // free target t with an edge chain the (s,t) and (t,t) blocks), so the
        // whole CTA works on one patch at a time
        int nw = 0;
        while (nw < kWarps && warp_ints(smem, L, nw)[1] >= 0) ++nw;
        auto ut6 = [](int u, int& r, int& c) {  // u-th entry of a 6x6 upper triangle, row-major
            r = 0;
            while (u >= 6 - r) {
                u -= 6 - r;
                ++r;
            }
            c = r + u;
        };
        auto packed = [&](int i, int j) { return i * np - i * (i - 1) / 2 + (j - i); };  // i <= j
        for (int w = 0; w < nw; ++w) {
            const int* wiw = warp_ints(smem, L, w);
            const int si = wiw[0];
            const int* p2e = wiw + 4;
            const int* nxt = p2e + kMaxFree;
            const int* tl = nxt + kMaxEdges;
            const int ntl = tl[kMaxFree];
            const double* recw = at<double>(smem, L.rec) + (size_t)w * kMaxEdges * kRec;
            const double* scw = at<double>(smem, L.scal) + w * kScal;
            const int nss = si >= 0 ? 21 : 0, per_t = si >= 0 ? 57 : 21;
            const int nitems = nss + ntl * per_t;
            for (int it = tid; it < nitems; it += kThreads) {
                int A, B, ra, rb;
                double val = 0.0;
                if (it < nss) {
                    ut6(it, ra, rb);
                    A = B = si;
                    val = scw[4 + 6 * ra + rb];
                } else {
                    const int j = it - nss, t = tl[j / per_t], r = j - (j / per_t) * per_t;
                    int oa, ob;
                    if (si >= 0 && r < 36) {  // (s, t): Gs on the source side, Jt on the target side
                        ra = r / 6;
                        rb = r - 6 * ra;
                        A = si < t ? si : t;
                        B = si < t ? t : si;
                        oa = (si < t ? kGs : kJt) + ra;
                        ob = (si < t ? kJt : kGs) + rb;
                    } else {  // (t, t)
                        ut6(si >= 0 ? r - 36 : r, ra, rb);
                        A = B = t;
                        oa = kJt + ra;
                        ob = kJt + rb;
                    }
                    for (int l = p2e[t]; l >= 0; l = nxt[l]) {  // one edge unless an edge repeats
                        const double* R = recw + l * kRec;
                        val += (R[oa] * R[kW]) * R[ob] + (R[oa + 6] * R[kW + 1]) * R[ob + 6];
                    }
                }
                S[packed(6 * A + ra, 6 * B + rb)] += val;
            }
            __syncthreads();
        }
        // (ii) the depth-Schur terms of all the batch's patches, S -= sum_w (v_w / h_w) v_w^T,
        // on 4x4 register tiles of the upper triangle
        {
            const int nt4 = (np + 3) >> 2;
            for (int t = tid; t < nt4 * (nt4 + 1) / 2; t += kThreads) {
                int ti = 0, u = t;
                while (u >= nt4 - ti) {
                    u -= nt4 - ti;
                    ++ti;
                }
                const int tj = ti + u, i0 = 4 * ti, j0 = 4 * tj;
                double acc[4][4] = {};
                for (int w = 0; w < nw; ++w) {
                    if (warp_ints(smem, L, w)[2] < 0) continue;  // depth fixed: no Schur term
                    const double* vw = at<double>(smem, L.vb) + (size_t)w * 2 * np;
                    const double hinv = at<double>(smem, L.scal)[w * kScal + 2];
                    double vi[4], vj[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        vi[q] = i0 + q < np ? vw[i0 + q] * hinv : 0.0;
                        vj[q] = j0 + q < np ? vw[j0 + q] : 0.0;
                    }
#pragma unroll
                    for (int r = 0; r < 4; ++r)
#pragma unroll
                        for (int c = 0; c < 4; ++c) acc[r][c] += vi[r] * vj[c];
                }
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const int i = i0 + r, j = j0 + c;
                        if (i < np && j < np && i <= j) S[packed(i, j)] -= acc[r][c];
                    }
            }
        }
        for (int i = tid; i < np; i += kThreads) {
            double racc = rhs[i];
            for (int w = 0; w < nw; ++w) {
                const bool dfree = warp_ints(smem, L, w)[2] >= 0;
                const double* vw = at<double>(smem, L.vb) + (size_t)w * 2 * np;
                const double* scw = at<double>(smem, L.scal) + w * kScal;
                double r = vw[np + i];
                if (dfree) r -= vw[i] * (scw[2] * scw[1]);
                racc += r;
            }
            rhs[i] = racc;
        }
        // stash the patches' Schur data for the back-substitution
        for (int w = 0; w < nw; ++w) {
            const int kw = warp_ints(smem, L, w)[3];
            const double* vw = at<double>(smem, L.vb) + (size_t)w * 2 * np;
            const double* scw = at<double>(smem, L.scal) + w * kScal;
            for (int i = tid; i < np; i += kThreads) a.patch_v[(size_t)kw * np + i] = vw[i];
            if (tid == 0) {
                a.patch_h[kw] = scw[0];
                a.patch_bd[kw] = scw[1];
            }
        }
        __syncthreads();
    }
    if (a.phase_clocks && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) a.phase_clocks[15 * 8 + 1] = clock64();
    // ---- write the CTA partial ----
    double* wr = at<double>(smem, L.wr);
    if (lane == 0) {
        wr[warp * 2] = wr_sum;
        wr[warp * 2 + 1] = wr_w;
    }
    __syncthreads();
    for (int i = tid; i < nent; i += kThreads) part[i] = S[i];
    for (int i = tid; i < np; i += kThreads) part[nent + i] = rhs[i];
    if (tid == 0) {
        double ws = 0, ww = 0;
        for (int w = 0; w < kWarps; ++w) {
            ws += wr[2 * w];
            ww += wr[2 * w + 1];
        }
        part[nent + np] = ws;
        part[nent + np + 1] = ww;
    }
}

// ---------------------------------------------------------------------------
// P4: depth back-substitution + residual at the candidate state.
// ---------------------------------------------------------------------------
__device__ void phase_update(const BAParams& a, unsigned char* smem, const Layout& L, const double* cand,
                             const double* cmats, int k0, int k1, int np, const double* delta, double* part_tail,
                             int* status) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const Cam K{a.K[0], a.K[1], a.K[2], a.K[3]};
    double* wr = at<double>(smem, L.wr);
    double wr_sum = 0, wr_w = 0;
    for (int k = k0 + warp; k < k1; k += kWarps) {
        // every global input of the patch and of the lane's edge is loaded up
        // front (independent loads in flight together), then used
        const int dslot = a.depth_slot[k];
        const double d0 = a.depth[k];
        const int eb = a.patch_edge_begin[k], ne = a.patch_edge_begin[k + 1] - eb;
        const int src = a.patch_src[k];
        const double ph = a.patch_h[k], pbd = a.patch_bd[k];
        double pv[kMaxNp / 32];
#pragma unroll
        for (int u = 0; u < kMaxNp / 32; ++u) {
            const int i = lane + 32 * u;
            pv[u] = i < np ? a.patch_v[(size_t)k * np + i] : 0.0;
        }
        const int e = eb + lane;
        const bool has_edge = lane < ne;  // <= 32 edges per patch (kMaxEdges)
        const int tgt = has_edge ? a.e_pose[e] : 0;
        const double t0 = has_edge ? a.e_target[2 * e] : 0.0, t1 = has_edge ? a.e_target[2 * e + 1] : 0.0;
        const double w0 = has_edge ? a.e_weight[2 * e] : 0.0, w1 = has_edge ? a.e_weight[2 * e + 1] : 0.0;
        double dnew = d0;
        if (dslot >= 0) {
            double dot = 0.0;
#pragma unroll
            for (int u = 0; u < kMaxNp / 32; ++u)
                if (lane + 32 * u < np) dot += pv[u] * delta[lane + 32 * u];
            dot = warp_sum(dot);
            const double inv_h = 1.0 / ph;
            const double dd = inv_h * (pbd - dot);  // bundle_adjust.cpp:88-89
            if (!isfinite(dd) && lane == 0) set_status(status, kDevNonFiniteDepth);
            dnew = fmax(0.0, dnew + dd);  // bundle_adjust.cpp:211
        }
        if (lane == 0) a.cand_depth[k] = dnew;
        const SE3 pi = se3_load(cand + 7 * src);
        double ws = 0, ww = 0;
        if (has_edge) {
            const SE3 pj = se3_load(cand + 7 * tgt);
            double cu, cv;
            bool behind;
            const Relative rel = rel_from_mats(cmats + 12 * src, cmats + 12 * tgt);
            center_behind(se3_equal(pi, pj), rel, K, a.patch_x + 9 * (size_t)k, a.patch_y + 9 * (size_t)k, dnew, &cu,
                          &cv, &behind);
            const double rx = cu - t0, ry = cv - t1;
            const double wx = behind ? 0.0 : w0;
            const double wy = behind ? 0.0 : w1;
            ws += wx * rx * rx + wy * ry * ry;
            ww += wx + wy;
        }
        ws = warp_sum(ws);
        ww = warp_sum(ww);
        wr_sum += ws;
        wr_w += ww;
    }
    if (lane == 0) {
        wr[warp * 2] = wr_sum;
        wr[warp * 2 + 1] = wr_w;
    }
    __syncthreads();
    if (tid == 0) {
        double ws = 0, ww = 0;
        for (int w = 0; w < kWarps; ++w) {
            ws += wr[2 * w];
            ww += wr[2 * w + 1];
        }
        part_tail[2] = ws;
        part_tail[3] = ww;
    }
}

// The window loop.  Single window: a cooperative grid of G CTAs (grid-wide
// barriers).  Batch of independent windows (pvo_batch_*): one CTA per window
// (blockIdx.y), so every barrier is a CTA barrier and windows never wait for
// each other (each keeps its own guard / attempt sequence).
__device__ __forceinline__ void window_sync(bool batched) {
    if (batched)
        __syncthreads();
    else
        cg::this_grid().sync();
}

__device__ void ba_window_body(const BAParams& a, bool batched) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int np_full = 6 * a.n_free_poses;
    const int G = batched ? 1 : gridDim.x, b = batched ? 0 : blockIdx.x, tid = threadIdx.x;
    const int k0 = (int)((long long)a.n_patches * b / G);
    const int k1 = (int)((long long)a.n_patches * (b + 1) / G);
    const Layout L = make_layout(np_full, a.n_poses);
    double* pose = at<double>(smem, L.pose);
    double* cand = at<double>(smem, L.cand);
    double* delta = at<double>(smem, L.delta);
    double* rmat = at<double>(smem, L.rmat);
    double* rmatc = at<double>(smem, L.rmatc);
    const size_t pstride = (size_t)nent_of(np_full) + np_full + 4;

    // entry -> (row, col, row pose block, col pose block) table of the joint
    // system; CTA copy of the pose state and its rotation matrices
    {
        unsigned* abt = at<unsigned>(smem, L.ab);
        const int nent = nent_of(np_full);
        auto row_base = [&](int r) { return r * np_full - r * (r - 1) / 2; };
        for (int ent = tid; ent < nent; ent += kThreads) {
            // row of a packed upper-triangle entry: closed form, then an exact fix-up
            const float q = (float)(2 * np_full + 1);
            int ia = (int)((q - sqrtf(q * q - 8.0f * (float)ent)) * 0.5f);
            ia = max(0, min(ia, np_full - 1));
            while (ia > 0 && row_base(ia) > ent) --ia;
            while (ia + 1 < np_full && row_base(ia + 1) <= ent) ++ia;
            const int base = row_base(ia);
            const int ib = ia + ent - base;
            abt[ent] = (unsigned)ia | ((unsigned)ib << 8) | ((unsigned)(ia / 6) << 16) | ((unsigned)(ib / 6) << 24);
        }
        for (int i = tid; i < 7 * a.n_poses; i += kThreads) pose[i] = a.poses[i];
    }
    __syncthreads();
    pose_mats(pose, rmat, a.n_poses);
    __syncthreads();
    phase_freeze(a, pose, k0, k1);
    __syncthreads();

    int attempt_no = 0;  // global attempt counter -> buffer parity
    const int total_iters = a.structure_only + a.iterations;
    for (int it = 0; it < total_iters; ++it) {
        const bool structure = it < a.structure_only;
        const int np = structure ? 0 : np_full;
        const int nent = nent_of(np);
        int attempt = 0;
        for (;;) {
            const int buf = attempt_no & 1;
            int* status = a.status2 + buf;
            double* partials = a.partials + (size_t)buf * G * pstride;
            const double lambda =
                attempt == 0 ? a.damping : a.damping * (attempt == 1 ? 1e3 : attempt == 2 ? 1e6 : 1e9);
            double* part = partials + (size_t)b * pstride;
            const bool clk = a.phase_clocks && b == 0 && tid == 0 && blockIdx.y == 0;
            long long* pc = a.phase_clocks ? a.phase_clocks + 8 * (attempt_no < 15 ? attempt_no : 15) : nullptr;
            if (clk) pc[0] = clock64();
            phase_assemble(a, smem, L, pose, rmat, k0, k1, np, structure, lambda, part, status);
            if (clk) pc[1] = clock64();
            window_sync(batched);
            if (clk) pc[2] = clock64();
            // P2: ordered reduction of the CTA partials (+ damping on the diagonal):
            // one warp per entry, lanes over CTAs in fixed order, shuffle tree
            {
                const unsigned* abt = at<unsigned>(smem, L.ab);
                const int lane = tid & 31;
                for (int ent = (b * kThreads + tid) >> 5; ent < nent + np; ent += (G * kThreads) >> 5) {
                    // the lane's CTA partials: all loads in flight first (G <= 160),
                    // then summed in CTA order (the same order as a plain loop)
                    double v[5];
#pragma unroll
                    for (int u = 0; u < 5; ++u) {
                        const int c = lane + 32 * u;
                        v[u] = c < G ? partials[(size_t)c * pstride + ent] : 0.0;
                    }
                    double acc = 0.0;
#pragma unroll
                    for (int u = 0; u < 5; ++u)
                        if (lane + 32 * u < G) acc += v[u];
                    for (int c = lane + 160; c < G; c += 32) acc += partials[(size_t)c * pstride + ent];
                    acc = warp_sum(acc);
                    if (lane == 0) {
                        if (ent < nent) {
                            const unsigned ab = abt[ent];
                            if ((ab & 0xff) == ((ab >> 8) & 0xff)) acc += lambda;
                        }
                        a.system[ent] = acc;
                    }
                }
            }
            if (clk) pc[3] = clock64();
            window_sync(batched);
            if (clk) pc[4] = clock64();
            // P3: every CTA solves the pose system and retracts its pose copy
            if (np > 0) {
                if (!ldlt_solve_cta(a.system, np, smem, L, delta)) {
                    if (tid == 0) set_status(status, kDevFactorization);
                } else {
                    bool bad = false;
                    for (int i = tid; i < np; i += kThreads) bad = bad || !isfinite(delta[i]);
                    if (__syncthreads_or(bad) && tid == 0) set_status(status, kDevNonFinitePose);
                }
            }
            if (clk && attempt_no == 0) a.phase_clocks[15 * 8 + 2] = clock64();  // solve done (first attempt)
            for (int i = tid; i < a.n_poses; i += kThreads) {
                const int slot = structure ? -1 : a.pose_free_slot[i];
                const SE3 p = se3_load(pose + 7 * i);
                if (slot >= 0 && np > 0) {
                    double xi[6];
#pragma unroll
                    for (int c = 0; c < 6; ++c) xi[c] = delta[6 * slot + c];
                    se3_store(se3_retract(p, xi), cand + 7 * i);  // bundle_adjust.cpp:202-207
                } else {
                    se3_store(p, cand + 7 * i);
                }
            }
            __syncthreads();
            pose_mats(cand, rmatc, a.n_poses);
            __syncthreads();
            if (clk) pc[5] = clock64();
            phase_update(a, smem, L, cand, rmatc, k0, k1, np, delta, part + nent + np, status);
            if (clk) pc[6] = clock64();
            window_sync(batched);
            if (clk) pc[7] = clock64();
            // P5: identical decision in every CTA
            const int st = *((volatile int*)status);
            if (st != 0) {
                if (b == 0 && tid == 0) atomicOr(a.status, st);
                return;
            }
            // residual sums over the CTA partials: warp 0, fixed lane order + shuffle tree
            double* s_res = at<double>(smem, L.flags);
            if (tid < 32) {
                double q[4] = {0, 0, 0, 0};
                double v[5][4];  // loads first, then the sums in CTA order
#pragma unroll
                for (int r = 0; r < 5; ++r) {
                    const int c = tid + 32 * r;
#pragma unroll
                    for (int u = 0; u < 4; ++u) v[r][u] = c < G ? partials[(size_t)c * pstride + nent + np + u] : 0.0;
                }
#pragma unroll
                for (int r = 0; r < 5; ++r)
                    if (tid + 32 * r < G)
#pragma unroll
                        for (int u = 0; u < 4; ++u) q[u] += v[r][u];
                for (int c = tid + 160; c < G; c += 32) {
                    const double* pt = partials + (size_t)c * pstride + nent + np;
#pragma unroll
                    for (int u = 0; u < 4; ++u) q[u] += pt[u];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) q[u] = warp_sum(q[u]);
                if (tid == 0)
                    for (int u = 0; u < 4; ++u) s_res[u] = q[u];
            }
            __syncthreads();
            const double sb = s_res[0], wb = s_res[1], sa = s_res[2], wa = s_res[3];
            __syncthreads();
            const double before = wb > 0 ? sqrt(sb / wb) : 0.0;
            const double after = wa > 0 ? sqrt(sa / wa) : 0.0;
            const double thr = 1.5 * before + 1e-9;
            ++attempt_no;
            if (b == 0 && tid == 0 && a.attempts) *a.attempts = attempt_no;
            bool accept, reject = false;
            if (structure || a.gn_step_mode) {
                accept = true;
            } else if (attempt == 0) {
                accept = !(after > thr);  // bundle_adjust.cpp:330
            } else {
                accept = after <= thr;  // bundle_adjust.cpp:339-340
            }
            if (!accept && !structure && !a.gn_step_mode) {
                if (attempt < 3) {
                    ++attempt;
                    continue;
                }
                reject = true;  // keep the state put (bundle_adjust.cpp:347-353)
            }
            if (b == 0 && tid == 0 && !structure) {
                int n = *a.n_norms;
                if (a.gn_step_mode) {
                    a.residual_norms[n++] = before;
                    a.residual_norms[n++] = after;
                } else {
                    if (n == 0) a.residual_norms[n++] = before;
                    a.residual_norms[n++] = reject ? before : after;
                }
                *a.n_norms = n;
            }
            if (!reject) {
                __syncthreads();
                for (int i = tid; i < 7 * a.n_poses; i += kThreads) pose[i] = cand[i];
                for (int i = tid; i < 12 * a.n_poses; i += kThreads) rmat[i] = rmatc[i];
                for (int k = k0 + tid; k < k1; k += kThreads) a.depth[k] = a.cand_depth[k];
                if (b == 0)
                    for (int i = tid; i < 7 * a.n_poses; i += kThreads) a.poses[i] = cand[i];
                __syncthreads();
            }
            break;
        }
    }
}

__global__ void __launch_bounds__(kThreads, 1) ba_kernel(const __grid_constant__ BAParams a) { ba_window_body(a, false); }

__global__ void __launch_bounds__(kThreads, 1) ba_batch_kernel(const BAParams* __restrict__ windows) {
    __shared__ BAParams sa;  // this CTA's window
    if (threadIdx.x == 0) sa = windows[blockIdx.y];
    __syncthreads();
    ba_window_body(sa, true);
}

// ---------------------------------------------------------------------------
// Debug: dense damped normal equations in the reference's order (tests only).
// ---------------------------------------------------------------------------
__global__ void normal_equations_debug_kernel(BAParams a, double* H, double* bvec) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int np = 6 * a.n_free_poses, nd = a.n_free_depths, n = np + nd;
    const Cam K{a.K[0], a.K[1], a.K[2], a.K[3]};
    for (int i = 0; i < n * n; ++i) H[i] = 0.0;
    for (int i = 0; i < n; ++i) bvec[i] = 0.0;
    for (int e = 0; e < a.n_edges; ++e) {
        const int k = a.e_patch[e];
        const int src = a.patch_src[k], tgt = a.e_pose[e];
        const Relative rel = relative_pose(se3_load(a.poses + 7 * src), se3_load(a.poses + 7 * tgt));
        const CenterJac J = center_jacobians(rel, K, a.depth[k], a.patch_x[9 * k + 4], a.patch_y[9 * k + 4]);
        const double r[2] = {J.cu - a.e_in[2 * e], J.cv - a.e_in[2 * e + 1]};
        const double w[2] = {J.behind ? 0.0 : a.e_weight_in[2 * e], J.behind ? 0.0 : a.e_weight_in[2 * e + 1]};
        if (w[0] == 0.0 && w[1] == 0.0) continue;
        int off[3], cols[3];
        const double* jac[3];
        double jd[12] = {J.dd[0], 0, 0, 0, 0, 0, J.dd[1], 0, 0, 0, 0, 0};
        int nb = 0;
        const int si = a.pose_free_slot[src], sj = a.pose_free_slot[tgt], sd = a.depth_slot[k];
        if (si >= 0) {
            off[nb] = 6 * si;
            cols[nb] = 6;
            jac[nb++] = J.di;
        }
        if (sj >= 0) {
            off[nb] = 6 * sj;
            cols[nb] = 6;
            jac[nb++] = J.dj;
        }
        if (sd >= 0) {
            off[nb] = np + sd;
            cols[nb] = 1;
            jac[nb++] = jd;
        }
        for (int x = 0; x < nb; ++x) {
            for (int ra = 0; ra < cols[x]; ++ra) {
                const double t0 = jac[x][ra] * w[0], t1 = jac[x][6 + ra] * w[1];
                bvec[off[x] + ra] -= t0 * r[0] + t1 * r[1];
                for (int y = 0; y < nb; ++y)
                    for (int rc = 0; rc < cols[y]; ++rc)
                        H[(off[x] + ra) * n + off[y] + rc] += t0 * jac[y][rc] + t1 * jac[y][6 + rc];
            }
        }
    }
    for (int i = 0; i < n; ++i) H[i * n + i] += a.damping;
}

// ---------------------------------------------------------------------------
// schur_solve on dense inputs (bundle_adjust.cpp:62-94), one CTA.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) schur_dense_kernel(int np, int nd, const double* hpp, const double* hpd,
                                                               const double* hdd, const double* bp, const double* bd,
                                                               double* dp, double* dd, double* system, int* status) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x;
    __shared__ int s_bad;
    if (tid == 0) s_bad = 0;
    __syncthreads();
    for (int k = tid; k < nd; k += kThreads)
        if (hdd[k] <= 0) s_bad = 1;
    __syncthreads();
    if (s_bad) {
        if (tid == 0) set_status(status, kDevNonPositiveDepth);
        return;
    }
    const int nent = nent_of(np);
    // reduced camera system S = H_pp - H_pd diag(1/h_dd) H_pd^T and its rhs
    for (int ent = tid; ent < nent; ent += kThreads) {
        int ia = 0, rowlen = np, base = 0;
        while (ent >= base + rowlen) {
            base += rowlen;
            --rowlen;
            ++ia;
        }
        const int ib = ia + ent - base;
        double s = 0;
        for (int k = 0; k < nd; ++k) s += (hpd[ia * nd + k] * (1.0 / hdd[k])) * hpd[ib * nd + k];
        system[ent] = hpp[ia * np + ib] - s;
    }
    for (int i = tid; i < np; i += kThreads) {
        double s = 0;
        for (int k = 0; k < nd; ++k) s += hpd[i * nd + k] * ((1.0 / hdd[k]) * bd[k]);
        system[nent + i] = bp[i] - s;
    }
    __syncthreads();
    if (np > 0) {
        const Layout L = make_layout(np, 0);
        if (!ldlt_solve_cta(system, np, smem, L, dp)) {
            if (tid == 0) set_status(status, kDevFactorization);
            return;
        }
        bool bad = false;
        for (int i = tid; i < np; i += kThreads) bad = bad || !isfinite(dp[i]);
        if (__syncthreads_or(bad)) {
            if (tid == 0) set_status(status, kDevNonFinitePose);
            return;
        }
    }
    for (int k = tid; k < nd; k += kThreads) {
        double s = 0;
        for (int i = 0; i < np; ++i) s += hpd[i * nd + k] * dp[i];
        const double v = (1.0 / hdd[k]) * (bd[k] - s);
        if (!isfinite(v)) set_status(status, kDevNonFiniteDepth);
        dd[k] = v;
    }
}

// camera entry points: thread per item
__global__ void reproject_kernel(int n, int pp, const double* pi, const double* pj, const double* Kd, const double* x,
                                 const double* y, const double* d, double* out, uint8_t* behind) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const SE3 a = se3_load(pi + 7 * i), b = se3_load(pj + 7 * i);
    const Cam K{Kd[0], Kd[1], Kd[2], Kd[3]};
    if (se3_equal(a, b)) {
        for (int k = 0; k < pp; ++k) {
            out[((size_t)i * pp + k) * 2] = x[(size_t)i * pp + k];
            out[((size_t)i * pp + k) * 2 + 1] = y[(size_t)i * pp + k];
        }
        behind[i] = 0;
        return;
    }
    const Relative rel = relative_pose(a, b);
    bool bh = false;
    for (int k = 0; k < pp; ++k) {
        double u, v;
        const double qz = reproject_point(rel, K, d[i], x[(size_t)i * pp + k], y[(size_t)i * pp + k], &u, &v);
        if (qz <= kDepthEpsilon) bh = true;
        out[((size_t)i * pp + k) * 2] = u;
        out[((size_t)i * pp + k) * 2 + 1] = v;
    }
    behind[i] = bh ? 1 : 0;
}

__global__ void jacobians_kernel(int n, int pp, const double* pi, const double* pj, const double* Kd, const double* x,
                                 const double* y, const double* d, double* out, uint8_t* behind) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Cam K{Kd[0], Kd[1], Kd[2], Kd[3]};
    // Patch::center (camera.cpp:34-45)
    double cx, cy;
    const int p = (int)lround(sqrt((double)pp));
    if (p % 2 == 1) {
        cx = x[(size_t)i * pp + pp / 2];
        cy = y[(size_t)i * pp + pp / 2];
    } else {
        double sx = 0, sy = 0;
        for (int k = 0; k < pp; ++k) {
            sx += x[(size_t)i * pp + k];
            sy += y[(size_t)i * pp + k];
        }
        cx = sx / pp;
        cy = sy / pp;
    }
    const Relative rel = relative_pose(se3_load(pi + 7 * i), se3_load(pj + 7 * i));
    const CenterJac J = center_jacobians(rel, K, d[i], cx, cy);
    double* o = out + (size_t)i * 28;
    o[0] = J.cu;
    o[1] = J.cv;
    for (int c = 0; c < 12; ++c) {
        o[2 + c] = J.di[c];
        o[14 + c] = J.dj[c];
    }
    o[26] = J.dd[0];
    o[27] = J.dd[1];
    behind[i] = J.behind ? 1 : 0;
}

}  // namespace

int ba_max_free_poses() { return kMaxFree; }
int ba_max_edges_per_patch() { return kMaxEdges; }
int ba_max_poses() { return kMaxPoses; }

size_t ba_partials_doubles(int n_free_poses, int grid) {
    const int np = 6 * n_free_poses;
    return 2 * (size_t)grid * ((size_t)nent_of(np) + np + 4);  // double-buffered by attempt parity
}

int ba_grid_size(int n_patches, int n_free_poses, int n_poses, int num_sms) {
    const Layout L = make_layout(6 * n_free_poses, n_poses);
    cudaFuncSetAttribute(ba_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ba_kernel, kThreads, L.total) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    // every SM: fewer patches per CTA shortens the ordered per-patch accumulation
    // (C2: 148 CTAs of 6-7 patches vs 120 of 8 -> -17% assembly, measured)
    int g = n_patches;
    if (g > num_sms * per_sm) g = num_sms * per_sm;
    if (g < 1) g = 1;
    return g;
}

cudaError_t launch_ba(BAParams& p, int num_sms, cudaStream_t stream, int* grid_out) {
    if (p.n_free_poses > kMaxFree || p.n_poses > kMaxPoses) return cudaErrorNotSupported;
    const Layout L = make_layout(6 * p.n_free_poses, p.n_poses);
    cudaError_t err = cudaFuncSetAttribute(ba_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
    if (err != cudaSuccess) return err;
    const int grid = ba_grid_size(p.n_patches, p.n_free_poses, p.n_poses, num_sms);
    if (grid_out) *grid_out = grid;
    err = cudaMemsetAsync(p.status2, 0, 2 * sizeof(int), stream);
    if (err != cudaSuccess) return err;
    void* args[] = {&p};
    return cudaLaunchCooperativeKernel((void*)ba_kernel, dim3(grid), dim3(kThreads), args, L.total, stream);
}

size_t ba_batch_smem(int n_free_poses, int n_poses) { return make_layout(6 * n_free_poses, n_poses).total; }

cudaError_t launch_ba_batch(const BAParams* windows_dev, int n_windows, int max_free_poses, int max_poses,
                            cudaStream_t stream) {
    if (n_windows <= 0) return cudaSuccess;
    if (max_free_poses > kMaxFree || max_poses > kMaxPoses) return cudaErrorNotSupported;
    const int smem = (int)ba_batch_smem(max_free_poses, max_poses);
    cudaError_t err = cudaFuncSetAttribute(ba_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    ba_batch_kernel<<<dim3(1, n_windows), kThreads, smem, stream>>>(windows_dev);
    return cudaGetLastError();
}

cudaError_t launch_normal_equations_debug(const BAParams& p, double* h, double* b, cudaStream_t stream) {
    normal_equations_debug_kernel<<<1, 32, 0, stream>>>(p, h, b);
    return cudaGetLastError();
}

cudaError_t launch_schur_dense(int np, int nd, const double* hpp, const double* hpd, const double* hdd,
                               const double* bp, const double* bd, double* dp, double* dd, int* status,
                               cudaStream_t stream) {
    if (np > kMaxNp) return cudaErrorNotSupported;
    const Layout L = make_layout(np, 0);
    cudaError_t err = cudaFuncSetAttribute(schur_dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
    if (err != cudaSuccess) return err;
    // `system` scratch lives right after dd in the caller's buffer (see capi.cu)
    double* system = dd + nd;
    schur_dense_kernel<<<1, kThreads, L.total, stream>>>(np, nd, hpp, hpd, hdd, bp, bd, dp, dd, system, status);
    return cudaGetLastError();
}

cudaError_t launch_reproject(int n, int pp, const double* pi, const double* pj, const double* K, const double* x,
                             const double* y, const double* d, double* out, uint8_t* behind, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    reproject_kernel<<<(n + 127) / 128, 128, 0, stream>>>(n, pp, pi, pj, K, x, y, d, out, behind);
    return cudaGetLastError();
}

cudaError_t launch_jacobians(int n, int pp, const double* pi, const double* pj, const double* K, const double* x,
                             const double* y, const double* d, double* out, uint8_t* behind, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    jacobians_kernel<<<(n + 127) / 128, 128, 0, stream>>>(n, pp, pi, pj, K, x, y, d, out, behind);
    return cudaGetLastError();
}

}  // namespace pvo_dev
