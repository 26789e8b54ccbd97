// kernels.cuh — parameter blocks and launchers of the sm_100a kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace pvo_dev {

// K2: correlation over a batch of edges (corr.cu).
struct CorrParams {
    int n_edges = 0;
    int channels = 0;
    const int* e_patch = nullptr;   // [E] patch index
    const int* e_pose = nullptr;    // [E] target pose index (state mode)
    const int* e_slot = nullptr;    // [E] frame-store slot (explicit mode) or null
    const int* pose_slot = nullptr; // [n_poses] pose -> frame-store slot (state mode)
    // Coordinates: explicit [E][9][2], or reprojected from the state below.
    const double* coords = nullptr;
    const double* poses = nullptr;
    const int* patch_src = nullptr;
    const double* patch_x = nullptr;
    const double* patch_y = nullptr;
    const double* depth = nullptr;
    const double* K = nullptr;      // device [4]
    // Frame store.
    const float* feat0 = nullptr;
    const float* feat1 = nullptr;
    const float* gram0 = nullptr;
    const float* gram1 = nullptr;
    int w0 = 0, h0 = 0, w1 = 0, h1 = 0;
    const float* patch_feats = nullptr;  // [P][2][9][C]
    float* out = nullptr;                // [E][2][9][49]
    int* status = nullptr;               // device status word (1 = non-finite coords)
};

int corr_smem_bytes(int channels);
cudaError_t launch_corr(const CorrParams& p, cudaStream_t stream);
// correlate() of ONE patch of any width p (pp = p * p pixels) evaluated
// directly as the reference does (FP64 samples and sums, corr_exact.cuh):
// feats [2][pp][C], coords [pp][2] -> out [2][pp][49].
cudaError_t launch_corr_direct(int pp, int channels, const float* feats, const double* coords, const float* f0,
                               int w0, int h0, const float* f1, int w1, int h1, float* out, cudaStream_t stream);

// K2 production path (corr_tma.cu): D = 128, TMA pipeline, persistent CTAs.
struct CorrTmaParams {
    int n_edges = 0;
    const int* order = nullptr;     // edge processing order (target-frame sorted) or null
    const int* e_patch = nullptr;
    const int* e_pose = nullptr;
    const int* e_slot = nullptr;    // explicit frame slot per edge, or null (pose_slot[e_pose])
    const int* pose_slot = nullptr;
    const double* coords_in = nullptr;  // explicit [E][9][2] or null (reproject the state)
    const double* poses = nullptr;
    const int* patch_src = nullptr;
    const double* patch_x = nullptr;
    const double* patch_y = nullptr;
    const double* depth = nullptr;
    const double* K = nullptr;
    int w0 = 0, h0 = 0, w1 = 0, h1 = 0;
    const float* patch_feats = nullptr;  // [P][2][9][128]
    int n_patches = 0;
    const float* feat0 = nullptr;        // frame store [slot][H][W][128] (direct re-evaluation
    const float* feat1 = nullptr;        // of outputs whose bilinear taps cancel, corr_exact.cuh)
    float* out = nullptr;
    double* coords = nullptr;     // scratch [E][9][2]
    int* meta = nullptr;          // scratch [list_cap][8]: the tile list (one record per box-sized pixel group)
    int list_cap = 0;             // >= 9 records per (edge, level) tile
    int* ctl = nullptr;           // [list length, queue head, warps done, -], zero between launches
    int* status = nullptr;
};
int corr_tma_smem_bytes();
// Frame-store layouts the TMA kernel reads (encoded by the host):
//   feat{0,1}: [slot][H][W][128] f32, box {16 ch, 9, 9, 1}, 64B swizzle
//   gram{0,1}: [slot][8 planes][H][gram_stride(W)] f32 (planes 0..4 used), box {12, 9, 5, 1}
//   patch:     [P * 2 * 9][128] f32, box {16 ch, 9 rows}
constexpr int kCorrMetaInts = 8;
// maps: feat0, feat1, gram0, gram1, patch, feat0 / feat1 with an 8x8 box (narrow tiles)
int corr_tma_grid(int n_edges, int num_sms);
int corr_tma_list_cap(int n_edges);
cudaError_t launch_corr_tma(const CorrTmaParams& p, const CUtensorMap* maps, int num_sms, cudaStream_t stream);
// Gram records of a level: planes [8][H][gram_stride(W)], rows padded to a 16-byte
// multiple (TMA global strides must be 16-byte multiples); pad cells stay zero.
__host__ __device__ inline int gram_stride(int W) { return (W + 3) & ~3; }
// both levels of a frame in one launch (a level with W * H == 0 is skipped)
cudaError_t launch_gram(const float* feat0, float* gram0, int W0, int H0, const float* feat1, float* gram1, int W1,
                        int H1, int D, int num_sms, cudaStream_t stream);

// Flow-provider measurement per edge (measure.cu): CorrelationFlowProvider::
// measure + propose's per-edge part (flow_provider.cpp:150-312), FP64.
struct MeasureParams {
    int n_edges = 0;
    int channels = 0;                   // <= 128
    const int* e_patch = nullptr;       // [E]
    const int* e_slot = nullptr;        // [E] frame-store slot, or null (pose_slot[e_pose])
    const int* e_pose = nullptr;
    const int* pose_slot = nullptr;
    // explicit centres [E][2] + behind flags, or null: reproject the state below
    const double* centers = nullptr;
    const uint8_t* behind = nullptr;
    const double* poses = nullptr;
    const int* patch_src = nullptr;
    const double* patch_x = nullptr;
    const double* patch_y = nullptr;
    const double* depth = nullptr;
    const double* K = nullptr;          // device [4]
    const float* patch_feats = nullptr; // [P][2][9][C]
    const float* feat0 = nullptr;       // frame store [slot][H][W][C]
    const float* feat1 = nullptr;
    int w0 = 0, h0 = 0, w1 = 0, h1 = 0;
    double* delta = nullptr;            // [E][2]
    double* weight = nullptr;           // [E][2]
    uint8_t* flags = nullptr;           // [E] 1 flat, 2 out of range, 4 behind, 8 non-finite (optional)
    int* status = nullptr;
    // FP64 neighbour-Gram maps of the frame store ([slot][H][W][kGram25], gram25_kernel):
    // when set, the Gram-form measurement kernel runs (else the direct one)
    const double* g25_0 = nullptr;
    const double* g25_1 = nullptr;
    // exact replay list of the Gram-form kernel ([0] count, [1 ..] edges; zero on
    // entry, left zero) and its completion counter; required with g25_0 / g25_1
    int* replay = nullptr;
    int* replay_done = nullptr;
    int* replay_stat = nullptr;  // receives the replayed-edge count of the call
};
cudaError_t launch_measure(const MeasureParams& p, cudaStream_t stream);

// FP64 Gram terms <f(x, y), f(x + dx, y + dy)> of every cell for the 25 offsets
// of the half plane |dx|, |dy| <= 3, (dy > 0) or (dy == 0, dx >= 0) — every
// tap pair of a 4x4 Catmull-Rom footprint (and of a 2x2 bilinear one); 0 when
// the neighbour lies outside the grid.  One level of one frame:
// feat [H][W][C] -> g25 [H][W][kGram25].
constexpr int kGram25 = 25;
cudaError_t launch_gram25(const float* feat, int W, int H, int C, double* g25, cudaStream_t stream);

// correlate_at / correlate_at_cubic at n free level-space points against one
// grid (measure.cu), FP64 like the reference (correlation.cpp:8-35).
struct PointsParams {
    int n = 0, channels = 0, cubic = 0;
    const float* features = nullptr;  // [n][C]
    const double* xy = nullptr;       // [n][2]
    const float* grid = nullptr;      // [H][W][C]
    int W = 0, H = 0;
    double* out = nullptr;            // [n]
};
cudaError_t launch_points(const PointsParams& p, cudaStream_t stream);

// OracleFlowProvider::propose on the resident window (measure.cu): two passes
// around the host-side RNG draws (the reference's sequential mt19937_64 stream).
struct OracleParams {
    int n_edges = 0;
    const int* e_patch = nullptr;
    const int* e_pose = nullptr;
    const int* patch_src = nullptr;
    const double* patch_x = nullptr;
    const double* patch_y = nullptr;
    const double* depth = nullptr;
    const double* poses = nullptr;
    const double* gt_poses = nullptr;   // [N][7] scene poses of the window's pose slots
    const double* gt_depth = nullptr;   // [P] scene inverse depth at each patch centre
    const double* K = nullptr;
    double flow_sigma = 0.0, weight_in_range = 0.99;
    const double* noise = nullptr;      // [E][2] gauss draws (non-behind edges), pass 1
    const uint8_t* outlier = nullptr;   // [E] or null
    const double* outlier_delta = nullptr;
    uint8_t* behind = nullptr;          // [E] pass 0 output
    double* delta = nullptr;            // [E][2]
    double* weight = nullptr;           // [E][2]
};
cudaError_t launch_oracle_propose(const OracleParams& p, int pass, cudaStream_t stream);

// Device-resident patch graph (dgraph.cu): SoA views.
struct DGraphView {
    int F = 0, P = 0;
    int* f_index = nullptr;   // [F] frame indices (ascending = position order)
    double* f_pose = nullptr; // [F][7]
    int* f_slot = nullptr;    // [F] frame-store slot of the frame's pyramid
    int* p_id = nullptr;      // [P] ascending
    int* p_src = nullptr;     // [P] source frame index
    double* p_x = nullptr;    // [P][9]
    double* p_y = nullptr;
    double* p_d = nullptr;    // [P] inverse depth
    float* p_feat = nullptr;  // [P][feat_stride] descriptors (2 levels x 9 px x C)
    size_t feat_stride = 0;
    int* ebeg = nullptr;      // [P+1] CSR into the edge arrays
    int* e_frame = nullptr;   // frame index per edge (ascending inside a patch)
    uint8_t* e_has = nullptr; // revision set
    double* e_rev = nullptr;  // [E][4] delta x y, weight x y
};
// The flattened window, written straight into a context's window / BA buffers.
struct WindowOut {
    int n_poses = 0, n_patches = 0, n_edges = 0;
    int* pose_frames = nullptr;
    double* poses = nullptr;
    uint8_t* fixed = nullptr;
    int* pose_slot = nullptr;
    int* free_slot = nullptr;
    int* n_fixed_dev = nullptr;
    int* patch_ids = nullptr;
    int* patch_src = nullptr;
    double* px = nullptr;
    double* py = nullptr;
    double* depth = nullptr;
    int* depth_slot = nullptr;
    int* edge_begin = nullptr;
    float* patch_feats = nullptr;
    int* e_patch = nullptr;
    int* e_pose = nullptr;
    double* e_delta = nullptr;
    double* e_weight = nullptr;
    int* e_graph = nullptr;   // graph edge index of each window edge
    int* order = nullptr;     // edges sorted by frame-store slot (stable), or null
    int* graph_patch = nullptr;  // [n_patches] graph patch index of each window patch (scratch)
};
cudaError_t dg_scan(int n, const int* in, int* out, cudaStream_t s);
cudaError_t dg_connect(const DGraphView& g, int radius, int pass, int* newlen, const int* new_ebeg, int* out_frame,
                       uint8_t* out_has, double* out_rev, cudaStream_t s);
cudaError_t dg_remove(const DGraphView& g, int frame, int pass, int* keep, int* newlen, const int* new_pidx,
                      const int* new_ebeg, const DGraphView& out, cudaStream_t s);
cudaError_t dg_set_revisions(const DGraphView& g, int n, const int* ids, const int* frames, const double* rev,
                             int* missing, cudaStream_t s);
cudaError_t dg_window_pass0(const DGraphView& g, int window_start, int all, int* inc, int* nrev, cudaStream_t s);
cudaError_t dg_window_used(const DGraphView& g, const int* inc, int all, int* used, cudaStream_t s);
cudaError_t dg_window_write(const DGraphView& g, int first_free, const int* inc, int all, const int* pslot,
                            const int* eoff, const int* used, const int* slot_of_pos, const WindowOut& w, int n_slots,
                            cudaStream_t s);
cudaError_t dg_window_nfixed(const DGraphView& g, int first_free, const int* used, int* n_fixed, cudaStream_t s);
cudaError_t dg_store_revisions(const DGraphView& g, int n_edges, const int* e_graph, const double* delta,
                               const double* weight, cudaStream_t s);
// K: host intrinsics (passed by value to the kernel)
cudaError_t dg_keyframe_flow(const DGraphView& g, int frame_a, int frame_b, const double* K, double* flow, int* ok,
                             double* out, cudaStream_t s);
cudaError_t dg_writeback(const DGraphView& g, int n_poses, const int* pose_frames, const uint8_t* fixed,
                         const double* poses, int n_patches, const int* patch_ids, const double* depth,
                         cudaStream_t s);

// Feature pyramid extraction + patch crop (features.cu; features.cpp:55-235).
cudaError_t launch_extract_features(const float* image, int iw, int ih, int base_channels, float* scratch,
                                    float* level0, float* level1, cudaStream_t s);
size_t extract_scratch_floats(int iw, int ih, int base_channels);
cudaError_t launch_crop_patches(int n, const double* px, const double* py, const float* l0, int w0, int h0,
                                const float* l1, int w1, int h1, int C, float* out, cudaStream_t s);

// Device status word values (ba.cu / corr.cu) -> pvo_status on the host.
enum DevStatus : int {
    kDevOk = 0,
    kDevBadCoords = 1,         // correlate: non-finite reprojection
    kDevNonFiniteResidual = 2, // ba: non-finite residual (bundle_adjust.cpp:147-149)
    kDevNonPositiveDepth = 3,  // schur: non-positive damped depth-block entry
    kDevFactorization = 4,     // schur: reduced camera system factorization failed
    kDevNonFinitePose = 5,     // schur: non-finite pose update
    kDevNonFiniteDepth = 6,    // schur: non-finite depth update
};

// K3-K6: the bundle-adjustment window, one persistent cooperative kernel (ba.cu).
struct BAParams {
    int n_poses = 0, n_patches = 0, n_edges = 0;
    int n_free_poses = 0;      // np = 6 * n_free_poses
    int n_free_depths = 0;
    // problem (device)
    double* poses = nullptr;          // [n_poses][7] current state (updated in place)
    const int* pose_free_slot = nullptr;  // [n_poses] free slot or -1
    const int* patch_src = nullptr;
    const double* patch_x = nullptr;  // [P][9]
    const double* patch_y = nullptr;
    double* depth = nullptr;          // [P] current state (updated in place)
    const int* depth_slot = nullptr;  // [P] free slot or -1
    const int* patch_edge_begin = nullptr;  // [P+1] CSR, edges grouped by patch
    const int* e_patch = nullptr;
    const int* e_pose = nullptr;
    const double* e_in = nullptr;     // [E][2] targets, or deltas when freeze_targets
    const double* e_weight_in = nullptr;  // [E][2]
    double* e_target = nullptr;       // [E][2] scratch: frozen targets
    double* e_weight = nullptr;       // [E][2] scratch: effective weights
    double K[4] = {0, 0, 0, 0};
    int image_w = 0, image_h = 0;
    int freeze_targets = 0;
    double damping = 1e-4;
    int iterations = 0;
    int structure_only = 0;
    int gn_step_mode = 0;   // 1: single gauss_newton_step (no guard, always accept)
    // scratch (device)
    double* cand_poses = nullptr;     // [n_poses][7]
    double* cand_depth = nullptr;     // [P]
    double* patch_v = nullptr;        // [P][np]  H_pd column of each patch
    double* patch_h = nullptr;        // [P] damped h_dd
    double* patch_bd = nullptr;       // [P]
    double* partials = nullptr;       // [grid][nent + np + 4]
    double* system = nullptr;         // [nent + np] reduced S (upper) + rhs
    double* delta = nullptr;          // [np] pose update
    double* residual_norms = nullptr; // [1 + iterations]
    int* n_norms = nullptr;
    int* status = nullptr;
    int* status2 = nullptr;           // [2] per-attempt-parity status words (scratch)
    int* attempts = nullptr;          // [1] Gauss-Newton attempts made (guard retries included)
    long long* phase_clocks = nullptr;  // [16][8] optional: CTA 0 clock64 at phase boundaries
};

// Large-window BA (ba_large.cu): pose systems beyond the single-kernel path.
constexpr int kMaxLocalPoses = 25;  // free poses one patch group may touch (150 local dims)
struct BALargeParams {
    BAParams a;                     // problem + the shared scratch of BAParams
    int structure = 0;              // current iteration is structure-only (set per launch)
    int n_groups = 0;               // patch groups (runs of one source pose, <= 64 patches)
    const int* g_begin = nullptr;   // [G+1] patch ranges
    const int* g_lo = nullptr;      // [G] first free pose slot of the group window
    const int* g_nl = nullptr;      // [G] window dims (6 x poses)
    const long long* g_off = nullptr;  // [G] offset of the group block in g_part (doubles)
    const int* patch_group = nullptr;  // [P]
    int max_nl = 0;                 // widest window (dims)
    int bw = 0;                     // half-bandwidth of the reduced system (scalars)
    double* g_part = nullptr;       // group blocks: local upper triangle + local rhs
    double* g_res = nullptr;        // [G][2] weighted residual sums at the current state
    double* patch_vl = nullptr;     // [P][max_nl] local H_pd column of each patch
    double* A = nullptr;            // [(np+1)][(np+1)] reduced system (row np = rhs), factorised in place
    double* mats = nullptr;         // [N][12] rotation + translation, current state
    double* cmats = nullptr;        // [N][12] ... candidate state
    double* u_res = nullptr;        // [n_update_ctas][2] residual sums at the candidate
    int n_update_ctas = 0;
    int* ctrl = nullptr;            // [4] settled, attempt, failed, pad
    double* dbg_A = nullptr;        // debug: copy of the first reduced system
};
cudaError_t launch_ba_large(BALargeParams& p, int num_sms, cudaStream_t stream, int* launches);
size_t ba_large_solver_smem(int n_free_poses, int bw);
int ba_large_assemble_smem(int nl);

// Returns cudaErrorNotSupported when the shape exceeds the kernel (np > 96
// or a patch with > 32 edges); the host maps that to PVO_UNSUPPORTED.
cudaError_t launch_ba(BAParams& p, int num_sms, cudaStream_t stream, int* grid_out);
int ba_max_free_poses();
int ba_max_edges_per_patch();
size_t ba_partials_doubles(int n_free_poses, int grid);
int ba_grid_size(int n_patches, int n_free_poses, int n_poses, int num_sms);
int ba_max_poses();
// Batch of independent windows: one CTA per window (params array on the device);
// each window's status word is its own (BAParams::status).
cudaError_t launch_ba_batch(const BAParams* windows_dev, int n_windows, int max_free_poses, int max_poses,
                            cudaStream_t stream);
size_t ba_batch_smem(int n_free_poses, int n_poses);

// Debug capture of the damped dense normal equations (sequential, tests only).
cudaError_t launch_normal_equations_debug(const BAParams& p, double* h, double* b, cudaStream_t stream);

// schur_solve on dense inputs (one CTA, np <= 96).
cudaError_t launch_schur_dense(int np, int nd, const double* hpp, const double* hpd, const double* hdd,
                               const double* bp, const double* bd, double* dp, double* dd, int* status,
                               cudaStream_t stream);

// Batched reprojection / Jacobians (camera entry points).
cudaError_t launch_reproject(int n, int pp, const double* pi, const double* pj, const double* K, const double* x,
                             const double* y, const double* d, double* out, uint8_t* behind, cudaStream_t stream);
cudaError_t launch_jacobians(int n, int pp, const double* pi, const double* pj, const double* K, const double* x,
                             const double* y, const double* d, double* out, uint8_t* behind, cudaStream_t stream);

}  // namespace pvo_dev
