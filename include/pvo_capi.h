/*
 * pvo_capi.h — C-ABI of the B200-native DPVO geometric hot path.
 *
 * This is the drop-in boundary.  Every entry point replaces one operator of
 * the reference's C++ API in /root/reference/proj/include/pvo (cited per
 * function as file:line) with plain pointers and sizes: no Eigen, no torch,
 * no C++ types.  Exceptions cannot cross extern "C", so each entry returns a
 * pvo_status that maps 1:1 onto the reference's exception types, and the
 * message is available from pvo_last_error() (thread-local) — see
 * include/pvo/ (C++ headers) for the C++ wrappers that rethrow the same types.
 *
 * Conventions shared by every entry point
 *   pose      7 doubles: quaternion (x, y, z, w) then translation (x, y, z);
 *             world -> camera, Eigen coefficient order (se3.hpp:38-61).
 *   K         4 doubles: fx, fy, cx, cy (camera.hpp:10-23).
 *   patch     p*p x-coordinates and p*p y-coordinates, row-major
 *             (camera.hpp:29-38); camera ops and pvo_correlate take any p,
 *             the batched correlation / BA kernels require p == 3.
 *   features  HWC fp32, data[(y*W + x)*C + c]  (features.hpp:14-36).
 *   corr out  [2][p*p][7][7] fp32 per edge, index ((v*p+u)*7+alpha)*7+beta
 *             (correlation.hpp:17-26).
 *   memspace  PVO_HOST (pageable or pinned host memory, copied inside the
 *             call) or PVO_DEVICE (device pointers, stream-ordered).
 * All compute runs on the GPU owned by the context; there is no CPU
 * fallback: without a usable sm_100 device every compute entry returns
 * PVO_CUDA_ERROR.
 */
#ifndef PVO_CAPI_H
#define PVO_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PVO_OK = 0,
    PVO_INVALID_ARGUMENT = 1, /* std::invalid_argument                          */
    PVO_DEGENERATE = 2,       /* pvo::DegenerateProblem (bundle_adjust.hpp:54-56) */
    PVO_DOMAIN_ERROR = 3,     /* std::domain_error (se3.cpp:58-60)                */
    PVO_OUT_OF_RANGE = 4,     /* std::out_of_range (map::at)                      */
    PVO_CUDA_ERROR = 5,       /* device / driver failure                          */
    PVO_UNSUPPORTED = 6       /* shape outside what the kernels implement         */
} pvo_status;

enum { PVO_HOST = 0, PVO_DEVICE = 1 };

typedef struct pvo_ctx pvo_ctx;     /* device, stream, scratch arena, frame store */
typedef struct pvo_graph pvo_graph;   /* host PatchGraph (patch_graph.hpp:66-136)   */
typedef struct pvo_dgraph pvo_dgraph; /* device-resident PatchGraph (dgraph.cu)    */

/* ---- library / context ------------------------------------------------- */
int pvo_version(void);
const char* pvo_last_error(void);
const char* pvo_status_string(int status);
int pvo_ctx_create(int device, pvo_ctx** out);
int pvo_ctx_destroy(pvo_ctx* ctx);
/* Run on an external cudaStream_t (e.g. torch's current stream); NULL = own stream. */
int pvo_ctx_set_stream(pvo_ctx* ctx, void* cuda_stream);
int pvo_ctx_synchronize(pvo_ctx* ctx);
/* Number of kernels this context has launched (profiling / gpu_launches). */
int64_t pvo_ctx_kernel_launches(pvo_ctx* ctx);
/* Tracing: when on, the BA kernel records clock64() at its phase boundaries
 * (per attempt, up to 16 attempts x 8 stamps: assemble start/end, reduce
 * start/end, solve start, update start/end, after the last barrier). */
int pvo_ctx_set_tracing(pvo_ctx* ctx, int on);
/* per-iteration timing events (pvo_ctx_last_timing), on by default; recorded as
 * external event nodes under stream capture (a replayed graph records them) */
int pvo_ctx_set_timing(pvo_ctx* ctx, int on);
int pvo_ctx_ba_phase_cycles(pvo_ctx* ctx, long long* out128);
/* Gauss-Newton attempts of the last BA run (divergence-guard retries included). */
int pvo_ctx_ba_attempts(pvo_ctx* ctx, int* attempts);
/* Device-side timing of the last pvo_window_iteration: corr ms, BA ms. */
int pvo_ctx_last_timing(pvo_ctx* ctx, double* corr_ms, double* ba_ms);

/* ---- SE(3) (se3.hpp:63-77), host utilities shared with the kernels ------ */
int pvo_se3_exp(const double* xi6, double* pose7);
int pvo_se3_log(const double* pose7, double* xi6);
int pvo_se3_compose(const double* a7, const double* b7, double* out7);
int pvo_se3_inverse(const double* a7, double* out7);
int pvo_se3_retract(const double* a7, const double* xi6, double* out7);

/* ---- camera (camera.hpp:56-72), batched on the GPU -------------------------
 * pvo_reproject_patches: n items; item i reprojects patch (x[i*pp..], y[i*pp..],
 * inv_depth[i]) from pose_i[i] into pose_j[i].  out_xy [n][pp][2], behind [n].
 * Keeps the bitwise-equal-pose shortcut of camera.cpp:52-57.
 * pvo_reprojection_jacobians: out [n][28] = center(2), d_pose_i (2x6 row-major),
 * d_pose_j (2x6), d_inverse_depth (2); behind [n].  (camera.cpp:73-108)   */
int pvo_reproject_patches(pvo_ctx* ctx, int n, int p, const double* poses_i, const double* poses_j,
                          const double* K, const double* x, const double* y, const double* inv_depth,
                          double* out_xy, uint8_t* behind);
int pvo_reprojection_jacobians(pvo_ctx* ctx, int n, int p, const double* poses_i, const double* poses_j,
                               const double* K, const double* x, const double* y, const double* inv_depth,
                               double* out, uint8_t* behind);

/* ---- correlation (correlation.hpp:33-44) ----------------------------------
 * pvo_correlate: one patch against one host pyramid (the reference signature,
 * correlation.cpp:37-71).  feats0/feats1: [p*p][C]; coords [p*p][2].  Any
 * patch width p (p = 3 runs the production Gram-form kernel, others the
 * direct FP64 form); the pyramid is cached on the device (below).
 * Throws (returns) INVALID_ARGUMENT on non-finite coordinates.            */
int pvo_correlate(pvo_ctx* ctx, int p, int channels, const float* feats0, const float* feats1,
                  const float* level0, int w0, int h0, const float* level1, int w1, int h1,
                  const double* coords, float* out);
/* correlate_at / correlate_at_cubic (correlation.hpp:37-44, correlation.cpp:8-35)
 * at n free level-space points: features [n][C] (one query descriptor per
 * point), xy [n][2], against ONE host grid [h][w][C]; cubic != 0 selects the
 * Catmull-Rom sampler (features.cpp:23-52).  out [n] FP64.                 */
int pvo_correlate_points(pvo_ctx* ctx, int n, int channels, const float* features, const float* grid, int w,
                         int h, const double* xy, int cubic, double* out);
/* The host grids passed to pvo_correlate / pvo_correlate_points stay on the
 * device, keyed by address + shape + a sampled-content fingerprint (LRU within
 * PVO_GRID_CACHE_MB, default 4096): a provider-owned pyramid is uploaded once,
 * not on every call.  Grids must not be modified in place while cached
 * (the reference never does: pyramids are built once per frame); clear the
 * cache if they are.                                                         */
int pvo_grid_cache_stats(pvo_ctx* ctx, int64_t* hits, int64_t* misses, int* entries, int64_t* bytes);
int pvo_grid_cache_clear(pvo_ctx* ctx);

/* Frame store: device-resident pyramids for n_frames slots, plus the per-cell
 * Gram terms the normalised correlation needs (computed at upload).
 * Replaces provider-owned FeaturePyramid storage (flow_provider.hpp:108).  */
int pvo_frames_reserve(pvo_ctx* ctx, int n_frames, int w0, int h0, int w1, int h1, int channels);
int pvo_frames_upload(pvo_ctx* ctx, int slot, const float* level0, const float* level1, int memspace);
/* Re-derive the Gram terms of one slot (after writing features in place). */
int pvo_frames_refresh(pvo_ctx* ctx, int slot);
/* Device pointers of the store (for zero-copy producers). */
int pvo_frames_device_ptrs(pvo_ctx* ctx, float** level0, float** level1);

/* pvo_correlate_batch: the batched form of correlate() over E edges.
 * e_patch[E] indexes patch_feats [P][2][pp][C]; e_slot[E] is the frame-store
 * slot of the target frame; coords [E][pp][2].  out [E][2][pp][7][7].
 * All arrays in `memspace`.                                                */
int pvo_correlate_batch(pvo_ctx* ctx, int n_edges, int n_patches, int p, const int* e_patch,
                        const int* e_slot, const double* coords, const float* patch_feats, float* out,
                        int memspace);

/* ---- bundle adjustment (bundle_adjust.hpp:20-111) --------------------------
 * Flattened BAProblem (bundle_adjust.hpp:30-40):
 *   poses [n_poses][7], pose_fixed [n_poses]
 *   patch_src [n_patches] (pose index), patch_x/patch_y [n_patches][pp],
 *   inv_depth [n_patches], depth_free [n_patches] or NULL (= all free)
 *   e_patch, e_pose [n_edges], e_target [n_edges][2], e_weight [n_edges][2]
 * Outputs: out_poses [n_poses][7] (fixed entries bit-identical),
 * out_depth [n_patches], residual_norms (1 + iterations entries).        */

/* gauss_newton_step (bundle_adjust.cpp:117-223).  residual_norms[2].
 * debug_h ((np+nd)^2, row-major) / debug_b (np+nd) may be NULL; when given
 * they receive the damped normal equations (NormalEquations, :65-72).    */
int pvo_gauss_newton_step(pvo_ctx* ctx, int n_poses, const double* poses, const uint8_t* pose_fixed,
                          int n_patches, int p, const int* patch_src, const double* patch_x,
                          const double* patch_y, const double* inv_depth, const uint8_t* depth_free,
                          int n_edges, const int* e_patch, const int* e_pose, const double* e_target,
                          const double* e_weight, const double* K, double damping, double* out_poses,
                          double* out_depth, double* residual_norms, double* debug_h, double* debug_b,
                          int* n_free_poses, int* n_free_depths);

/* schur_solve (bundle_adjust.cpp:62-94), dense row-major inputs:
 * hpp [np][np], hpd [np][nd], hdd [nd], bp [np], bd [nd] -> dp [np], dd [nd]. */
int pvo_schur_solve(pvo_ctx* ctx, int np, int nd, const double* hpp, const double* hpd, const double* hdd,
                    const double* bp, const double* bd, double* dp, double* dd);

/* The iteration loop of optimize_window on an already-flattened problem
 * (bundle_adjust.cpp:309-366): structure-only steps, damped GN steps with
 * the divergence guard (x1e3, x1e6, x1e9 retries), all on the device.
 * freeze_targets != 0: e_target holds the revision delta and the frozen
 * target / observability weight are derived on the device exactly as
 * bundle_adjust.cpp:288-307 does (needs image_w/h).                        */
int pvo_ba_window(pvo_ctx* ctx, int n_poses, const double* poses, const uint8_t* pose_fixed, int n_patches,
                  int p, const int* patch_src, const double* patch_x, const double* patch_y,
                  const double* inv_depth, int n_edges, const int* e_patch, const int* e_pose,
                  const double* e_target, const double* e_weight, const double* K, int image_w, int image_h,
                  int freeze_targets, double damping, int iterations, int structure_only, double* out_poses,
                  double* out_depth, double* residual_norms, int* n_norms);

/* ---- resident window: the per-frame hot path ------------------------------
 * pvo_window_load uploads one active window (the flattened optimize_window
 * problem with revision deltas, freeze_targets semantics) plus per-patch
 * features and the pose -> frame-store slot map, and keeps it on the device.
 * pvo_window_iteration runs  corr(all edges, coords = reproject at the current
 * state) + optimize_window(iterations) on it, entirely stream-ordered; no
 * host synchronisation inside.  pvo_window_read copies the state back.    */
int pvo_window_load(pvo_ctx* ctx, int n_poses, const double* poses, const uint8_t* pose_fixed,
                    const int* pose_slot, int n_patches, int p, const int* patch_src, const double* patch_x,
                    const double* patch_y, const double* inv_depth, const float* patch_feats, int n_edges,
                    const int* e_patch, const int* e_pose, const double* e_delta, const double* e_weight,
                    const double* K, int image_w, int image_h, int memspace);
/* Restore poses / depths of the loaded window (memspace as given). */
int pvo_window_set_state(pvo_ctx* ctx, const double* poses, const double* inv_depth, int memspace);
int pvo_window_iteration(pvo_ctx* ctx, int iterations, double damping, float* corr_out, int corr_memspace);
int pvo_window_correlate(pvo_ctx* ctx, float* corr_out, int memspace);
/* optimize_window's iterations only (no correlation pass): propose -> BA. */
int pvo_window_ba(pvo_ctx* ctx, int iterations, double damping);
/* residual_norms must hold iterations + 2 doubles of the last call; iteration
 * counts above PVO_MAX_WINDOW_ITERATIONS are rejected (INVALID_ARGUMENT). */
#define PVO_MAX_WINDOW_ITERATIONS 128
int pvo_window_read(pvo_ctx* ctx, double* poses, double* inv_depth, double* residual_norms, int* n_norms);
/* Device pointer of the window's correlation volume buffer [E][2][pp][49]. */
int pvo_window_corr_ptr(pvo_ctx* ctx, float** corr);

/* ---- feature extraction (features.cpp:55-235) ---------
 * pvo_frames_extract: extract_features (pool 4x4, whiten, lift 5x5 -> 25 * bc
 * unit descriptors; level 1 from the 4x4-pooled base grid) of an image
 * [ih][iw] into frame-store slot `slot` (+ Gram terms), bit-identical to the
 * reference's CPU arithmetic.  The store must be reserved with C = 25 * bc and
 * levels (iw/4, ih/4), (iw/16, ih/16).  pvo_crop_patches:
 * crop_patch_features at the 3x3 grids of n centroids -> out [n][2][9][C].  */
int pvo_frames_extract(pvo_ctx* ctx, int slot, const float* image, int image_w, int image_h, int base_channels,
                       int memspace);
int pvo_crop_patches(pvo_ctx* ctx, int slot, int n, const double* centroids, float* out, int memspace);
/* A slot's pyramid back to the host (either pointer may be NULL). */
int pvo_frames_download(pvo_ctx* ctx, int slot, float* level0, float* level1);

/* ---- correlation flow provider (flow_provider.cpp:150-312) --
 * pvo_measure_batch: CorrelationFlowProvider::measure per edge against the
 * frame store: centers [E][2] = reproject_patch(...).points[centre], behind
 * [E] (may be NULL), patch_feats [P][2][9][C] (C <= 128).  Out: delta [E][2],
 * weight [E][2] (FP64), flags [E] (1 flat, 2 out of range, 4 behind camera;
 * may be NULL).  pvo_window_propose: the same over the resident window at its
 * current state (propose, flow_provider.cpp:289-314); the revisions replace
 * the window's edge deltas / weights for the next pvo_window_iteration
 * (pipeline.cpp: propose -> set_revision -> optimize_window).  Outputs may
 * be NULL (no read-back).                                                   */
int pvo_measure_batch(pvo_ctx* ctx, int n_edges, int n_patches, int p, const int* e_patch, const int* e_slot,
                      const double* centers, const uint8_t* behind, const float* patch_feats, double* delta,
                      double* weight, uint8_t* flags);
int pvo_window_propose(pvo_ctx* ctx, double* delta, double* weight, uint8_t* flags);
/* Edges of the last measurement whose Gram-form decisions lay within the
 * rounding margin of a flip (tied argmax, hill-climb comparison, parabola
 * denominator, flatness / level-consistency threshold) and were measured again
 * with the reference's exact per-channel arithmetic (synchronises).         */
int pvo_measure_replayed(pvo_ctx* ctx, int* count);

/* ---- device-resident patch graph ---------------------
 * The PatchGraph operations of patch_graph.hpp:66-136 on device arrays
 * (frames by position, patches by id, edges in key order as a CSR by patch),
 * each a count -> scan -> scatter pass, bit-identical to pvo_graph_*.  Frames
 * carry the frame-store slot of their pyramid, patches their descriptors
 * ([n][2][9][C] or NULL).  pvo_window_load_dgraph flattens the active window
 * (bundle_adjust.cpp:231-307) on the device straight into the context's
 * resident window; pvo_dgraph_store_window writes the window's revisions
 * (e.g. from pvo_window_propose) and/or its BA state back into the graph.   */
int pvo_dgraph_create(pvo_ctx* ctx, const double* K, int image_w, int image_h, int patch_width, int channels,
                      pvo_dgraph** out);
int pvo_dgraph_destroy(pvo_dgraph* g);
// Capacity hint (no reference counterpart: the reference's std::vectors grow on
// the host): size the graph's device buffers for `patches` / `edges` / `frames`
// so a per-frame loop does not allocate inside a frame; growth past it is automatic.
int pvo_dgraph_reserve(pvo_dgraph* g, int patches, int edges, int frames);
int pvo_dgraph_add_frame(pvo_dgraph* g, double timestamp, const double* pose, int frame_slot, int* out_index);
int pvo_dgraph_add_patches(pvo_dgraph* g, int frame, int n, const double* centroids, const double* inv_depths,
                           const float* feats, int* out_ids);
int pvo_dgraph_connect(pvo_dgraph* g, int radius, int* n_added);
int pvo_dgraph_remove_frame(pvo_dgraph* g, int frame);
int pvo_dgraph_set_revisions(pvo_dgraph* g, int n, const int* patch_ids, const int* frames, const double* deltas,
                             const double* weights);
int pvo_dgraph_counts(pvo_dgraph* g, int* n_frames, int* n_patches, int* n_edges);
/* Pipeline::keyframe (pipeline.cpp:208-245) on the device graph: removes keyframe t-4 when the mean
 * reprojected displacement t-5 -> t-3 is below threshold_px; removed = frame index or -1.          */
int pvo_dgraph_keyframe(pvo_dgraph* g, double threshold_px, int* removed, double* mean_flow, int* n_used);
int pvo_dgraph_edges(pvo_dgraph* g, int* kk, int* jj, double* rev, uint8_t* has_rev);
int pvo_dgraph_frames(pvo_dgraph* g, int* indices, double* poses);
int pvo_dgraph_patches(pvo_dgraph* g, int* ids, int* src, double* inv_depth);
/* all_active: flatten every active edge (pipeline.cpp:164-181, the set propose measures) instead of the
 * revised ones only (bundle_adjust.cpp:245).                                                           */
int pvo_window_load_dgraph(pvo_ctx* ctx, pvo_dgraph* g, int window, int all_active, int* n_poses, int* n_patches,
                           int* n_edges);
int pvo_dgraph_store_window(pvo_ctx* ctx, pvo_dgraph* g, int revisions, int state);
/* The resident window's flattened problem (any pointer may be NULL). */
int pvo_window_problem_read(pvo_ctx* ctx, double* poses, uint8_t* fixed, int* pose_slot, int* patch_src, double* px,
                            double* py, double* inv_depth, int* e_patch, int* e_pose, double* e_delta,
                            double* e_weight);

/* ---- simulator oracle provider (flow_provider.cpp:34-93)
 * pvo_window_oracle_propose: revisions for every edge of the resident window
 * from the scene's ground truth (gt_poses [N][7] per window pose slot,
 * gt_inv_depth [P] per window patch), Gaussian noise and an exact outlier
 * fraction, drawn from a context-owned mt19937_64 (pvo_oracle_seed) in the
 * reference's order; they replace the window's deltas / weights.  Outputs may
 * be NULL.                                                                   */
int pvo_oracle_seed(pvo_ctx* ctx, uint64_t seed);
int pvo_window_oracle_propose(pvo_ctx* ctx, const double* gt_poses, const double* gt_inv_depth, double flow_sigma,
                              double outlier_fraction, double* delta, double* weight);

/* ---- batch of independent windows (config 5: sequences sharded per device) -
 * Windows are concatenated: pose/patch/edge offsets [n_windows + 1] (starting
 * at 0); inside a window every index is window-local (as pvo_window_load);
 * pose_slot is the frame-store slot of every pose (global).  One correlation
 * launch covers all edges, one BA launch runs a CTA per window; each window
 * keeps its own divergence guard (bundle_adjust.cpp:327-366).  Each window
 * has <= 16 free poses.  residual_norms: [n_windows][pvo_batch_norm_stride()]. */
int pvo_batch_load(pvo_ctx* ctx, int n_windows, const int* pose_off, const int* patch_off, const int* edge_off,
                   const double* poses, const uint8_t* pose_fixed, const int* pose_slot, int p,
                   const int* patch_src, const double* patch_x, const double* patch_y, const double* inv_depth,
                   const float* patch_feats, const int* e_patch, const int* e_pose, const double* e_delta,
                   const double* e_weight, const double* K, int image_w, int image_h);
int pvo_batch_reset(pvo_ctx* ctx);
int pvo_batch_iteration(pvo_ctx* ctx, int iterations, double damping, float* corr_out, int corr_memspace);
int pvo_batch_read(pvo_ctx* ctx, double* poses, double* inv_depth, double* residual_norms, int* n_norms);
int pvo_batch_norm_stride(void);

/* ---- patch graph (patch_graph.hpp:66-136), host C++ ------------------------ */
int pvo_graph_create(const double* K, int image_w, int image_h, int patch_width, pvo_graph** out);
int pvo_graph_destroy(pvo_graph* g);
int pvo_graph_add_frame(pvo_graph* g, double timestamp, const double* pose, int* out_index);
int pvo_graph_add_patches(pvo_graph* g, int frame, int n, const double* centroids, const double* inv_depths,
                          int* out_ids);
int pvo_graph_connect(pvo_graph* g, int radius, int* n_added);
int pvo_graph_remove_frame(pvo_graph* g, int frame);
int pvo_graph_set_revision(pvo_graph* g, int patch_id, int frame, const double* delta, const double* weight);
int pvo_graph_set_pose(pvo_graph* g, int frame, const double* pose);
int pvo_graph_set_inverse_depth(pvo_graph* g, int patch_id, double inv_depth);
int pvo_graph_num_frames(pvo_graph* g);
int pvo_graph_num_patches(pvo_graph* g);
int pvo_graph_num_edges(pvo_graph* g);
/* Edges in reference key order (patch id, then frame index); rev [E][4] =
 * dx dy wx wy, zeros when unset (dump_edges, patch_graph.cpp:144-151).   */
int pvo_graph_edges(pvo_graph* g, int* kk, int* jj, double* rev, uint8_t* has_rev);
int pvo_graph_frames(pvo_graph* g, int* indices, double* poses);
int pvo_graph_patches(pvo_graph* g, int* ids, int* src, double* inv_depth);
/* Pipeline::active_edges (pipeline.cpp:164-181); sizes first with NULL arrays. */
int pvo_graph_active_edges(pvo_graph* g, int window, int* kk, int* jj, int* n);
/* build_target (bundle_adjust.cpp:47-60). */
int pvo_graph_build_target(pvo_graph* g, int patch_id, int frame, double* out2);
/* The optimize_window problem build (bundle_adjust.cpp:231-307) flattened;
 * sizes first with NULL arrays.  e_target receives the frozen targets.    */
int pvo_graph_window_problem(pvo_graph* g, int window, int* n_poses, int* n_patches, int* n_edges,
                             int* pose_frames, double* poses, uint8_t* fixed, int* patch_ids, int* patch_src,
                             double* patch_x, double* patch_y, double* inv_depth, int* e_patch, int* e_pose,
                             double* e_target, double* e_weight);
/* optimize_window (bundle_adjust.cpp:225-375): flatten on the host, iterate
 * on the device, write poses / depths back into the graph.              */
int pvo_optimize_window(pvo_ctx* ctx, pvo_graph* g, int window, int iterations, int structure_only,
                        double damping, double* residual_norms, int* n_norms, int* num_edges);

#ifdef __cplusplus
}
#endif
#endif /* PVO_CAPI_H */
