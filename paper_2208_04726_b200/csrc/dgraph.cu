// dgraph.cu — device-resident patch graph maintenance and active-window
// flattening, sm_100a.
//
// Reference: PatchGraph::connect / remove_frame / set_revision
// (patch_graph.cpp:62-164), Pipeline::active_edges (pipeline.cpp:164-181) and
// the optimize_window problem build (bundle_adjust.cpp:231-307).
//
// Layout (structure of arrays, all on the device): frames in position order
// (index, pose, frame-store slot); patches in id order (id, source frame
// index, 3x3 pixel grid, inverse depth, descriptors); edges grouped by patch
// (CSR `ebeg`) and ordered by frame index inside a patch — iterating patches
// then edges IS the reference's std::map<(patch, frame)> key order.  Every
// structural update is count -> exclusive scan -> scatter with one thread per
// patch (or per frame), so the result is deterministic and bit-identical to
// the host graph (tests/test_gpu_parity.py compares them after random
// add / connect / remove / revise sequences).  The flattening writes the
// window problem straight into the BA / correlation buffers of a context, so
// a per-frame update never round-trips the graph through the host.
#include <cuda_runtime.h>

#include <cstdint>

#include "ba_common.cuh"
#include "kernels.cuh"

namespace pvo_dev {

namespace {

constexpr int kScanThreads = 1024;

// position of frame `index` in the sorted frame list, -1 if absent
__device__ __forceinline__ int frame_pos(const int* f_index, int F, int index) {
    int lo = 0, hi = F;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (f_index[mid] < index)
            lo = mid + 1;
        else
            hi = mid;
    }
    return (lo < F && f_index[lo] == index) ? lo : -1;
}

// Exclusive scan of n ints into out[0..n] (out[n] = total), one CTA.
__global__ void __launch_bounds__(kScanThreads) scan_kernel(int n, const int* __restrict__ in, int* __restrict__ out) {
    __shared__ int part[kScanThreads];
    const int t = threadIdx.x;
    const int per = (n + kScanThreads - 1) / kScanThreads;
    const int b = t * per, e = min(n, b + per);
    int s = 0;
    for (int i = b; i < e; ++i) s += in[i];
    part[t] = s;
    __syncthreads();
    for (int off = 1; off < kScanThreads; off <<= 1) {  // Hillis-Steele inclusive scan of the partials
        const int v = t >= off ? part[t - off] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    int run = t ? part[t - 1] : 0;
    for (int i = b; i < e; ++i) {
        out[i] = run;
        run += in[i];
    }
    if (t == kScanThreads - 1) out[n] = part[t];
}

// connect (patch_graph.cpp:62-85): edge iff |pos(src) - pos(j)| <= r - 1, merged
// into each patch's frame-ordered run.  Pass 0 counts, pass 1 writes.
__global__ void connect_kernel(DGraphView g, int radius, int pass, int* newlen, const int* new_ebeg, int* out_frame,
                               uint8_t* out_has, double* out_rev) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= g.P) return;
    const int s = frame_pos(g.f_index, g.F, g.p_src[k]);
    const int lo = max(0, s - (radius - 1)), hi = min(g.F - 1, s + (radius - 1));
    int i = g.ebeg[k];
    const int iend = g.ebeg[k + 1];
    int n = 0, o = pass ? new_ebeg[k] : 0;
    auto emit_old = [&](int idx) {
        if (pass) {
            out_frame[o] = g.e_frame[idx];
            out_has[o] = g.e_has[idx];
            for (int c = 0; c < 4; ++c) out_rev[4 * (size_t)o + c] = g.e_rev[4 * (size_t)idx + c];
            ++o;
        }
        ++n;
    };
    for (int pos = lo; pos <= hi; ++pos) {
        const int fi = g.f_index[pos];
        while (i < iend && g.e_frame[i] < fi) emit_old(i++);
        if (i < iend && g.e_frame[i] == fi) {
            emit_old(i++);
        } else {
            if (pass) {
                out_frame[o] = fi;
                out_has[o] = 0;
                for (int c = 0; c < 4; ++c) out_rev[4 * (size_t)o + c] = 0.0;
                ++o;
            }
            ++n;
        }
    }
    while (i < iend) emit_old(i++);
    if (!pass) newlen[k] = n;
}

// remove_frame (patch_graph.cpp:87-128): drop edges to the frame and patches
// sourced at it.  Pass 0: keep flags + surviving run lengths; pass 1: scatter.
__global__ void remove_kernel(DGraphView g, int frame, int pass, int* keep, int* newlen, const int* new_pidx,
                              const int* new_ebeg, DGraphView out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= g.P) return;
    const bool kp = g.p_src[k] != frame;
    if (!pass) {
        int n = 0;
        if (kp)
            for (int i = g.ebeg[k]; i < g.ebeg[k + 1]; ++i) n += g.e_frame[i] != frame;
        keep[k] = kp;
        newlen[k] = n;
        return;
    }
    if (!kp) return;
    const int q = new_pidx[k];
    out.p_id[q] = g.p_id[k];
    out.p_src[q] = g.p_src[k];
    for (int c = 0; c < 9; ++c) {
        out.p_x[9 * (size_t)q + c] = g.p_x[9 * (size_t)k + c];
        out.p_y[9 * (size_t)q + c] = g.p_y[9 * (size_t)k + c];
    }
    out.p_d[q] = g.p_d[k];
    for (size_t c = 0; c < g.feat_stride; ++c) out.p_feat[g.feat_stride * q + c] = g.p_feat[g.feat_stride * k + c];
    int o = new_ebeg[k];
    for (int i = g.ebeg[k]; i < g.ebeg[k + 1]; ++i) {
        if (g.e_frame[i] == frame) continue;
        out.e_frame[o] = g.e_frame[i];
        out.e_has[o] = g.e_has[i];
        for (int c = 0; c < 4; ++c) out.e_rev[4 * (size_t)o + c] = g.e_rev[4 * (size_t)i + c];
        ++o;
    }
}

// set_revision (patch_graph.cpp:153-164) for a batch of keys
__global__ void set_rev_kernel(DGraphView g, int n, const int* ids, const int* frames, const double* rev, int* missing) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    int lo = 0, hi = g.P;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (g.p_id[mid] < ids[t])
            lo = mid + 1;
        else
            hi = mid;
    }
    int hit = -1;
    if (lo < g.P && g.p_id[lo] == ids[t])
        for (int i = g.ebeg[lo]; i < g.ebeg[lo + 1]; ++i)
            if (g.e_frame[i] == frames[t]) hit = i;
    if (hit < 0) {
        atomicMin(missing, t);
        return;
    }
    g.e_has[hit] = 1;
    for (int c = 0; c < 4; ++c) g.e_rev[4 * (size_t)hit + c] = rev[4 * (size_t)t + c];
}

// ---- window flattening (bundle_adjust.cpp:231-307, pipeline.cpp:164-181) ----
// pass 0: per patch, included (source position >= window_start and at least one
// revised edge) and its revised-edge count
__global__ void win_patch_kernel(DGraphView g, int window_start, int all, int* inc, int* nrev) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= g.P) return;
    const int s = frame_pos(g.f_index, g.F, g.p_src[k]);
    int n = 0;
    if (s >= window_start)
        for (int i = g.ebeg[k]; i < g.ebeg[k + 1]; ++i) n += all || g.e_has[i];
    inc[k] = n > 0;
    nrev[k] = n;
}
// referenced frames (the pose set): plain stores of 1, order-independent
__global__ void win_used_kernel(DGraphView g, const int* inc, int all, int* used) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= g.P || !inc[k]) return;
    used[frame_pos(g.f_index, g.F, g.p_src[k])] = 1;
    for (int i = g.ebeg[k]; i < g.ebeg[k + 1]; ++i)
        if (all || g.e_has[i]) used[frame_pos(g.f_index, g.F, g.e_frame[i])] = 1;
}
__global__ void win_poses_kernel(DGraphView g, int first_free, const int* used, const int* slot_of_pos, WindowOut w) {
    const int pos = blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= g.F || !used[pos]) return;
    const int s = slot_of_pos[pos];
    w.pose_frames[s] = g.f_index[pos];
    for (int c = 0; c < 7; ++c) w.poses[7 * (size_t)s + c] = g.f_pose[7 * (size_t)pos + c];
    w.fixed[s] = pos < first_free;
    w.pose_slot[s] = g.f_slot[pos];
    // free poses are the newest positions: free slot = slot - (number of fixed slots)
    w.free_slot[s] = pos < first_free ? -1 : s - w.n_fixed_dev[0];
}
__global__ void win_nfixed_kernel(DGraphView g, int first_free, const int* used, int* n_fixed) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        int n = 0;
        for (int pos = 0; pos < min(first_free, g.F); ++pos) n += used[pos];
        *n_fixed = n;
    }
}
__global__ void win_patches_kernel(DGraphView g, const int* inc, int all, const int* pslot, const int* eoff,
                                   const int* slot_of_pos, WindowOut w) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= g.P || !inc[k]) return;
    const int q = pslot[k];
    w.patch_ids[q] = g.p_id[k];
    w.patch_src[q] = slot_of_pos[frame_pos(g.f_index, g.F, g.p_src[k])];
    for (int c = 0; c < 9; ++c) {
        w.px[9 * (size_t)q + c] = g.p_x[9 * (size_t)k + c];
        w.py[9 * (size_t)q + c] = g.p_y[9 * (size_t)k + c];
    }
    w.depth[q] = g.p_d[k];
    w.depth_slot[q] = q;  // every included patch has a free depth (bundle_adjust.cpp:123-133)
    w.edge_begin[q] = eoff[k];
    if (q == 0) w.edge_begin[w.n_patches] = eoff[g.P];
    w.graph_patch[q] = k;
    int o = eoff[k];
    for (int i = g.ebeg[k]; i < g.ebeg[k + 1]; ++i) {
        if (!all && !g.e_has[i]) continue;
        w.e_patch[o] = q;
        w.e_pose[o] = slot_of_pos[frame_pos(g.f_index, g.F, g.e_frame[i])];
        w.e_delta[2 * (size_t)o] = g.e_rev[4 * (size_t)i];
        w.e_delta[2 * (size_t)o + 1] = g.e_rev[4 * (size_t)i + 1];
        w.e_weight[2 * (size_t)o] = g.e_rev[4 * (size_t)i + 2];
        w.e_weight[2 * (size_t)o + 1] = g.e_rev[4 * (size_t)i + 3];
        w.e_graph[o] = i;
        ++o;
    }
}
// the window patches' descriptors, coalesced (one float4 per thread)
__global__ void win_feats_kernel(DGraphView g, WindowOut w) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g.feat_stride % 4 == 0) {
        const size_t n4 = g.feat_stride / 4;
        if (t >= (size_t)w.n_patches * n4) return;
        const size_t q = t / n4, c = t - q * n4;
        reinterpret_cast<float4*>(w.patch_feats)[q * n4 + c] =
            reinterpret_cast<const float4*>(g.p_feat)[(size_t)w.graph_patch[q] * n4 + c];
    } else {  // odd channel counts: one float per thread
        if (t >= (size_t)w.n_patches * g.feat_stride) return;
        const size_t q = t / g.feat_stride, c = t - q * g.feat_stride;
        w.patch_feats[q * g.feat_stride + c] = g.p_feat[(size_t)w.graph_patch[q] * g.feat_stride + c];
    }
}

// stable counting sort of the window edges by frame-store slot (the correlation
// kernel's L2-friendly order), one CTA: slot-major, edge order inside a slot
__global__ void __launch_bounds__(kScanThreads) slot_order_kernel(int E, const int* e_pose, const int* pose_slot,
                                                                   int n_slots, int* order) {
    __shared__ int base;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    __shared__ int part[kScanThreads];
    const int t = threadIdx.x;
    const int per = (E + kScanThreads - 1) / kScanThreads;
    const int b = t * per, e = min(E, b + per);
    for (int s = 0; s < n_slots; ++s) {
        int c = 0;
        for (int i = b; i < e; ++i) c += pose_slot[e_pose[i]] == s;
        part[t] = c;
        __syncthreads();
        for (int off = 1; off < kScanThreads; off <<= 1) {
            const int v = t >= off ? part[t - off] : 0;
            __syncthreads();
            part[t] += v;
            __syncthreads();
        }
        int o = base + (t ? part[t - 1] : 0);
        for (int i = b; i < e; ++i)
            if (pose_slot[e_pose[i]] == s) order[o++] = i;
        __syncthreads();
        if (t == kScanThreads - 1) base += part[t];
        __syncthreads();
    }
}

// write-back after the window's BA (bundle_adjust.cpp:368-373): free poses and
// every included patch's depth
__global__ void writeback_kernel(DGraphView g, int n_poses, const int* pose_frames, const uint8_t* fixed,
                                 const double* poses, int n_patches, const int* patch_ids, const double* depth) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_poses && !fixed[t]) {
        const int pos = frame_pos(g.f_index, g.F, pose_frames[t]);
        for (int c = 0; c < 7; ++c) g.f_pose[7 * (size_t)pos + c] = poses[7 * (size_t)t + c];
    }
    if (t < n_patches) {
        int lo = 0, hi = g.P;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (g.p_id[mid] < patch_ids[t])
                lo = mid + 1;
            else
                hi = mid;
        }
        g.p_d[lo] = depth[t];
    }
}

// revisions measured on the window (pvo_window_propose) back into the graph's edges
__global__ void store_rev_kernel(DGraphView g, int n_edges, const int* e_graph, const double* delta,
                                 const double* weight) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_edges) return;
    const int i = e_graph[e];
    g.e_has[i] = 1;
    g.e_rev[4 * (size_t)i] = delta[2 * (size_t)e];
    g.e_rev[4 * (size_t)i + 1] = delta[2 * (size_t)e + 1];
    g.e_rev[4 * (size_t)i + 2] = weight[2 * (size_t)e];
    g.e_rev[4 * (size_t)i + 3] = weight[2 * (size_t)e + 1];
}

// Pipeline::keyframe's flow test (pipeline.cpp:208-245), per patch: both edges
// (patch, frame_a) and (patch, frame_b) present and neither reprojection behind
// the camera -> |center_b - center_a|
__global__ void keyframe_flow_kernel(DGraphView g, int frame_a, int frame_b, Cam K, double* flow, int* ok) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= g.P) return;
    bool ha = false, hb = false;
    for (int i = g.ebeg[k]; i < g.ebeg[k + 1]; ++i) {
        ha = ha || g.e_frame[i] == frame_a;
        hb = hb || g.e_frame[i] == frame_b;
    }
    ok[k] = 0;
    if (!ha || !hb) return;
    const int ps = frame_pos(g.f_index, g.F, g.p_src[k]);
    const int pa = frame_pos(g.f_index, g.F, frame_a), pb = frame_pos(g.f_index, g.F, frame_b);
    const SE3 src = se3_load(g.f_pose + 7 * (size_t)ps);
    double ua, va, ub, vb;
    bool ba, bb;
    reproject_center(src, se3_load(g.f_pose + 7 * (size_t)pa), K, g.p_x + 9 * (size_t)k, g.p_y + 9 * (size_t)k, g.p_d[k],
                     &ua, &va, &ba);
    reproject_center(src, se3_load(g.f_pose + 7 * (size_t)pb), K, g.p_x + 9 * (size_t)k, g.p_y + 9 * (size_t)k, g.p_d[k],
                     &ub, &vb, &bb);
    if (ba || bb) return;
    const double dx = ub - ua, dy = vb - va;
    flow[k] = sqrt(dx * dx + dy * dy);
    ok[k] = 1;
}
// the mean in the reference's (patch id) order: one thread, sequential sum
__global__ void keyframe_mean_kernel(int P, const double* flow, const int* ok, double* out) {
    if (threadIdx.x || blockIdx.x) return;
    double sum = 0;
    int count = 0;
    for (int k = 0; k < P; ++k)
        if (ok[k]) {
            sum += flow[k];
            ++count;
        }
    out[0] = count ? sum / count : 0.0;
    out[1] = count;
}

int blocks(int n) { return n > 0 ? (n + 127) / 128 : 1; }

}  // namespace

cudaError_t dg_scan(int n, const int* in, int* out, cudaStream_t s) {
    scan_kernel<<<1, kScanThreads, 0, s>>>(n, in, out);
    return cudaGetLastError();
}
cudaError_t dg_connect(const DGraphView& g, int radius, int pass, int* newlen, const int* new_ebeg, int* out_frame,
                       uint8_t* out_has, double* out_rev, cudaStream_t s) {
    if (g.P <= 0) return cudaSuccess;
    connect_kernel<<<blocks(g.P), 128, 0, s>>>(g, radius, pass, newlen, new_ebeg, out_frame, out_has, out_rev);
    return cudaGetLastError();
}
cudaError_t dg_remove(const DGraphView& g, int frame, int pass, int* keep, int* newlen, const int* new_pidx,
                      const int* new_ebeg, const DGraphView& out, cudaStream_t s) {
    if (g.P <= 0) return cudaSuccess;
    remove_kernel<<<blocks(g.P), 128, 0, s>>>(g, frame, pass, keep, newlen, new_pidx, new_ebeg, out);
    return cudaGetLastError();
}
cudaError_t dg_set_revisions(const DGraphView& g, int n, const int* ids, const int* frames, const double* rev,
                             int* missing, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    set_rev_kernel<<<blocks(n), 128, 0, s>>>(g, n, ids, frames, rev, missing);
    return cudaGetLastError();
}
cudaError_t dg_window_pass0(const DGraphView& g, int window_start, int all, int* inc, int* nrev, cudaStream_t s) {
    if (g.P <= 0) return cudaSuccess;
    win_patch_kernel<<<blocks(g.P), 128, 0, s>>>(g, window_start, all, inc, nrev);
    return cudaGetLastError();
}
cudaError_t dg_window_used(const DGraphView& g, const int* inc, int all, int* used, cudaStream_t s) {
    if (g.P <= 0) return cudaSuccess;
    win_used_kernel<<<blocks(g.P), 128, 0, s>>>(g, inc, all, used);
    return cudaGetLastError();
}
cudaError_t dg_window_write(const DGraphView& g, int first_free, const int* inc, int all, const int* pslot,
                            const int* eoff, const int* used, const int* slot_of_pos, const WindowOut& w, int n_slots,
                            cudaStream_t s) {
    win_poses_kernel<<<blocks(g.F), 128, 0, s>>>(g, first_free, used, slot_of_pos, w);
    if (g.P > 0) win_patches_kernel<<<blocks(g.P), 128, 0, s>>>(g, inc, all, pslot, eoff, slot_of_pos, w);
    if (g.feat_stride && w.n_patches) {
        const size_t n = (size_t)w.n_patches * (g.feat_stride % 4 == 0 ? g.feat_stride / 4 : g.feat_stride);
        win_feats_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, w);
    }
    if (w.order && w.n_edges > 0) slot_order_kernel<<<1, kScanThreads, 0, s>>>(w.n_edges, w.e_pose, w.pose_slot, n_slots, w.order);
    return cudaGetLastError();
}
cudaError_t dg_window_nfixed(const DGraphView& g, int first_free, const int* used, int* n_fixed, cudaStream_t s) {
    win_nfixed_kernel<<<1, 32, 0, s>>>(g, first_free, used, n_fixed);
    return cudaGetLastError();
}
cudaError_t dg_store_revisions(const DGraphView& g, int n_edges, const int* e_graph, const double* delta,
                               const double* weight, cudaStream_t s) {
    if (n_edges <= 0) return cudaSuccess;
    store_rev_kernel<<<blocks(n_edges), 128, 0, s>>>(g, n_edges, e_graph, delta, weight);
    return cudaGetLastError();
}
cudaError_t dg_keyframe_flow(const DGraphView& g, int frame_a, int frame_b, const double* K, double* flow, int* ok,
                             double* out, cudaStream_t s) {
    if (g.P > 0) keyframe_flow_kernel<<<blocks(g.P), 128, 0, s>>>(g, frame_a, frame_b, Cam{K[0], K[1], K[2], K[3]}, flow, ok);
    keyframe_mean_kernel<<<1, 32, 0, s>>>(g.P, flow, ok, out);
    return cudaGetLastError();
}
cudaError_t dg_writeback(const DGraphView& g, int n_poses, const int* pose_frames, const uint8_t* fixed,
                         const double* poses, int n_patches, const int* patch_ids, const double* depth,
                         cudaStream_t s) {
    const int n = n_poses > n_patches ? n_poses : n_patches;
    writeback_kernel<<<blocks(n), 128, 0, s>>>(g, n_poses, pose_frames, fixed, poses, n_patches, patch_ids, depth);
    return cudaGetLastError();
}

}  // namespace pvo_dev
