"""Synthetic DPVO-shaped workloads for the five BASELINE configurations.

Inputs only — nothing here is on the measured path.  The recipe follows
SURVEY.md §8(d):
  * GT poses: frame 0 = identity, then the kSmoothRandom recurrence of
    simulator.cpp:89-103 (target flow 16 px, mid depth 8) with numpy's RNG.
  * Patches: M per frame, centroids U[3, W-4] x U[3, H-4] (pipeline.cpp:56-66),
    GT inverse depth 1/Z with Z log-uniform on [1, 15].
  * Current state: free poses <- retract(GT, twist of norm 1e-2); depths
    d_GT (1 + U(-0.1, 0.1)).
  * Revisions on the active edges (pipeline.cpp:164-181): delta = GT center -
    current center + N(0, 0.5^2), clamped to +-64, weight 0.8 = 1/(1+sigma^2);
    exactly floor(0.05 E) outliers with delta ~ U(-32, 32), weight 0.01
    (flow_provider.cpp:64-91).
  * Features: level0 [F][H/4][W/4][D] N(0,1), 3x3 binomial blur, unit norm per
    cell; level1 = 4x4 stride-4 mean of level0, re-normalised; patch features
    are Catmull-Rom crops of the source frame at coords/4 and /16
    (features.cpp:23-52, :216-235), so self-edges peak at the centre.
The graph is built through the product PatchGraph exactly like
Pipeline::admit does: add_frame, add_patches, connect(r) per frame.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TARTANAIR = dict(image=(640, 480), K=(320.0, 320.0, 320.0, 240.0))
EUROC = dict(image=(752, 480), K=(458.654, 457.296, 367.215, 248.375))

CONFIGS = {
    # name: frames, patches/frame, window W, graph radius r, camera
    "c1": dict(frames=8, patches=96, window=10, radius=13, **TARTANAIR,
               desc="synthetic 8 fr x 96 patches, 128-d @ 120x160, 2-level corr r=3, 2 BA iters"),
    "c2": dict(frames=22, patches=96, window=10, radius=13, **TARTANAIR,
               desc="DPVO default window: 96 patches/frame, 22-frame span, W=10, r=13, 480x640"),
    "c3": dict(frames=19, patches=48, window=7, radius=13, **EUROC,
               desc="DPVO fast: 48 patches/frame, W=7, r=13, 480x752 (EuRoC)"),
    "c4": dict(frames=64, patches=512, window=64, radius=7, **TARTANAIR,
               desc="stress: 512 patches/frame, 64-frame window, r=7 (404,480 edges)"),
}
CHANNELS = 128
SEED_BASE = 2208047260


# --- numpy SE(3) for input generation (Eigen formulas, se3.cpp) -------------
def _qmul(a, b):
    ax, ay, az, aw = a
    bx, by, bz, bw = b
    return np.array([aw * bx + ax * bw + ay * bz - az * by, aw * by + ay * bw + az * bx - ax * bz,
                     aw * bz + az * bw + ax * by - ay * bx, aw * bw - ax * bx - ay * by - az * bz])


def _qrot(q, v):
    vec = q[:3]
    uv = np.cross(vec, v)
    uv = uv + uv
    return v + q[3] * uv + np.cross(vec, uv)


def _norm(q):
    return q / np.sqrt((q * q).sum())


def se3_exp(xi):
    w = np.asarray(xi[3:], float)
    t2 = float(w @ w)
    th = np.sqrt(t2)
    W = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
    if th < 1e-8:
        q = np.array([0.5 * w[0], 0.5 * w[1], 0.5 * w[2], 1.0])
        V = np.eye(3) + 0.5 * W + (1 / 6) * W @ W
    else:
        s = np.sin(0.5 * th) / th
        q = np.array([s * w[0], s * w[1], s * w[2], np.cos(0.5 * th)])
        V = np.eye(3) + (1 - np.cos(th)) / t2 * W + (th - np.sin(th)) / (t2 * th) * W @ W
    return np.concatenate([_norm(q), V @ np.asarray(xi[:3], float)])


def compose(a, b):
    return np.concatenate([_norm(_qmul(a[:4], b[:4])), _qrot(a[:4], b[4:]) + a[4:]])


def inverse(a):
    qi = np.array([-a[0], -a[1], -a[2], a[3]])
    return np.concatenate([_norm(qi), -_qrot(qi, a[4:])])


def retract(a, xi):
    return compose(se3_exp(xi), a)


def _rotmat(q):
    x, y, z, w = q
    tx, ty, tz = 2 * x, 2 * y, 2 * z
    return np.array([[1 - (ty * y + tz * z), ty * x - tz * w, tz * x + ty * w],
                     [ty * x + tz * w, 1 - (tx * x + tz * z), tz * y - tx * w],
                     [tz * x - ty * w, tz * y + tx * w, 1 - (tx * x + ty * y)]])


def reproject_centers(poses, src, tgt, cx, cy, d, K):
    """Vectorised center reprojection (camera.cpp:47-71, bitwise shortcut kept)."""
    fx, fy, ccx, ccy = K
    out = np.empty((len(src), 2))
    behind = np.zeros(len(src), bool)
    rel_cache = {}
    for e in range(len(src)):
        i, j = int(src[e]), int(tgt[e])
        if np.array_equal(poses[i], poses[j]):
            out[e] = (cx[e], cy[e])
            continue
        if (i, j) not in rel_cache:
            rel = compose(poses[j], inverse(poses[i]))
            rel_cache[(i, j)] = (_rotmat(rel[:4]), rel[4:])
        R, t = rel_cache[(i, j)]
        ray = np.array([(cx[e] - ccx) / fx, (cy[e] - ccy) / fy, 1.0])
        q = R @ ray + t * d[e]
        behind[e] = q[2] <= 1e-6
        z = max(q[2], 1e-6)
        out[e] = (fx * q[0] / z + ccx, fy * q[1] / z + ccy)
    return out, behind


# --- features ------------------------------------------------------------------
def make_level0(rng, F, H, W, D):
    f = rng.standard_normal((F, H, W, D), dtype=np.float32)
    # 3x3 binomial blur, zero padded
    k = np.array([1.0, 2.0, 1.0], np.float32)
    pad = np.zeros((F, H + 2, W + 2, D), np.float32)
    pad[:, 1:-1, 1:-1] = f
    tmp = k[0] * pad[:, :, :-2] + k[1] * pad[:, :, 1:-1] + k[2] * pad[:, :, 2:]
    out = k[0] * tmp[:, :-2] + k[1] * tmp[:, 1:-1] + k[2] * tmp[:, 2:]
    out /= np.sqrt((out * out).sum(-1, keepdims=True)) + 1e-12
    return np.ascontiguousarray(out, np.float32)


def make_level1(level0):
    F, H, W, D = level0.shape
    h, w = H // 4, W // 4
    pooled = level0[:, : 4 * h, : 4 * w].reshape(F, h, 4, w, 4, D).mean(axis=(2, 4))
    pooled /= np.sqrt((pooled * pooled).sum(-1, keepdims=True)) + 1e-12
    return np.ascontiguousarray(pooled, np.float32)


def _cubic_w(t):
    return np.stack([((-0.5 * t + 1.0) * t - 0.5) * t, (1.5 * t - 2.5) * t * t + 1.0,
                     ((-1.5 * t + 2.0) * t + 0.5) * t, (0.5 * t - 0.5) * t * t], -1)


def crop_cubic(grid, xs, ys):
    """Catmull-Rom zero-padded samples (features.cpp:23-52); grid [H, W, D], xs/ys [n]."""
    H, W, D = grid.shape
    x0, y0 = np.floor(xs).astype(np.int64), np.floor(ys).astype(np.int64)
    wx, wy = _cubic_w(xs - x0), _cubic_w(ys - y0)
    out = np.zeros((len(xs), D))
    for j in range(4):
        yi = y0 - 1 + j
        oky = (yi >= 0) & (yi < H)
        row = np.zeros((len(xs), D))
        for i in range(4):
            xi = x0 - 1 + i
            ok = oky & (xi >= 0) & (xi < W)
            vals = np.zeros((len(xs), D))
            vals[ok] = grid[yi[ok], xi[ok]]
            row += wx[:, i : i + 1] * vals
        out += wy[:, j : j + 1] * row
    return out.astype(np.float32)


@dataclass
class Workload:
    name: str
    cfg: dict
    K: np.ndarray
    image: tuple
    gt_poses: np.ndarray       # [F, 7]
    poses: np.ndarray          # [F, 7] current state
    centroids: np.ndarray      # [F*M, 2]
    gt_depth: np.ndarray       # [F*M]
    depth: np.ndarray          # [F*M] current state
    patch_src: np.ndarray      # [F*M] frame index
    active_kk: np.ndarray      # active edges (reference order)
    active_jj: np.ndarray
    deltas: np.ndarray         # [E, 2]
    weights: np.ndarray        # [E, 2]
    level0: np.ndarray | None  # [F, H0, W0, D]
    level1: np.ndarray | None
    patch_feats: np.ndarray | None  # [F*M, 2, 9, D]

    @property
    def n_edges(self):
        return len(self.active_kk)


def generate(name: str = "c2", seed: int | None = None, channels: int = CHANNELS, features: bool = True,
             frames: int | None = None, patches: int | None = None) -> Workload:
    cfg = dict(CONFIGS[name])
    if frames is not None:
        cfg["frames"] = frames
    if patches is not None:
        cfg["patches"] = patches
    F, M = cfg["frames"], cfg["patches"]
    Wimg, Himg = cfg["image"]
    K = np.array(cfg["K"], float)
    rng = np.random.default_rng(SEED_BASE + (seed if seed is not None else int(name[1:])))

    # GT trajectory: kSmoothRandom (simulator.cpp:89-103)
    mid_depth = 8.0
    speed = 16.0 * mid_depth / K[0]
    vel_t = speed * np.array([1.0, 0.0, 0.0])
    vel_r = np.zeros(3)
    gt = [np.array([0, 0, 0, 1.0, 0, 0, 0])]
    for _ in range(1, F):
        g = rng.standard_normal(6)
        dt = 0.35 * speed * np.array([g[0], 0.6 * g[1], 0.4 * g[2]])
        dr = 0.25 * speed / mid_depth * g[3:]
        vel_t = 0.85 * vel_t + dt
        vel_r = 0.85 * vel_r + dr
        n = np.linalg.norm(vel_t)
        if n > 1e-12:
            vel_t = vel_t * (speed / n)
        gt.append(retract(gt[-1], np.concatenate([vel_t, vel_r])))
    gt = np.array(gt)

    # patches
    cx = rng.uniform(3.0, Wimg - 4.0, F * M)
    cy = rng.uniform(3.0, Himg - 4.0, F * M)
    z = np.exp(rng.uniform(np.log(1.0), np.log(15.0), F * M))
    gt_d = 1.0 / z
    src = np.repeat(np.arange(F), M)

    # current state
    window = cfg["window"]
    first_free = max(F - window, 1)
    poses = gt.copy()
    for f in range(first_free, F):
        tw = rng.standard_normal(6)
        tw *= 1e-2 / np.linalg.norm(tw)
        poses[f] = retract(gt[f], tw)
    depth = gt_d * (1.0 + rng.uniform(-0.1, 0.1, F * M))

    # active edges in reference order: patches with src >= oldest window frame,
    # targets within the graph radius (patch_graph.cpp:62-85, pipeline.cpp:164-181)
    r = cfg["radius"]
    oldest = max(F - window, 0)
    kk, jj = [], []
    for k in range(F * M):
        s = src[k]
        if s < oldest:
            continue
        for j in range(max(0, s - (r - 1)), min(F - 1, s + (r - 1)) + 1):
            kk.append(k)
            jj.append(j)
    kk, jj = np.array(kk, np.int32), np.array(jj, np.int32)

    # revisions
    gt_c, gt_b = reproject_centers(gt, src[kk], jj, cx[kk], cy[kk], gt_d[kk], K)
    cur_c, cur_b = reproject_centers(poses, src[kk], jj, cx[kk], cy[kk], depth[kk], K)
    sigma = 0.5
    delta = np.clip(gt_c - cur_c + rng.normal(0.0, sigma, (len(kk), 2)), -64.0, 64.0)
    weight = np.full((len(kk), 2), min(max(1.0 / (1.0 + sigma * sigma), 0.01), 0.99))
    n_out = int(np.floor(0.05 * len(kk)))
    out_idx = rng.choice(len(kk), n_out, replace=False)
    delta[out_idx] = rng.uniform(-32.0, 32.0, (n_out, 2))
    weight[out_idx] = 0.01

    lvl0 = lvl1 = pfeat = None
    if features:
        H0, W0 = Himg // 4, Wimg // 4
        lvl0 = make_level0(rng, F, H0, W0, channels)
        lvl1 = make_level1(lvl0)
        pfeat = np.empty((F * M, 2, 9, channels), np.float32)
        offs = np.array([-1.0, 0.0, 1.0])
        ox = np.tile(offs, 3)
        oy = np.repeat(offs, 3)
        for f in range(F):
            ks = np.arange(f * M, (f + 1) * M)
            px = ((cx[ks, None] + (ox + 1.0)) - 1.0).ravel()  # Patch::make: (c + col) - half
            py = ((cy[ks, None] + (oy + 1.0)) - 1.0).ravel()
            pfeat[ks, 0] = crop_cubic(lvl0[f], px / 4.0, py / 4.0).reshape(M, 9, channels)
            pfeat[ks, 1] = crop_cubic(lvl1[f], px / 16.0, py / 16.0).reshape(M, 9, channels)

    return Workload(name, cfg, K, (Wimg, Himg), gt, poses, np.stack([cx, cy], 1), gt_d, depth, src, kk, jj,
                    delta, weight, lvl0, lvl1, pfeat)


def build_graph(w: Workload, graph_cls, with_revisions: bool = True, patch_width: int = 3):
    """Build a PatchGraph (product or oracle class) the way Pipeline::admit does."""
    F, M = w.cfg["frames"], w.cfg["patches"]
    g = graph_cls(w.K, w.image[0], w.image[1], patch_width)
    for f in range(F):
        idx = g.add_frame(0.05 * f, w.poses[f])
        assert idx == f
        ks = slice(f * M, (f + 1) * M)
        g.add_patches(f, w.centroids[ks], w.depth[ks])
        g.connect(w.cfg["radius"])
    if with_revisions:
        for i in range(w.n_edges):
            g.set_revision((int(w.active_kk[i]), int(w.active_jj[i])), w.deltas[i], w.weights[i])
    return g


def window_arrays(w: Workload, prob: dict):
    """Attach revision deltas and raw weights (freeze-on-device form) to a flattened
    window problem, plus the patch features of the window's patches."""
    kk = w.active_kk
    # flattened edges are the active edges restricted to included patches, same order
    pid = prob["patch_ids"]
    sel = np.isin(kk, pid)
    out = dict(prob)
    out["e_delta"] = w.deltas[sel]
    out["e_weight"] = w.weights[sel]
    out["patch_feats"] = w.patch_feats[pid] if w.patch_feats is not None else None
    return out
