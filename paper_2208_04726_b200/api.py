"""Python mirror of the reference operator API over the C-ABI.

Names and argument meaning follow /root/reference/proj/include/pvo:
``reproject_patch`` / ``reprojection_jacobians`` (camera.hpp:56-72),
``correlate`` (correlation.hpp:33-34), ``gauss_newton_step`` /
``schur_solve`` / ``optimize_window`` / ``build_target``
(bundle_adjust.hpp:62-111) and ``PatchGraph`` (patch_graph.hpp:66-136).
Errors are raised as the exception types the reference throws
(``ValueError`` for std::invalid_argument, ``DegenerateProblem`` for
pvo::DegenerateProblem, ``ArithmeticError`` for std::domain_error,
``IndexError`` for std::out_of_range).

Every numeric result comes from the sm_100a kernels behind the C-ABI; this
module only marshals numpy arrays.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _capi
from ._capi import lib

# ---------------------------------------------------------------------------
# errors
# ---------------------------------------------------------------------------


class DegenerateProblem(RuntimeError):
    """pvo::DegenerateProblem (bundle_adjust.hpp:54-56)."""


class CudaError(RuntimeError):
    pass


class Unsupported(NotImplementedError):
    pass


_EXC = {
    _capi.PVO_INVALID_ARGUMENT: ValueError,
    _capi.PVO_DEGENERATE: DegenerateProblem,
    _capi.PVO_DOMAIN_ERROR: ArithmeticError,
    _capi.PVO_OUT_OF_RANGE: IndexError,
    _capi.PVO_CUDA_ERROR: CudaError,
    _capi.PVO_UNSUPPORTED: Unsupported,
}


def check(status: int) -> None:
    if status != _capi.PVO_OK:
        msg = lib.pvo_last_error().decode(errors="replace")
        raise _EXC.get(status, RuntimeError)(msg)


def _f64(a, shape=None) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.float64)
    return out.reshape(shape) if shape is not None else out


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _u8(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint8)


def _ptr(a: Optional[np.ndarray]):
    # `a.ctypes` (not `.data`) keeps a temporary array alive during the call
    return None if a is None else a.ctypes


# pvo_capi.h PVO_MAX_WINDOW_ITERATIONS: the window path's norms hold iterations + 2
MAX_WINDOW_ITERATIONS = 128


def _check_corr_out(corr_out, n_edges: int) -> None:
    """A host volume the C side DMAs n_edges * 2 * 9 * 49 floats into."""
    if corr_out is None:
        return
    if not isinstance(corr_out, np.ndarray) or corr_out.dtype != np.float32 or not corr_out.flags.c_contiguous \
            or not corr_out.flags.writeable:
        raise ValueError("corr_out: need a writeable C-contiguous float32 array")
    if corr_out.size < n_edges * 2 * 9 * 49:
        raise ValueError(f"corr_out: {corr_out.size} floats < {n_edges} edges x 882")


# ---------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------


class Context:
    """Device + stream + scratch arena + frame store (one per host thread)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib.pvo_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    def close(self) -> None:
        if self.handle:
            lib.pvo_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, cuda_stream: int | None) -> None:
        check(lib.pvo_ctx_set_stream(self.handle, cuda_stream or None))

    def synchronize(self) -> None:
        check(lib.pvo_ctx_synchronize(self.handle))

    @property
    def kernel_launches(self) -> int:
        return int(lib.pvo_ctx_kernel_launches(self.handle))

    @property
    def ba_attempts(self) -> int:
        n = C.c_int()
        check(lib.pvo_ctx_ba_attempts(self.handle, C.addressof(n)))
        return n.value

    @property
    def measure_replayed(self) -> int:
        """Edges of the last provider measurement re-run with the reference's exact
        arithmetic because a decision lay within the rounding margin (synchronises)."""
        n = C.c_int()
        check(lib.pvo_measure_replayed(self.handle, C.addressof(n)))
        return n.value

    def set_timing(self, on: bool = True) -> None:
        """Per-iteration timing events (last_timing); on by default."""
        check(lib.pvo_ctx_set_timing(self.handle, int(bool(on))))

    def set_tracing(self, on: bool = True) -> None:
        check(lib.pvo_ctx_set_tracing(self.handle, int(bool(on))))

    def ba_phase_cycles(self) -> np.ndarray:
        """[16 attempts][8] clock64 stamps of the last BA run (tracing on)."""
        out = np.zeros(128, np.int64)
        check(lib.pvo_ctx_ba_phase_cycles(self.handle, _ptr(out)))
        return out.reshape(16, 8)

    def last_timing(self) -> tuple[float, float]:
        a, b = C.c_double(), C.c_double()
        check(lib.pvo_ctx_last_timing(self.handle, C.addressof(a), C.addressof(b)))
        return a.value, b.value

    # ---- frame store ----
    def frames_reserve(self, n_frames: int, w0: int, h0: int, w1: int, h1: int, channels: int) -> None:
        check(lib.pvo_frames_reserve(self.handle, n_frames, w0, h0, w1, h1, channels))
        self.frame_shape = (w0, h0, w1, h1, channels)

    def frames_upload(self, slot: int, level0, level1, device: bool = False) -> None:
        """Copy a pyramid into a frame-store slot (+ its Gram terms).  device=True:
        torch tensors / device pointers, read in order on the context's stream
        (set_stream) — the producer must have finished or run on that stream."""
        if device:  # torch tensors / raw device pointers
            p0 = level0 if isinstance(level0, int) else level0.data_ptr()
            p1 = level1 if isinstance(level1, int) else level1.data_ptr()
            check(lib.pvo_frames_upload(self.handle, slot, p0, p1, _capi.PVO_DEVICE))
            return
        l0, l1 = _f32(level0), _f32(level1)
        check(lib.pvo_frames_upload(self.handle, slot, _ptr(l0), _ptr(l1), _capi.PVO_HOST))

    def frames_refresh(self, slot: int) -> None:
        check(lib.pvo_frames_refresh(self.handle, slot))

    def frames_extract(self, slot: int, image, base_channels: int = 1) -> None:
        """extract_features (features.cpp:55-235) of an image [H][W] into a store slot."""
        img = _f32(image)
        check(lib.pvo_frames_extract(self.handle, slot, _ptr(img), img.shape[1], img.shape[0], base_channels,
                                     _capi.PVO_HOST))

    def frames_download(self, slot: int):
        w0, h0, w1, h1, C = self.frame_shape
        l0, l1 = np.empty((h0, w0, C), np.float32), np.empty((h1, w1, C), np.float32)
        check(lib.pvo_frames_download(self.handle, slot, _ptr(l0), _ptr(l1)))
        return l0, l1

    def crop_patches(self, slot: int, centroids) -> np.ndarray:
        """crop_patch_features (features.cpp:204-224) at n centroids -> [n, 2, 9, C]."""
        c = _f64(centroids).reshape(-1, 2)
        out = np.empty((c.shape[0], 2, 9, self.frame_shape[4]), np.float32)
        check(lib.pvo_crop_patches(self.handle, slot, c.shape[0], _ptr(c), _ptr(out), _capi.PVO_HOST))
        return out

    def frames_device_ptrs(self) -> tuple[int, int]:
        a, b = C.c_void_p(), C.c_void_p()
        check(lib.pvo_frames_device_ptrs(self.handle, C.addressof(a), C.addressof(b)))
        return a.value, b.value


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


def _ctx(ctx: Optional[Context]) -> Context:
    return ctx if ctx is not None else default_context()


# ---------------------------------------------------------------------------
# SE(3) (se3.hpp:63-77): 7-vectors (qx qy qz qw tx ty tz), 6-vector twists
# ---------------------------------------------------------------------------


def se3_exp(xi) -> np.ndarray:
    x, out = _f64(xi, (6,)), np.empty(7)
    check(lib.pvo_se3_exp(_ptr(x), _ptr(out)))
    return out


def se3_log(pose) -> np.ndarray:
    p, out = _f64(pose, (7,)), np.empty(6)
    check(lib.pvo_se3_log(_ptr(p), _ptr(out)))
    return out


def compose(a, b) -> np.ndarray:
    x, y, out = _f64(a, (7,)), _f64(b, (7,)), np.empty(7)
    check(lib.pvo_se3_compose(_ptr(x), _ptr(y), _ptr(out)))
    return out


def inverse(a) -> np.ndarray:
    x, out = _f64(a, (7,)), np.empty(7)
    check(lib.pvo_se3_inverse(_ptr(x), _ptr(out)))
    return out


def retract(a, xi) -> np.ndarray:
    x, t, out = _f64(a, (7,)), _f64(xi, (6,)), np.empty(7)
    check(lib.pvo_se3_retract(_ptr(x), _ptr(t), _ptr(out)))
    return out


IDENTITY = np.array([0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0])

# ---------------------------------------------------------------------------
# camera (camera.hpp:10-72)
# ---------------------------------------------------------------------------


@dataclass
class Patch:
    source_frame: int
    width: int
    x: np.ndarray
    y: np.ndarray
    inverse_depth: float

    @staticmethod
    def make(source_frame: int, centroid, width: int, inverse_depth: float) -> "Patch":
        """Patch::make (camera.cpp:15-32)."""
        if width < 1:
            raise ValueError("patch: width must be >= 1")
        if inverse_depth < 0:
            raise ValueError("patch: inverse depth must be >= 0")
        half = 0.5 * (width - 1)
        col, row = np.meshgrid(np.arange(width, dtype=np.float64), np.arange(width, dtype=np.float64))
        x = (float(centroid[0]) + col.ravel()) - half
        y = (float(centroid[1]) + row.ravel()) - half
        return Patch(source_frame, width, x, y, float(inverse_depth))

    @property
    def size(self) -> int:
        return self.width * self.width

    def center(self) -> np.ndarray:
        if self.width % 2 == 1:
            m = self.size // 2
            return np.array([self.x[m], self.y[m]])
        return np.array([self.x.sum() / self.size, self.y.sum() / self.size])


def reproject_patches(poses_i, poses_j, K, x, y, inv_depth, ctx: Optional[Context] = None):
    """Batched reproject_patch (camera.cpp:47-71). Returns (points [n,pp,2], behind [n])."""
    pi, pj = _f64(poses_i).reshape(-1, 7), _f64(poses_j).reshape(-1, 7)
    n = pi.shape[0]
    xs, ys = _f64(x).reshape(n, -1), _f64(y).reshape(n, -1)
    pp = xs.shape[1]
    p = int(round(pp ** 0.5))
    d = _f64(inv_depth).reshape(n)
    out = np.empty((n, pp, 2))
    behind = np.empty(n, np.uint8)
    check(lib.pvo_reproject_patches(_ctx(ctx).handle, n, p, _ptr(pi), _ptr(pj), _ptr(_f64(K, (4,))), _ptr(xs),
                                    _ptr(ys), _ptr(d), _ptr(out), _ptr(behind)))
    return out, behind.astype(bool)


def reproject_patch(pose_i, pose_j, K, patch: Patch, ctx: Optional[Context] = None):
    pts, behind = reproject_patches(pose_i, pose_j, K, patch.x[None], patch.y[None], [patch.inverse_depth], ctx)
    return pts[0], bool(behind[0])


@dataclass
class ReprojectionJacobians:
    center: np.ndarray
    d_pose_i: np.ndarray  # 2x6
    d_pose_j: np.ndarray  # 2x6
    d_inverse_depth: np.ndarray  # 2
    behind_camera: bool


def reprojection_jacobians_batch(poses_i, poses_j, K, x, y, inv_depth, ctx: Optional[Context] = None):
    pi, pj = _f64(poses_i).reshape(-1, 7), _f64(poses_j).reshape(-1, 7)
    n = pi.shape[0]
    xs, ys = _f64(x).reshape(n, -1), _f64(y).reshape(n, -1)
    pp = xs.shape[1]
    d = _f64(inv_depth).reshape(n)
    out = np.empty((n, 28))
    behind = np.empty(n, np.uint8)
    check(lib.pvo_reprojection_jacobians(_ctx(ctx).handle, n, int(round(pp ** 0.5)), _ptr(pi), _ptr(pj),
                                         _ptr(_f64(K, (4,))), _ptr(xs), _ptr(ys), _ptr(d), _ptr(out),
                                         _ptr(behind)))
    return out, behind.astype(bool)


def reprojection_jacobians(pose_i, pose_j, K, patch: Patch, ctx: Optional[Context] = None) -> ReprojectionJacobians:
    out, behind = reprojection_jacobians_batch(pose_i, pose_j, K, patch.x[None], patch.y[None],
                                               [patch.inverse_depth], ctx)
    o = out[0]
    return ReprojectionJacobians(o[0:2].copy(), o[2:14].reshape(2, 6).copy(), o[14:26].reshape(2, 6).copy(),
                                 o[26:28].copy(), bool(behind[0]))


# ---------------------------------------------------------------------------
# correlation (correlation.hpp:11-44)
# ---------------------------------------------------------------------------

kCorrRadius = 3
kCorrSize = 7


def correlate(patch_features, pyramid, reprojection, ctx: Optional[Context] = None) -> np.ndarray:
    """correlate() (correlation.cpp:37-71).

    patch_features: (level0 [pp, C], level1 [pp, C]); pyramid: (level0 [H0, W0, C],
    level1 [H1, W1, C]); reprojection [pp, 2].  Returns [2, p, p, 7, 7] float32
    indexed [level, v, u, alpha, beta] (CorrelationGrid::at order).
    """
    g0, g1 = _f32(patch_features[0]), _f32(patch_features[1])
    l0, l1 = _f32(pyramid[0]), _f32(pyramid[1])
    coords = _f64(reprojection).reshape(-1, 2)
    pp = coords.shape[0]
    p = int(round(pp ** 0.5))
    if p * p != pp or g0.reshape(pp, -1).shape[0] != pp:
        raise ValueError("correlate: reprojection size mismatch")
    Cc = g0.reshape(pp, -1).shape[1]
    out = np.empty((2, p, p, kCorrSize, kCorrSize), np.float32)
    check(lib.pvo_correlate(_ctx(ctx).handle, p, Cc, _ptr(g0), _ptr(g1), _ptr(l0), l0.shape[1], l0.shape[0],
                            _ptr(l1), l1.shape[1], l1.shape[0], _ptr(coords), _ptr(out)))
    return out


def correlate_points(features, grid, xy, cubic: bool = False, ctx: Optional[Context] = None) -> np.ndarray:
    """correlate_at / correlate_at_cubic (correlation.cpp:8-35) at n level-space
    points: features [n, C], grid [H, W, C], xy [n, 2] -> [n] float64."""
    f = _f32(features)
    g = _f32(grid)
    q = _f64(xy).reshape(-1, 2)
    n = q.shape[0]
    if g.ndim != 3 or f.reshape(n, -1).shape[1] != g.shape[2]:
        raise ValueError("correlate_at: channel count mismatch")
    out = np.empty(n, np.float64)
    check(lib.pvo_correlate_points(_ctx(ctx).handle, n, g.shape[2], _ptr(f), _ptr(g), g.shape[1], g.shape[0], _ptr(q),
                                   1 if cubic else 0, _ptr(out)))
    return out


def correlate_at(feature, grid, x: float, y: float, ctx: Optional[Context] = None) -> float:
    """correlate_at (correlation.cpp:8-23) of one descriptor at one position."""
    return float(correlate_points(np.asarray(feature)[None], grid, [[x, y]], False, ctx)[0])


def correlate_at_cubic(feature, grid, x: float, y: float, ctx: Optional[Context] = None) -> float:
    """correlate_at_cubic (correlation.cpp:25-35) of one descriptor at one position."""
    return float(correlate_points(np.asarray(feature)[None], grid, [[x, y]], True, ctx)[0])


def grid_cache_stats(ctx: Optional[Context] = None) -> dict:
    """Device grid cache of the reference-signature correlation calls."""
    v = [C.c_int64(), C.c_int64(), C.c_int(), C.c_int64()]
    check(lib.pvo_grid_cache_stats(_ctx(ctx).handle, *[C.addressof(x) for x in v]))
    return {"hits": v[0].value, "misses": v[1].value, "entries": v[2].value, "bytes": v[3].value}


def correlate_batch(e_patch, e_slot, coords, patch_feats, ctx: Optional[Context] = None) -> np.ndarray:
    """Batched correlate over the context's frame store: out [E, 2, 9, 7, 7]."""
    c = _ctx(ctx)
    ep, es = _i32(e_patch), _i32(e_slot)
    cs = _f64(coords)
    pf = _f32(patch_feats)
    E = ep.shape[0]
    out = np.empty((E, 2, 9, kCorrSize, kCorrSize), np.float32)
    check(lib.pvo_correlate_batch(c.handle, E, pf.shape[0], 3, _ptr(ep), _ptr(es), _ptr(cs), _ptr(pf), _ptr(out),
                                  _capi.PVO_HOST))
    return out


def measure_batch(e_patch, e_slot, centers, patch_feats, behind=None, ctx: Optional[Context] = None):
    """CorrelationFlowProvider::measure per edge (flow_provider.cpp:209-312) against the
    context's frame store -> (delta [E, 2], weight [E, 2], flags [E]: 1 flat,
    2 out of range, 4 behind the camera)."""
    c = _ctx(ctx)
    ep, es = _i32(e_patch), _i32(e_slot)
    cs = _f64(centers).reshape(-1, 2)
    bh = None if behind is None else _u8(behind)
    pf = _f32(patch_feats)
    E = ep.shape[0]
    d, w, fl = np.empty((E, 2)), np.empty((E, 2)), np.empty(E, np.uint8)
    check(lib.pvo_measure_batch(c.handle, E, pf.shape[0], 3, _ptr(ep), _ptr(es), _ptr(cs),
                                None if bh is None else _ptr(bh), _ptr(pf), _ptr(d), _ptr(w), _ptr(fl)))
    return d, w, fl


# ---------------------------------------------------------------------------
# bundle adjustment (bundle_adjust.hpp:15-111)
# ---------------------------------------------------------------------------

kDefaultDamping = 1e-4
kMaxObservableMarginPx = 32.0


@dataclass
class BAProblem:
    """Flattened BAProblem (bundle_adjust.hpp:30-40)."""

    poses: np.ndarray           # [N, 7]
    pose_fixed: np.ndarray      # [N] bool
    patch_src: np.ndarray       # [P] pose index
    patch_x: np.ndarray         # [P, pp]
    patch_y: np.ndarray         # [P, pp]
    inverse_depth: np.ndarray   # [P]
    edge_patch: np.ndarray      # [E]
    edge_pose: np.ndarray       # [E]
    edge_target: np.ndarray     # [E, 2]
    edge_weight: np.ndarray     # [E, 2]
    K: np.ndarray               # [4]
    damping: float = kDefaultDamping
    depth_free: Optional[np.ndarray] = None  # [P] bool or None (all free)
    patch_width: int = 3

    def arrays(self):
        return dict(
            poses=_f64(self.poses).reshape(-1, 7), fixed=_u8(self.pose_fixed), src=_i32(self.patch_src),
            px=_f64(self.patch_x), py=_f64(self.patch_y), d=_f64(self.inverse_depth),
            dfree=None if self.depth_free is None else _u8(self.depth_free), ep=_i32(self.edge_patch),
            eo=_i32(self.edge_pose), et=_f64(self.edge_target), ew=_f64(self.edge_weight), K=_f64(self.K, (4,)))


@dataclass
class BASolution:
    poses: np.ndarray
    inverse_depths: np.ndarray
    residual_norms: list = field(default_factory=list)
    num_edges: int = 0


@dataclass
class NormalEquations:
    h: np.ndarray
    b: np.ndarray
    num_free_poses: int
    num_free_depths: int


def gauss_newton_step(problem: BAProblem, debug: bool = False, ctx: Optional[Context] = None):
    """gauss_newton_step (bundle_adjust.cpp:117-223). Returns BASolution (and NormalEquations if debug)."""
    a = problem.arrays()
    N, Pn, E = a["poses"].shape[0], a["d"].shape[0], a["ep"].shape[0]
    out_p, out_d, norms = np.empty((N, 7)), np.empty(Pn), np.empty(2)
    nfp, nfd = C.c_int(), C.c_int()
    dh = db = None
    if debug:
        nf = int((~np.asarray(problem.pose_fixed, bool)).sum())
        nd = Pn if problem.depth_free is None else int(np.asarray(problem.depth_free, bool).sum())
        n = 6 * nf + nd
        dh, db = np.empty((n, n)), np.empty(n)
    check(lib.pvo_gauss_newton_step(
        _ctx(ctx).handle, N, _ptr(a["poses"]), _ptr(a["fixed"]), Pn, problem.patch_width, _ptr(a["src"]),
        _ptr(a["px"]), _ptr(a["py"]), _ptr(a["d"]), _ptr(a["dfree"]), E, _ptr(a["ep"]), _ptr(a["eo"]),
        _ptr(a["et"]), _ptr(a["ew"]), _ptr(a["K"]), float(problem.damping), _ptr(out_p), _ptr(out_d),
        _ptr(norms), _ptr(dh), _ptr(db), C.addressof(nfp), C.addressof(nfd)))
    sol = BASolution(out_p, out_d, list(norms), E)
    if debug:
        return sol, NormalEquations(dh, db, nfp.value, nfd.value)
    return sol


def schur_solve(h_pp, h_pd, h_dd, b_p, b_d, ctx: Optional[Context] = None):
    """schur_solve (bundle_adjust.cpp:62-94). Returns (pose_delta, depth_delta)."""
    hpp = _f64(h_pp)
    np_ = hpp.shape[0] if hpp.ndim == 2 else 0
    hdd = _f64(h_dd).reshape(-1)
    nd = hdd.shape[0]
    hpd = _f64(h_pd).reshape(np_, nd)
    bp, bd = _f64(b_p).reshape(np_), _f64(b_d).reshape(nd)
    dp, dd = np.empty(np_), np.empty(nd)
    check(lib.pvo_schur_solve(_ctx(ctx).handle, np_, nd, _ptr(hpp.reshape(np_, np_)), _ptr(hpd), _ptr(hdd),
                              _ptr(bp), _ptr(bd), _ptr(dp), _ptr(dd)))
    return dp, dd


def ba_window(problem: BAProblem, iterations: int = 2, structure_only_iterations: int = 0,
              freeze_targets: bool = False, image_size=(0, 0), ctx: Optional[Context] = None) -> BASolution:
    """The iteration loop of optimize_window (bundle_adjust.cpp:309-366) on a flattened problem."""
    a = problem.arrays()
    N, Pn, E = a["poses"].shape[0], a["d"].shape[0], a["ep"].shape[0]
    out_p, out_d = np.empty((N, 7)), np.empty(Pn)
    norms = np.empty(iterations + 2)
    nn = C.c_int()
    check(lib.pvo_ba_window(
        _ctx(ctx).handle, N, _ptr(a["poses"]), _ptr(a["fixed"]), Pn, problem.patch_width, _ptr(a["src"]),
        _ptr(a["px"]), _ptr(a["py"]), _ptr(a["d"]), E, _ptr(a["ep"]), _ptr(a["eo"]), _ptr(a["et"]),
        _ptr(a["ew"]), _ptr(a["K"]), int(image_size[0]), int(image_size[1]), int(bool(freeze_targets)),
        float(problem.damping), iterations, structure_only_iterations, _ptr(out_p), _ptr(out_d), _ptr(norms),
        C.addressof(nn)))
    return BASolution(out_p, out_d, list(norms[: nn.value]), E)


# ---------------------------------------------------------------------------
# patch graph (patch_graph.hpp:66-136) and optimize_window
# ---------------------------------------------------------------------------


@dataclass
class WindowOptions:
    window: int = 10
    iterations: int = 2
    structure_only_iterations: int = 0
    damping: float = kDefaultDamping


class PatchGraph:
    def __init__(self, K, image_width: int, image_height: int, patch_width: int = 3):
        h = C.c_void_p()
        self.K = _f64(K, (4,))
        check(lib.pvo_graph_create(_ptr(self.K), image_width, image_height, patch_width, C.byref(h)))
        self.handle = h
        self.image_width, self.image_height, self.patch_width = image_width, image_height, patch_width

    def __del__(self):  # pragma: no cover
        if getattr(self, "handle", None):
            lib.pvo_graph_destroy(self.handle)
            self.handle = None

    def add_frame(self, timestamp: float, pose) -> int:
        idx = C.c_int()
        check(lib.pvo_graph_add_frame(self.handle, float(timestamp), _ptr(_f64(pose, (7,))), C.addressof(idx)))
        return idx.value

    def add_patches(self, frame: int, centroids, inverse_depths) -> list:
        c = _f64(centroids).reshape(-1, 2)
        d = _f64(inverse_depths).reshape(-1)
        if c.shape[0] != d.shape[0]:
            raise ValueError("patch graph: centroid/depth count mismatch")
        ids = np.empty(c.shape[0], np.int32)
        check(lib.pvo_graph_add_patches(self.handle, frame, c.shape[0], _ptr(c), _ptr(d), _ptr(ids)))
        return ids.tolist()

    def connect(self, radius: int) -> int:
        n = C.c_int()
        check(lib.pvo_graph_connect(self.handle, radius, C.addressof(n)))
        return n.value

    def remove_frame(self, frame: int) -> None:
        check(lib.pvo_graph_remove_frame(self.handle, frame))

    def set_revision(self, key, delta, weight) -> None:
        check(lib.pvo_graph_set_revision(self.handle, int(key[0]), int(key[1]), _ptr(_f64(delta, (2,))),
                                         _ptr(_f64(weight, (2,)))))

    def set_revisions(self, kk, jj, deltas, weights) -> None:
        d, w = _f64(deltas).reshape(-1, 2), _f64(weights).reshape(-1, 2)
        for i, (k, j) in enumerate(zip(kk, jj)):
            check(lib.pvo_graph_set_revision(self.handle, int(k), int(j), d[i].ctypes.data, w[i].ctypes.data))

    def set_pose(self, frame: int, pose) -> None:
        check(lib.pvo_graph_set_pose(self.handle, frame, _ptr(_f64(pose, (7,)))))

    def set_inverse_depth(self, patch_id: int, d: float) -> None:
        check(lib.pvo_graph_set_inverse_depth(self.handle, patch_id, float(d)))

    @property
    def num_edges(self) -> int:
        return lib.pvo_graph_num_edges(self.handle)

    def edges(self):
        """(kk, jj, rev [E,4], has_rev) in the reference key order."""
        n = self.num_edges
        kk, jj = np.empty(n, np.int32), np.empty(n, np.int32)
        rev, has = np.empty((n, 4)), np.empty(n, np.uint8)
        check(lib.pvo_graph_edges(self.handle, _ptr(kk), _ptr(jj), _ptr(rev), _ptr(has)))
        return kk, jj, rev, has.astype(bool)

    def frames(self):
        n = lib.pvo_graph_num_frames(self.handle)
        idx, poses = np.empty(n, np.int32), np.empty((n, 7))
        check(lib.pvo_graph_frames(self.handle, _ptr(idx), _ptr(poses)))
        return idx, poses

    def patches(self):
        n = lib.pvo_graph_num_patches(self.handle)
        ids, src, d = np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n)
        check(lib.pvo_graph_patches(self.handle, _ptr(ids), _ptr(src), _ptr(d)))
        return ids, src, d

    def active_edges(self, window: int):
        n = C.c_int()
        check(lib.pvo_graph_active_edges(self.handle, window, None, None, C.addressof(n)))
        kk, jj = np.empty(n.value, np.int32), np.empty(n.value, np.int32)
        check(lib.pvo_graph_active_edges(self.handle, window, _ptr(kk), _ptr(jj), C.addressof(n)))
        return kk, jj

    def build_target(self, key) -> np.ndarray:
        out = np.empty(2)
        check(lib.pvo_graph_build_target(self.handle, int(key[0]), int(key[1]), _ptr(out)))
        return out

    def window_problem(self, window: int) -> Optional[dict]:
        """The flattened optimize_window problem (bundle_adjust.cpp:231-307)."""
        n_p, n_k, n_e = C.c_int(), C.c_int(), C.c_int()
        nulls = [None] * 13
        check(lib.pvo_graph_window_problem(self.handle, window, C.addressof(n_p), C.addressof(n_k),
                                           C.addressof(n_e), *nulls))
        if n_e.value == 0:
            return None
        N, Pn, E = n_p.value, n_k.value, n_e.value
        pp = self.patch_width ** 2
        r = dict(pose_frames=np.empty(N, np.int32), poses=np.empty((N, 7)), fixed=np.empty(N, np.uint8),
                 patch_ids=np.empty(Pn, np.int32), patch_src=np.empty(Pn, np.int32), patch_x=np.empty((Pn, pp)),
                 patch_y=np.empty((Pn, pp)), depth=np.empty(Pn), e_patch=np.empty(E, np.int32),
                 e_pose=np.empty(E, np.int32), e_target=np.empty((E, 2)), e_weight=np.empty((E, 2)))
        order = ["pose_frames", "poses", "fixed", "patch_ids", "patch_src", "patch_x", "patch_y", "depth",
                 "e_patch", "e_pose", "e_target", "e_weight"]
        check(lib.pvo_graph_window_problem(self.handle, window, C.addressof(n_p), C.addressof(n_k),
                                           C.addressof(n_e), *[_ptr(r[k]) for k in order]))
        return r


def build_target(graph: PatchGraph, key) -> np.ndarray:
    return graph.build_target(key)


def optimize_window(graph: PatchGraph, options: WindowOptions = WindowOptions(),
                    ctx: Optional[Context] = None) -> BASolution:
    """optimize_window (bundle_adjust.cpp:225-375); mutates the graph."""
    norms = np.empty(options.iterations + 2)
    nn, ne = C.c_int(), C.c_int()
    check(lib.pvo_optimize_window(_ctx(ctx).handle, graph.handle, options.window, options.iterations,
                                  options.structure_only_iterations, float(options.damping), _ptr(norms),
                                  C.addressof(nn), C.addressof(ne)))
    idx, poses = graph.frames()
    ids, src, d = graph.patches()
    return BASolution(poses, d, list(norms[: nn.value]), ne.value)


# ---------------------------------------------------------------------------
# resident window (the per-frame hot path)
# ---------------------------------------------------------------------------


class Window:
    """A device-resident active window: corr + BA iterations without host round trips."""

    def __init__(self, ctx: Context):
        self.ctx = ctx

    def load(self, prob: dict, pose_slot, patch_feats, K, image_size) -> None:
        """prob: flattened window with revision *deltas* in e_delta (freeze_targets semantics)."""
        self.n_poses = int(prob["poses"].shape[0])
        self.n_patches = int(prob["depth"].shape[0])
        self.n_edges = int(prob["e_patch"].shape[0])
        keep = dict(poses=_f64(prob["poses"]), fixed=_u8(prob["fixed"]), slot=_i32(pose_slot),
                    src=_i32(prob["patch_src"]), px=_f64(prob["patch_x"]), py=_f64(prob["patch_y"]),
                    d=_f64(prob["depth"]), pf=_f32(patch_feats), ep=_i32(prob["e_patch"]),
                    eo=_i32(prob["e_pose"]), ed=_f64(prob["e_delta"]), ew=_f64(prob["e_weight"]),
                    K=_f64(K, (4,)))
        check(lib.pvo_window_load(self.ctx.handle, self.n_poses, _ptr(keep["poses"]), _ptr(keep["fixed"]),
                                  _ptr(keep["slot"]), self.n_patches, 3, _ptr(keep["src"]), _ptr(keep["px"]),
                                  _ptr(keep["py"]), _ptr(keep["d"]), _ptr(keep["pf"]), self.n_edges,
                                  _ptr(keep["ep"]), _ptr(keep["eo"]), _ptr(keep["ed"]), _ptr(keep["ew"]),
                                  _ptr(keep["K"]), int(image_size[0]), int(image_size[1]), _capi.PVO_HOST))

    def reset(self) -> None:
        check(lib.pvo_window_set_state(self.ctx.handle, None, None, _capi.PVO_HOST))

    def set_state(self, poses, depth) -> None:
        p, d = _f64(poses), _f64(depth)
        check(lib.pvo_window_set_state(self.ctx.handle, _ptr(p), _ptr(d), _capi.PVO_HOST))

    def iteration(self, iterations: int = 2, damping: float = kDefaultDamping, corr_out=None,
                  corr_device_ptr: int | None = None) -> None:
        _check_corr_out(corr_out, self.n_edges)
        if corr_device_ptr is not None:
            check(lib.pvo_window_iteration(self.ctx.handle, iterations, damping, corr_device_ptr, _capi.PVO_DEVICE))
        elif corr_out is not None:
            check(lib.pvo_window_iteration(self.ctx.handle, iterations, damping, _ptr(corr_out), _capi.PVO_HOST))
        else:
            check(lib.pvo_window_iteration(self.ctx.handle, iterations, damping, None, _capi.PVO_DEVICE))

    def ba(self, iterations: int = 2, damping: float = kDefaultDamping) -> None:
        """optimize_window's iterations only (no correlation pass)."""
        check(lib.pvo_window_ba(self.ctx.handle, iterations, damping))

    def correlate(self) -> np.ndarray:
        out = np.empty((self.n_edges, 2, 9, 7, 7), np.float32)
        check(lib.pvo_window_correlate(self.ctx.handle, _ptr(out), _capi.PVO_HOST))
        return out

    def read(self):
        poses, d = np.empty((self.n_poses, 7)), np.empty(self.n_patches)
        norms = np.empty(MAX_WINDOW_ITERATIONS + 2)
        nn = C.c_int()
        check(lib.pvo_window_read(self.ctx.handle, _ptr(poses), _ptr(d), _ptr(norms), C.addressof(nn)))
        return poses, d, list(norms[: nn.value])

    def propose(self, read_back: bool = True):
        """CorrelationFlowProvider::propose at the current state; the revisions become
        the window's edge deltas / weights for the next iteration."""
        if not read_back:
            check(lib.pvo_window_propose(self.ctx.handle, None, None, None))
            return None
        d, w, fl = np.empty((self.n_edges, 2)), np.empty((self.n_edges, 2)), np.empty(self.n_edges, np.uint8)
        check(lib.pvo_window_propose(self.ctx.handle, _ptr(d), _ptr(w), _ptr(fl)))
        return d, w, fl

    def oracle_propose(self, gt_poses, gt_inv_depth, flow_sigma: float = 0.0, outlier_fraction: float = 0.0,
                       seed=None):
        """OracleFlowProvider::propose (flow_provider.cpp:34-93) over the window's edges;
        the revisions become the window's deltas / weights.  seed re-seeds the
        context's provider RNG first (else the stream continues)."""
        if seed is not None:
            check(lib.pvo_oracle_seed(self.ctx.handle, int(seed)))
        d, w = np.empty((self.n_edges, 2)), np.empty((self.n_edges, 2))
        check(lib.pvo_window_oracle_propose(self.ctx.handle, _ptr(_f64(gt_poses).reshape(-1, 7)),
                                            _ptr(_f64(gt_inv_depth)), float(flow_sigma), float(outlier_fraction),
                                            _ptr(d), _ptr(w)))
        return d, w

    def corr_device_ptr(self) -> int:
        p = C.c_void_p()
        check(lib.pvo_window_corr_ptr(self.ctx.handle, C.addressof(p)))
        return p.value


class Batch:
    """Many independent windows on one device (config 5): one correlation launch
    over every edge, one BA launch with a CTA per window (pvo_batch_*)."""

    def __init__(self, ctx: Context):
        self.ctx = ctx

    def load(self, probs: list, pose_slots: list, patch_feats: list, K, image_size) -> None:
        """probs: flattened windows (window-local indices, revision deltas in e_delta);
        pose_slots: frame-store slot of every pose of each window."""
        self.n_windows = len(probs)
        self.pose_off = np.concatenate([[0], np.cumsum([len(p["poses"]) for p in probs])]).astype(np.int32)
        self.patch_off = np.concatenate([[0], np.cumsum([len(p["depth"]) for p in probs])]).astype(np.int32)
        self.edge_off = np.concatenate([[0], np.cumsum([len(p["e_patch"]) for p in probs])]).astype(np.int32)
        cat = lambda key, conv: conv(np.concatenate([p[key] for p in probs]))  # noqa: E731
        keep = dict(poses=cat("poses", _f64), fixed=cat("fixed", _u8), slot=_i32(np.concatenate(pose_slots)),
                    src=cat("patch_src", _i32), px=cat("patch_x", _f64), py=cat("patch_y", _f64),
                    d=cat("depth", _f64), pf=_f32(np.concatenate(patch_feats)), ep=cat("e_patch", _i32),
                    eo=cat("e_pose", _i32), ed=cat("e_delta", _f64), ew=cat("e_weight", _f64), K=_f64(K, (4,)),
                    po=self.pose_off, ko=self.patch_off, eo_=self.edge_off)
        self.n_poses, self.n_patches, self.n_edges = int(self.pose_off[-1]), int(self.patch_off[-1]), int(self.edge_off[-1])
        check(lib.pvo_batch_load(self.ctx.handle, self.n_windows, _ptr(keep["po"]), _ptr(keep["ko"]),
                                 _ptr(keep["eo_"]), _ptr(keep["poses"]), _ptr(keep["fixed"]), _ptr(keep["slot"]), 3,
                                 _ptr(keep["src"]), _ptr(keep["px"]), _ptr(keep["py"]), _ptr(keep["d"]),
                                 _ptr(keep["pf"]), _ptr(keep["ep"]), _ptr(keep["eo"]), _ptr(keep["ed"]),
                                 _ptr(keep["ew"]), _ptr(keep["K"]), int(image_size[0]), int(image_size[1])))

    def reset(self) -> None:
        check(lib.pvo_batch_reset(self.ctx.handle))

    def iteration(self, iterations: int = 2, damping: float = kDefaultDamping, corr_out=None,
                  corr_device_ptr: int | None = None) -> None:
        """corr_out: host volume [E, 2, 9, 7, 7]; corr_device_ptr: a device buffer of
        the same size (e.g. a torch tensor's data_ptr()) that receives the volume."""
        _check_corr_out(corr_out, self.n_edges)
        if corr_device_ptr is not None:
            check(lib.pvo_batch_iteration(self.ctx.handle, iterations, damping, corr_device_ptr, _capi.PVO_DEVICE))
        elif corr_out is not None:
            check(lib.pvo_batch_iteration(self.ctx.handle, iterations, damping, _ptr(corr_out), _capi.PVO_HOST))
        else:
            check(lib.pvo_batch_iteration(self.ctx.handle, iterations, damping, None, _capi.PVO_DEVICE))

    def read(self):
        """-> per-window lists of (poses [N_w, 7], depths [P_w], residual_norms)."""
        stride = lib.pvo_batch_norm_stride()
        poses, d = np.empty((self.n_poses, 7)), np.empty(self.n_patches)
        norms = np.empty((self.n_windows, stride))
        nn = np.empty(self.n_windows, np.int32)
        check(lib.pvo_batch_read(self.ctx.handle, _ptr(poses), _ptr(d), _ptr(norms), _ptr(nn)))
        out = []
        for w in range(self.n_windows):
            out.append((poses[self.pose_off[w]:self.pose_off[w + 1]], d[self.patch_off[w]:self.patch_off[w + 1]],
                        list(norms[w, : nn[w]])))
        return out


class DeviceGraph:
    """PatchGraph kept on the device (pvo_dgraph_*; patch_graph.hpp:66-136): the same
    operations and edge order as PatchGraph, plus an on-device window flatten into a
    context's resident Window."""

    def __init__(self, ctx: Context, K, image_width: int, image_height: int, channels: int = 0, patch_width: int = 3):
        h = C.c_void_p()
        self.ctx = ctx
        self.K = _f64(K, (4,))
        self.channels = channels
        check(lib.pvo_dgraph_create(ctx.handle, _ptr(self.K), image_width, image_height, patch_width, channels,
                                    C.byref(h)))
        self.handle = h

    def __del__(self):  # pragma: no cover
        if getattr(self, "handle", None):
            lib.pvo_dgraph_destroy(self.handle)
            self.handle = None

    def reserve(self, patches: int, edges: int, frames: int) -> None:
        """Capacity hint: size the device buffers up front so a per-frame loop does
        not allocate inside a frame (growth past the hint stays automatic)."""
        check(lib.pvo_dgraph_reserve(self.handle, int(patches), int(edges), int(frames)))

    def add_frame(self, timestamp: float, pose, frame_slot: int = 0) -> int:
        idx = C.c_int()
        check(lib.pvo_dgraph_add_frame(self.handle, float(timestamp), _ptr(_f64(pose, (7,))), int(frame_slot),
                                       C.addressof(idx)))
        return idx.value

    def add_patches(self, frame: int, centroids, inverse_depths, feats=None) -> list:
        c = _f64(centroids).reshape(-1, 2)
        d = _f64(inverse_depths).reshape(-1)
        f = None if feats is None else _f32(feats)
        ids = np.empty(c.shape[0], np.int32)
        check(lib.pvo_dgraph_add_patches(self.handle, frame, c.shape[0], _ptr(c), _ptr(d),
                                         None if f is None else _ptr(f), _ptr(ids)))
        return ids.tolist()

    def connect(self, radius: int) -> int:
        n = C.c_int()
        check(lib.pvo_dgraph_connect(self.handle, radius, C.addressof(n)))
        return n.value

    def remove_frame(self, frame: int) -> None:
        check(lib.pvo_dgraph_remove_frame(self.handle, frame))

    def set_revisions(self, kk, jj, deltas, weights) -> None:
        k, j = _i32(kk), _i32(jj)
        check(lib.pvo_dgraph_set_revisions(self.handle, k.shape[0], _ptr(k), _ptr(j), _ptr(_f64(deltas).reshape(-1, 2)),
                                           _ptr(_f64(weights).reshape(-1, 2))))

    def keyframe(self, threshold_px: float):
        """Pipeline::keyframe (pipeline.cpp:208-245) -> (removed frame or -1, mean flow, patches used)."""
        r, m, n = C.c_int(), C.c_double(), C.c_int()
        check(lib.pvo_dgraph_keyframe(self.handle, float(threshold_px), C.addressof(r), C.addressof(m), C.addressof(n)))
        return r.value, m.value, n.value

    def counts(self):
        a, b, c = C.c_int(), C.c_int(), C.c_int()
        check(lib.pvo_dgraph_counts(self.handle, C.addressof(a), C.addressof(b), C.addressof(c)))
        return a.value, b.value, c.value

    def edges(self):
        _, _, E = self.counts()
        kk, jj = np.empty(E, np.int32), np.empty(E, np.int32)
        rev, has = np.empty((E, 4)), np.empty(E, np.uint8)
        check(lib.pvo_dgraph_edges(self.handle, _ptr(kk), _ptr(jj), _ptr(rev), _ptr(has)))
        rev[has == 0] = 0.0
        return kk, jj, rev, has.astype(bool)

    def frames(self):
        F, _, _ = self.counts()
        idx, poses = np.empty(F, np.int32), np.empty((F, 7))
        check(lib.pvo_dgraph_frames(self.handle, _ptr(idx), _ptr(poses)))
        return idx, poses

    def patches(self):
        _, P, _ = self.counts()
        ids, src, d = np.empty(P, np.int32), np.empty(P, np.int32), np.empty(P)
        check(lib.pvo_dgraph_patches(self.handle, _ptr(ids), _ptr(src), _ptr(d)))
        return ids, src, d

    def load_window(self, window: int, all_active: bool = False) -> tuple:
        """Flatten the active window on the device into the context's resident Window
        (revised edges, as optimize_window; all_active: every active edge, the set
        propose() measures); returns (n_poses, n_patches, n_edges)."""
        a, b, c = C.c_int(), C.c_int(), C.c_int()
        check(lib.pvo_window_load_dgraph(self.ctx.handle, self.handle, window, int(all_active), C.addressof(a),
                                         C.addressof(b), C.addressof(c)))
        win = Window(self.ctx)
        win.n_poses, win.n_patches, win.n_edges = a.value, b.value, c.value
        self.window = win
        return a.value, b.value, c.value

    def store_window(self, revisions: bool = True, state: bool = True) -> None:
        check(lib.pvo_dgraph_store_window(self.ctx.handle, self.handle, int(revisions), int(state)))


def window_problem_read(ctx: Context, n_poses: int, n_patches: int, n_edges: int) -> dict:
    """The resident window's flattened problem (pvo_window_problem_read)."""
    out = dict(poses=np.empty((n_poses, 7)), fixed=np.empty(n_poses, np.uint8), pose_slot=np.empty(n_poses, np.int32),
               patch_src=np.empty(n_patches, np.int32), patch_x=np.empty((n_patches, 9)),
               patch_y=np.empty((n_patches, 9)), depth=np.empty(n_patches), e_patch=np.empty(n_edges, np.int32),
               e_pose=np.empty(n_edges, np.int32), e_delta=np.empty((n_edges, 2)), e_weight=np.empty((n_edges, 2)))
    k = ["poses", "fixed", "pose_slot", "patch_src", "patch_x", "patch_y", "depth", "e_patch", "e_pose", "e_delta",
         "e_weight"]
    check(lib.pvo_window_problem_read(ctx.handle, *[_ptr(out[n]) for n in k]))
    return out
