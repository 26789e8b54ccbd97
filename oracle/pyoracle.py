"""ctypes binding of the CPU oracle.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu-baseline leg of bench.py, never by the product package.  Two backends
with one flat orc_* C surface: the reference's OWN sources compiled by
oracle/ref_build.py (oracle/_ref/libpvo_ref.so, preferred when present) and
the restatement oracle/pvo_oracle.cpp (always built; it covers the one entry
the reference exposes only through its simulator, orc_oracle_propose).  The
functions here mirror the product's Python API so parity tests read side by
side.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle_pvo.so"  # the restatement (oracle/pvo_oracle.cpp)
REF_LIB_PATH = HERE / "_ref" / "libpvo_ref.so"  # the reference itself (oracle/ref_build.py)

STATUS_EXC = {1: ValueError, 2: RuntimeError, 3: ArithmeticError, 4: IndexError, 5: RuntimeError}


class OracleDegenerate(RuntimeError):
    pass


STATUS_EXC[2] = OracleDegenerate


def _load(path: Path):
    if not path.exists():
        raise OSError(f"{path} missing")
    lib = C.CDLL(str(path))
    lib.orc_last_error.restype = C.c_char_p
    lib.orc_graph_create.restype = C.c_void_p
    lib.orc_graph_create.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
    for name in ["orc_graph_destroy"]:
        getattr(lib, name).argtypes = [C.c_void_p]
    return lib


try:
    lib_restated = _load(LIB_PATH)
except Exception:  # pragma: no cover - build on demand from the repo root
    import subprocess
    import sys

    subprocess.run([sys.executable, str(HERE / "build.py")], check=True)
    lib_restated = _load(LIB_PATH)


class _Dispatch:
    """Each orc_* entry from the reference build when it exports it (every
    entry but the simulator-bound orc_oracle_propose), else the restatement.
    Error messages come from whichever library ran the last call."""

    def __init__(self, ref, restated):
        self._ref, self._restated, self._last = ref, restated, restated

    def __getattr__(self, name):
        if name == "orc_last_error":
            return self._last.orc_last_error
        try:
            fn, src = getattr(self._ref, name), self._ref
        except AttributeError:
            fn, src = getattr(self._restated, name), self._restated

        def call(*args):
            self._last = src
            return fn(*args)

        call.restype = fn.restype
        return call

    def source(self, name: str) -> str:
        try:
            getattr(self._ref, name)
            return "reference"
        except AttributeError:
            return "restatement"


# PVO_ORACLE=restated|ref|auto (default auto: the reference build when present)
_MODE = os.environ.get("PVO_ORACLE", "auto")
lib_ref = None
if _MODE in ("auto", "ref") and REF_LIB_PATH.exists():
    lib_ref = _load(REF_LIB_PATH)
elif _MODE == "ref":
    raise OSError(f"PVO_ORACLE=ref but {REF_LIB_PATH} is missing (python oracle/ref_build.py)")
lib = _Dispatch(lib_ref, lib_restated) if lib_ref is not None else lib_restated
BACKEND = "reference (oracle/_ref/libpvo_ref.so)" if lib_ref is not None else "restatement (oracle/liboracle_pvo.so)"


class using:
    """with using("restated"|"reference"): run the oracle calls on one backend."""

    def __init__(self, which: str):
        if which not in ("restated", "reference"):
            raise ValueError(which)
        if which == "reference" and lib_ref is None:
            raise OSError(f"{REF_LIB_PATH} missing (python oracle/ref_build.py)")
        self.which = which

    def __enter__(self):
        global lib
        self._saved = lib
        lib = lib_restated if self.which == "restated" else _Dispatch(lib_ref, lib_restated)
        return self

    def __exit__(self, *exc):
        global lib
        lib = self._saved
        return False


def check(status: int) -> None:
    if status != 0:
        raise STATUS_EXC.get(status, RuntimeError)(lib.orc_last_error().decode())


def _f64(a, shape=None):
    out = np.ascontiguousarray(a, dtype=np.float64)
    return out.reshape(shape) if shape is not None else out


def _p(a):
    # `a.ctypes` keeps the (possibly temporary) array alive for the call
    return None if a is None else a.ctypes


D = C.c_double
I = C.c_int


# ---- se3 ----
def se3_exp(xi):
    out = np.empty(7)
    check(lib.orc_se3_exp(_p(_f64(xi, (6,))), _p(out)))
    return out


def se3_log(pose):
    out = np.empty(6)
    check(lib.orc_se3_log(_p(_f64(pose, (7,))), _p(out)))
    return out


def compose(a, b):
    out = np.empty(7)
    check(lib.orc_se3_compose(_p(_f64(a, (7,))), _p(_f64(b, (7,))), _p(out)))
    return out


def inverse(a):
    out = np.empty(7)
    check(lib.orc_se3_inverse(_p(_f64(a, (7,))), _p(out)))
    return out


def retract(a, xi):
    out = np.empty(7)
    check(lib.orc_se3_retract(_p(_f64(a, (7,))), _p(_f64(xi, (6,))), _p(out)))
    return out


def make_pose(q_xyzw, t):
    out = np.empty(7)
    check(lib.orc_se3_make_pose(_p(_f64(q_xyzw, (4,))), _p(_f64(t, (3,))), _p(out)))
    return out


def pose_distance(a, b):
    d, ang = D(), D()
    check(lib.orc_se3_pose_distance(_p(_f64(a, (7,))), _p(_f64(b, (7,))), C.byref(d), C.byref(ang)))
    return d.value, ang.value


# ---- camera ----
def patch_make(centroid, width, inverse_depth):
    n = width * width
    x, y = np.empty(n), np.empty(n)
    check(lib.orc_patch_make(D(centroid[0]), D(centroid[1]), I(width), D(inverse_depth), _p(x), _p(y)))
    return x, y


def reproject_patch(pose_i, pose_j, K, x, y, inv_depth):
    x, y = _f64(x).ravel(), _f64(y).ravel()
    p = int(round(len(x) ** 0.5))
    out = np.empty((len(x), 2))
    b = I()
    check(lib.orc_reproject_patch(_p(_f64(pose_i, (7,))), _p(_f64(pose_j, (7,))), _p(_f64(K, (4,))), I(p), _p(x),
                                  _p(y), D(inv_depth), _p(out), C.byref(b)))
    return out, bool(b.value)


def reprojection_jacobians(pose_i, pose_j, K, x, y, inv_depth):
    x, y = _f64(x).ravel(), _f64(y).ravel()
    p = int(round(len(x) ** 0.5))
    out = np.empty(28)
    b = I()
    check(lib.orc_reprojection_jacobians(_p(_f64(pose_i, (7,))), _p(_f64(pose_j, (7,))), _p(_f64(K, (4,))), I(p),
                                         _p(x), _p(y), D(inv_depth), _p(out), C.byref(b)))
    return out, bool(b.value)


# ---- correlation ----
def correlate(patch_features, pyramid, reprojection):
    g0 = np.ascontiguousarray(patch_features[0], np.float32)
    g1 = np.ascontiguousarray(patch_features[1], np.float32)
    l0 = np.ascontiguousarray(pyramid[0], np.float32)
    l1 = np.ascontiguousarray(pyramid[1], np.float32)
    coords = _f64(reprojection).reshape(-1, 2)
    pp = coords.shape[0]
    p = int(round(pp ** 0.5))
    ch = g0.reshape(pp, -1).shape[1]
    out = np.empty((2, p, p, 7, 7), np.float32)
    check(lib.orc_correlate(I(p), I(ch), _p(g0), _p(g1), _p(l0), I(l0.shape[1]), I(l0.shape[0]), _p(l1),
                            I(l1.shape[1]), I(l1.shape[0]), _p(coords), _p(out)))
    return out


def correlate_batch(e_patch, e_frame, coords, patch_feats, frames0, frames1, threads=1):
    ep = np.ascontiguousarray(e_patch, np.int32)
    ef = np.ascontiguousarray(e_frame, np.int32)
    cs = _f64(coords)
    pf = np.ascontiguousarray(patch_feats, np.float32)
    f0 = np.ascontiguousarray(frames0, np.float32)
    f1 = np.ascontiguousarray(frames1, np.float32)
    ch = pf.shape[-1]
    out = np.empty((ep.shape[0], 2, 9, 7, 7), np.float32)
    check(lib.orc_correlate_batch(I(ep.shape[0]), _p(ep), _p(ef), _p(cs), I(3), I(ch), _p(pf), _p(f0),
                                  I(f0.shape[2]), I(f0.shape[1]), _p(f1), I(f1.shape[2]), I(f1.shape[1]), _p(out),
                                  I(threads)))
    return out


def measure_batch(e_patch, e_frame, centers, behind, patch_feats, frames0, frames1, threads=1):
    """CorrelationFlowProvider::measure per edge (flow_provider.cpp:209-312):
    -> delta [E, 2], weight [E, 2], flags [E] (1 flat, 2 out of range, 4 behind)."""
    ep = np.ascontiguousarray(e_patch, np.int32)
    ef = np.ascontiguousarray(e_frame, np.int32)
    cs = _f64(centers)
    bh = None if behind is None else np.ascontiguousarray(behind, np.uint8)
    pf = np.ascontiguousarray(patch_feats, np.float32)
    f0 = np.ascontiguousarray(frames0, np.float32)
    f1 = np.ascontiguousarray(frames1, np.float32)
    E = ep.shape[0]
    d, w, fl = np.empty((E, 2)), np.empty((E, 2)), np.empty(E, np.uint8)
    check(lib.orc_measure_batch(I(E), _p(ep), _p(ef), _p(cs), _p(bh), I(3), I(pf.shape[-1]), _p(pf), _p(f0),
                                I(f0.shape[2]), I(f0.shape[1]), _p(f1), I(f1.shape[2]), I(f1.shape[1]), _p(d), _p(w),
                                _p(fl), I(threads)))
    return d, w, fl


def correlate_at(feature, grid, x, y):
    f = np.ascontiguousarray(feature, np.float32)
    g = np.ascontiguousarray(grid, np.float32)
    out = D()
    check(lib.orc_correlate_at(_p(f), I(f.shape[0]), _p(g), I(g.shape[1]), I(g.shape[0]), D(x), D(y),
                               C.byref(out)))
    return out.value


def correlate_at_cubic(feature, grid, x, y):
    f = np.ascontiguousarray(feature, np.float32)
    g = np.ascontiguousarray(grid, np.float32)
    out = D()
    check(lib.orc_correlate_at_cubic(_p(f), I(f.shape[0]), _p(g), I(g.shape[1]), I(g.shape[0]), D(x), D(y),
                                     C.byref(out)))
    return out.value


def sample_zero_padded(grid, x, y, c):
    g = np.ascontiguousarray(grid, np.float32)
    out = D()
    check(lib.orc_sample_zero_padded(_p(g), I(g.shape[1]), I(g.shape[0]), I(g.shape[2]), D(x), D(y), I(c),
                                     C.byref(out)))
    return out.value


# ---- graph ----
class PatchGraph:
    def __init__(self, K, w, h, p=3):
        self.K = _f64(K, (4,))
        self.h = lib.orc_graph_create(_p(self.K), w, h, p)
        if not self.h:
            raise ValueError(lib.orc_last_error().decode())
        self.p = p

    def __del__(self):
        if getattr(self, "h", None):
            lib.orc_graph_destroy(C.c_void_p(self.h))
            self.h = None

    @property
    def _h(self):
        return C.c_void_p(self.h)

    def add_frame(self, ts, pose):
        idx = I()
        check(lib.orc_graph_add_frame(self._h, D(ts), _p(_f64(pose, (7,))), C.byref(idx)))
        return idx.value

    def add_patches(self, frame, centroids, depths):
        c = _f64(centroids).reshape(-1, 2)
        d = _f64(depths).reshape(-1)
        ids = np.empty(len(c), np.int32)
        check(lib.orc_graph_add_patches(self._h, I(frame), I(len(c)), _p(c), _p(d), _p(ids)))
        return ids.tolist()

    def connect(self, r):
        n = I()
        check(lib.orc_graph_connect(self._h, I(r), C.byref(n)))
        return n.value

    def remove_frame(self, f):
        check(lib.orc_graph_remove_frame(self._h, I(f)))

    def set_revision(self, key, delta, weight):
        check(lib.orc_graph_set_revision(self._h, I(int(key[0])), I(int(key[1])), _p(_f64(delta, (2,))),
                                         _p(_f64(weight, (2,)))))

    def set_pose(self, f, pose):
        check(lib.orc_graph_set_pose(self._h, I(f), _p(_f64(pose, (7,)))))

    def set_inverse_depth(self, k, d):
        check(lib.orc_graph_set_inverse_depth(self._h, I(k), D(d)))

    def edges(self):
        n = lib.orc_graph_num_edges(self._h)
        kk, jj = np.empty(n, np.int32), np.empty(n, np.int32)
        rev, has = np.empty((n, 4)), np.empty(n, np.uint8)
        check(lib.orc_graph_edges(self._h, _p(kk), _p(jj), _p(rev), _p(has)))
        return kk, jj, rev, has.astype(bool)

    def frames(self):
        n = lib.orc_graph_num_frames(self._h)
        idx, poses = np.empty(n, np.int32), np.empty((n, 7))
        check(lib.orc_graph_frames(self._h, _p(idx), _p(poses)))
        return idx, poses

    def patches(self):
        n = lib.orc_graph_num_patches(self._h)
        ids, src, d = np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n)
        check(lib.orc_graph_patches(self._h, _p(ids), _p(src), _p(d)))
        return ids, src, d

    def active_edges(self, window):
        n = I()
        check(lib.orc_graph_active_edges(self._h, I(window), None, None, C.byref(n)))
        kk, jj = np.empty(n.value, np.int32), np.empty(n.value, np.int32)
        check(lib.orc_graph_active_edges(self._h, I(window), _p(kk), _p(jj), C.byref(n)))
        return kk, jj

    def build_target(self, key):
        out = np.empty(2)
        check(lib.orc_graph_build_target(self._h, I(int(key[0])), I(int(key[1])), _p(out)))
        return out

    def window_problem(self, window, damping=1e-4):
        n_p, n_k, n_e = I(), I(), I()
        nulls = [None] * 13
        check(lib.orc_window_problem(self._h, I(window), D(damping), C.byref(n_p), C.byref(n_k), C.byref(n_e),
                                     *nulls))
        if n_e.value == 0:
            return None
        N, Pn, E = n_p.value, n_k.value, n_e.value
        pp = self.p * self.p
        r = dict(pose_frames=np.empty(N, np.int32), poses=np.empty((N, 7)), fixed=np.empty(N, np.uint8),
                 patch_ids=np.empty(Pn, np.int32), patch_src=np.empty(Pn, np.int32), patch_x=np.empty((Pn, pp)),
                 patch_y=np.empty((Pn, pp)), depth=np.empty(Pn), e_patch=np.empty(E, np.int32),
                 e_pose=np.empty(E, np.int32), e_target=np.empty((E, 2)), e_weight=np.empty((E, 2)))
        order = ["pose_frames", "poses", "fixed", "patch_ids", "patch_src", "patch_x", "patch_y", "depth",
                 "e_patch", "e_pose", "e_target", "e_weight"]
        check(lib.orc_window_problem(self._h, I(window), D(damping), C.byref(n_p), C.byref(n_k), C.byref(n_e),
                                     *[_p(r[k]) for k in order]))
        return r

    def optimize_window(self, window=10, iterations=2, structure_only=0, damping=1e-4):
        norms = np.empty(iterations + 2)
        nn, ne = I(), I()
        check(lib.orc_optimize_window(self._h, I(window), I(iterations), I(structure_only), D(damping), _p(norms),
                                      C.byref(nn), C.byref(ne)))
        return list(norms[: nn.value]), ne.value


# ---- bundle adjustment on flat problems ----
def _patch_width(px):
    """p of a [P, p*p] patch-pixel array (Patch::make's row-major grid)."""
    pp = px.shape[1] if px.ndim == 2 and px.shape[0] else 9
    p = int(round(pp ** 0.5))
    if p * p != pp:
        raise ValueError("patch pixel arrays must hold p*p entries per patch")
    return p


def _prob_args(pr):
    poses = _f64(pr["poses"]).reshape(-1, 7)
    fixed = np.ascontiguousarray(pr["fixed"], np.uint8)
    src = np.ascontiguousarray(pr["patch_src"], np.int32)
    px, py, d = _f64(pr["patch_x"]), _f64(pr["patch_y"]), _f64(pr["depth"])
    ep = np.ascontiguousarray(pr["e_patch"], np.int32)
    eo = np.ascontiguousarray(pr["e_pose"], np.int32)
    et, ew = _f64(pr["e_target"]), _f64(pr["e_weight"])
    return poses, fixed, src, px, py, d, ep, eo, et, ew


def gauss_newton_step(pr, K, damping=1e-4, depth_free=None, debug=False):
    poses, fixed, src, px, py, d, ep, eo, et, ew = _prob_args(pr)
    N, Pn, E = len(poses), len(d), len(ep)
    dfree = None if depth_free is None else np.ascontiguousarray(depth_free, np.uint8)
    out_p, out_d, norms = np.empty((N, 7)), np.empty(Pn), np.empty(2)
    nfp, nfd = I(), I()
    nf = int((fixed == 0).sum())
    nd = Pn if dfree is None else int(dfree.sum())
    n = 6 * nf + nd
    dh, db = (np.empty((n, n)), np.empty(n)) if debug else (None, None)
    check(lib.orc_gauss_newton_step(I(N), _p(poses), _p(fixed), I(Pn), I(_patch_width(px)), _p(src), _p(px), _p(py), _p(d),
                                    _p(dfree), I(E), _p(ep), _p(eo), _p(et), _p(ew), _p(_f64(K, (4,))), D(damping),
                                    _p(out_p), _p(out_d), _p(norms), _p(dh), _p(db), C.byref(nfp), C.byref(nfd)))
    res = dict(poses=out_p, depth=out_d, residual_norms=list(norms))
    if debug:
        res.update(h=dh, b=db, num_free_poses=nfp.value, num_free_depths=nfd.value)
    return res


def ba_window(pr, K, damping=1e-4, iterations=2, structure_only=0):
    """optimize_window's iteration loop on a flat problem whose e_target holds frozen targets."""
    poses, fixed, src, px, py, d, ep, eo, et, ew = _prob_args(pr)
    N, Pn, E = len(poses), len(d), len(ep)
    out_p, out_d, norms = np.empty((N, 7)), np.empty(Pn), np.empty(iterations + 2)
    nn = I()
    check(lib.orc_ba_window(I(N), _p(poses), _p(fixed), I(Pn), I(_patch_width(px)), _p(src), _p(px), _p(py), _p(d), I(E), _p(ep),
                            _p(eo), _p(et), _p(ew), _p(_f64(K, (4,))), D(damping), I(iterations), I(structure_only),
                            _p(out_p), _p(out_d), _p(norms), C.byref(nn)))
    return dict(poses=out_p, depth=out_d, residual_norms=list(norms[: nn.value]))


def schur_solve(hpp, hpd, hdd, bp, bd):
    hpp = _f64(hpp)
    np_ = hpp.shape[0] if hpp.ndim == 2 else 0
    hdd = _f64(hdd).ravel()
    nd = len(hdd)
    dp, dd = np.empty(np_), np.empty(nd)
    check(lib.orc_schur_solve(I(np_), I(nd), _p(hpp.reshape(np_, np_)), _p(_f64(hpd).reshape(np_, nd)), _p(hdd),
                              _p(_f64(bp).ravel()), _p(_f64(bd).ravel()), _p(dp), _p(dd)))
    return dp, dd


def ldlt_solve(a, rhs):
    a = _f64(a)
    n = a.shape[0]
    x = np.empty(n)
    ok = I()
    check(lib.orc_ldlt_solve(I(n), _p(a), _p(_f64(rhs).ravel()), _p(x), C.byref(ok)))
    return x, bool(ok.value)


def extract_features(image, base_channels=1):
    """extract_features (features.cpp:55-235): -> (level0 [H/4, W/4, 25 bc], level1 [H/16, W/16, 25 bc])."""
    img = np.ascontiguousarray(image, np.float32)
    ih, iw = img.shape
    C = 25 * base_channels
    l0 = np.empty((ih // 4, iw // 4, C), np.float32)
    l1 = np.empty((ih // 16, iw // 16, C), np.float32)
    check(lib.orc_extract_features(_p(img), I(iw), I(ih), I(base_channels), _p(l0), _p(l1)))
    return l0, l1


def crop_patches(px, py, level0, level1):
    """crop_patch_features (features.cpp:204-224) for n patches: -> [n, 2, 9, C]."""
    x, y = _f64(px).reshape(-1, 9), _f64(py).reshape(-1, 9)
    l0, l1 = np.ascontiguousarray(level0, np.float32), np.ascontiguousarray(level1, np.float32)
    C = l0.shape[2]
    out = np.empty((x.shape[0], 2, 9, C), np.float32)
    check(lib.orc_crop_patches(I(x.shape[0]), _p(x), _p(y), _p(l0), I(l0.shape[1]), I(l0.shape[0]), _p(l1),
                               I(l1.shape[1]), I(l1.shape[0]), I(C), _p(out)))
    return out


def oracle_propose(pr, gt_poses, gt_d, K, flow_sigma=0.0, outlier_fraction=0.0, seed=0):
    """OracleFlowProvider::propose (flow_provider.cpp:34-93) on a flattened window:
    -> delta [E, 2], weight [E, 2] (one mt19937_64 seeded per call)."""
    poses, fixed, src, px, py, d, ep, eo, et, ew = _prob_args(pr)
    E = len(ep)
    dl, wt = np.empty((E, 2)), np.empty((E, 2))
    check(lib.orc_oracle_propose(I(len(poses)), _p(poses), _p(_f64(gt_poses)), I(len(d)), _p(src), _p(px), _p(py),
                                 _p(d), _p(_f64(gt_d)), I(E), _p(ep), _p(eo), _p(_f64(K, (4,))), D(flow_sigma),
                                 D(outlier_fraction), C.c_uint64(seed), _p(dl), _p(wt)))
    return dl, wt


# ---- timing helpers for bench.py's CPU legs (wall seconds measured in C++) ----
def bench_corr(pr, K, e_frame, patch_feats, frames0, frames1, threads=1):
    """reproject_patch + correlate over every edge of a flat window; -> seconds."""
    poses, fixed, src, px, py, d, ep, eo, et, ew = _prob_args(pr)
    ef = np.ascontiguousarray(e_frame, np.int32)
    pf = np.ascontiguousarray(patch_feats, np.float32)
    f0 = np.ascontiguousarray(frames0, np.float32)
    f1 = np.ascontiguousarray(frames1, np.float32)
    sec = D()
    check(lib.orc_bench_corr(I(len(poses)), _p(poses), I(len(d)), I(3), _p(src), _p(px), _p(py), _p(d), I(len(ep)),
                             _p(ep), _p(eo), _p(ef), _p(_f64(K, (4,))), I(pf.shape[-1]), _p(pf), _p(f0),
                             I(f0.shape[2]), I(f0.shape[1]), _p(f1), I(f1.shape[2]), I(f1.shape[1]), I(threads),
                             C.byref(sec)))
    return sec.value


def bench_optimize_window(graph, window=10, iterations=2, damping=1e-4):
    """optimize_window on a copy of the graph; -> seconds of the call."""
    sec = D()
    check(lib.orc_bench_optimize_window(graph._h, I(window), I(iterations), D(damping), C.byref(sec)))
    return sec.value
