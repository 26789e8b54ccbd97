"""Generality against the reference, and the limits that remain.

The reference's BA takes patches of any width (Patch::make, camera.cpp:15-32)
and graphs of any radius (patch_graph.cpp:62-85).  Odd widths run on the 3x3
kernels through a corners + centre stand-in (capi_core.cu as_3x3: the BA reads a
patch only through its centre pixel and the behind-camera test, whose affine
q_z is minimal at a grid corner) and are checked against the reference here.
What the sm_100a kernels still refuse must raise Unsupported (never a wrong
answer): even widths, more than 32 edges on one patch (lane per edge), a
large-window patch run touching more than 25 free poses, the normal-equation
capture beyond 16 free poses, window / batch correlation of non-3x3 patches,
more than 128 channels in the provider measurement."""
import numpy as np
import pytest

import oracle.pyoracle as orc
import paper_2208_04726_b200 as pvo
import pvo_synth as synth
from tests.test_gpu_parity import pose_parity

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("width", [1, 5, 7])
def test_optimize_window_any_odd_patch_width(ctx, width):
    """optimize_window on graphs of p x p patches equals the reference's
    (poses / depths 1e-3, residual norms 1e-6)."""
    w = synth.generate("c1", features=False)
    g = synth.build_graph(w, pvo.PatchGraph, patch_width=width)
    o = synth.build_graph(w, orc.PatchGraph, patch_width=width)
    sol = pvo.optimize_window(g, pvo.WindowOptions(window=w.cfg["window"]), ctx=ctx)
    norms, ne = o.optimize_window(window=w.cfg["window"])
    assert sol.num_edges == ne == w.n_edges
    assert np.allclose(sol.residual_norms, norms, rtol=1e-6)
    _, pg = g.frames()
    _, po = o.frames()
    dt, dq = pose_parity(pg, po)
    assert dt.max() <= 1e-3 and dq.max() <= 1e-3
    _, _, dg = g.patches()
    _, _, do = o.patches()
    assert (np.abs(dg - do) <= 1e-3 * np.maximum(np.abs(do), 1e-3)).all()


def test_wide_patches_behind_camera_follow_the_corners(ctx):
    """A 7x7 patch whose corner pixels (not its centre) cross the camera plane is
    'behind' in the reference (any pixel, camera.cpp:47-71): its edges get zero
    weight.  The stand-in keeps the corners, so the step equals the reference."""
    K = np.array([320.0, 320.0, 320.0, 240.0])
    src_pose = np.array([0, 0, 0, 1, 0, 0, 0], float)
    # target camera rotated ~80 deg about y and shifted: the patch straddles its z = 0 plane
    tgt = orc.se3_exp(np.array([1.5, 0.0, 0.2, 0.0, 1.35, 0.0]))
    poses = np.stack([src_pose, tgt, orc.se3_exp(np.array([0.05, 0, 0, 0, 0.01, 0]))])
    p = 7
    cents = np.array([[40.0, 240.0], [320.0, 240.0], [600.0, 240.0], [320.0, 30.0]])
    half = (p - 1) / 2
    xs = np.stack([np.tile(np.arange(p) - half, p) + c[0] for c in cents])
    ys = np.stack([np.repeat(np.arange(p) - half, p) + c[1] for c in cents])
    depth = np.array([0.9, 0.5, 0.7, 0.3])
    e_patch = np.repeat(np.arange(4), 2).astype(np.int32)
    e_pose = np.tile([1, 2], 4).astype(np.int32)
    targets = np.stack([cents[k] + 1.5 for k in e_patch])
    weights = np.full((8, 2), 0.5)
    # the rotated camera is fixed (its edges only weigh depths and the residual norms)
    prob = {"poses": poses, "fixed": np.array([1, 1, 0], np.uint8), "patch_src": np.zeros(4, np.int32),
            "patch_x": xs, "patch_y": ys, "depth": depth, "e_patch": e_patch, "e_pose": e_pose,
            "e_target": targets, "e_weight": weights}
    # the scene has a patch whose centre is in front but a corner is behind the target camera
    rel = orc.compose(tgt, orc.inverse(src_pose))
    x, y, z, qw = rel[:4]
    r3 = np.array([2 * (x * z - y * qw), 2 * (y * z + x * qw), 1 - 2 * (x * x + y * y)])
    qz = [r3 @ np.stack([(xs[k] - K[2]) / K[0], (ys[k] - K[3]) / K[1], np.ones(p * p)]) + rel[6] * depth[k]
          for k in range(4)]
    assert any(q[p * p // 2] > 1e-6 and q.min() <= 1e-6 for q in qz)
    ref = orc.ba_window(prob, K, iterations=1)
    pr = pvo.BAProblem(poses, np.array([True, True, False]), prob["patch_src"], xs, ys, depth, e_patch, e_pose,
                       targets, weights, K, patch_width=p)
    sol = pvo.ba_window(pr, iterations=1, ctx=ctx)
    assert np.allclose(sol.residual_norms, ref["residual_norms"], rtol=1e-6)
    dt, dq = pose_parity(sol.poses, ref["poses"])
    assert dt.max() <= 1e-3 and dq.max() <= 1e-3
    assert (np.abs(sol.inverse_depths - ref["depth"]) <= 1e-3 * np.maximum(np.abs(ref["depth"]), 1e-3)).all()


def _star_problem(n_poses, n_edges_on_patch, p=3):
    """One patch seen from n_edges_on_patch poses (plus filler)."""
    rng = np.random.default_rng(0)
    poses = np.stack([orc.se3_exp(np.concatenate([rng.normal(0, 0.02, 3) + [0.02 * i, 0, 0], rng.normal(0, 0.01, 3)]))
                      for i in range(n_poses)])
    fixed = np.zeros(n_poses, bool)
    fixed[0] = True
    half = (p - 1) / 2
    xs = (np.tile(np.arange(p) - half, p) + 320.0)[None]
    ys = (np.repeat(np.arange(p) - half, p) + 240.0)[None]
    E = n_edges_on_patch
    e_pose = np.arange(1, E + 1, dtype=np.int32) % n_poses
    return pvo.BAProblem(poses, fixed, np.zeros(1, np.int32), xs, ys, np.array([0.5]), np.zeros(E, np.int32), e_pose,
                         np.full((E, 2), 320.0), np.full((E, 2), 0.5), [320.0, 320.0, 320.0, 240.0], patch_width=p)


def test_remaining_limits_raise_unsupported(ctx):
    with pytest.raises(pvo.Unsupported):  # even widths: the Jacobian centre is the pixel mean
        pvo.ba_window(_star_problem(4, 3, p=4), iterations=1, ctx=ctx)
    with pytest.raises(pvo.Unsupported):  # more than 32 edges on one patch (radius > 16)
        pvo.ba_window(_star_problem(40, 33), iterations=1, ctx=ctx)
    with pytest.raises(pvo.Unsupported):  # normal-equation capture beyond 16 free poses
        pvo.gauss_newton_step(_star_problem(20, 19), debug=True, ctx=ctx)
    with pytest.raises(pvo.Unsupported):  # a large-window patch run touching > 25 free poses
        pvo.ba_window(_star_problem(32, 30), iterations=1, ctx=ctx)
    # exactly 32 edges on one patch is fine (and so is the same star through the large path)
    sol = pvo.ba_window(_star_problem(17, 32), iterations=1, ctx=ctx)
    assert np.isfinite(sol.poses).all()
    ctx.frames_reserve(1, 16, 12, 4, 3, 129)
    with pytest.raises(pvo.Unsupported):  # the provider measurement holds <= 128 channels per warp
        pvo.measure_batch(np.zeros(1, np.int32), np.zeros(1, np.int32), np.zeros((1, 2)) + 8.0,
                          np.zeros((1, 2, 9, 129), np.float32), ctx=ctx)
