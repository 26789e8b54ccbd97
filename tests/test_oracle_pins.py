"""Pin the CPU oracle against the reference's own known-answer and property
tests (the reference ships no golden vectors).

Each test names the reference test it ports.  CPU only.
"""
import numpy as np
import pytest
import scipy.linalg

import oracle.pyoracle as orc
from tests.helpers import pose_parity, random_pose, random_twist, smooth_features

I7 = np.array([0, 0, 0, 1.0, 0, 0, 0])
KCAM = np.array([160.0, 155.0, 128.0, 126.0])  # test_camera.cpp:12


# ---------------------------------------------------------------- se3 (test_se3.cpp)
def test_exp_zero_is_identity():
    p = orc.se3_exp(np.zeros(6))
    assert p[3] == pytest.approx(1.0) and np.linalg.norm(p[4:]) == pytest.approx(0.0)


def test_exp_pure_translation():  # test_se3.cpp:18-25
    p = orc.se3_exp([1, 0, 0, 0, 0, 0])
    assert np.allclose(p, [0, 0, 0, 1, 1, 0, 0])


def test_log_90_deg_z():  # test_se3.cpp:32-39
    xi = orc.se3_log(orc.se3_exp([0, 0, 0, 0, 0, np.pi / 2]))
    assert abs(xi[3]) < 1e-12 and abs(xi[4]) < 1e-12 and xi[5] == pytest.approx(np.pi / 2)


def test_exp_log_round_trip_1000():  # test_se3.cpp:41-50
    rng = np.random.default_rng(7)
    worst = 0.0
    for _ in range(1000):
        xi = random_twist(rng, 2.0, np.pi - 0.1)
        worst = max(worst, np.abs(orc.se3_log(orc.se3_exp(xi)) - xi).max())
    assert worst < 1e-8


def test_small_angle_round_trip():  # test_se3.cpp:52-59
    rng = np.random.default_rng(8)
    for _ in range(100):
        xi = random_twist(rng, 1.0, 1e-9)
        assert np.abs(orc.se3_log(orc.se3_exp(xi)) - xi).max() < 1e-12


def test_group_axioms():  # test_se3.cpp:61-82
    rng = np.random.default_rng(9)
    for _ in range(300):
        a, b, c = random_pose(rng), random_pose(rng), random_pose(rng)
        d, ang = orc.pose_distance(orc.compose(orc.compose(a, b), c), orc.compose(a, orc.compose(b, c)))
        assert d < 1e-9 and ang < 1e-9
        d, ang = orc.pose_distance(orc.compose(a, orc.inverse(a)), I7)
        assert d < 1e-9 and ang < 1e-9
        assert abs(np.linalg.norm(orc.compose(a, b)[:4]) - 1) < 1e-9


def test_log_branch_cut_throws():  # test_se3.cpp:92-95
    with pytest.raises(ArithmeticError):
        orc.se3_log(orc.se3_exp([0, 0, 0, 0, 0, np.pi - 1e-9]))


# ---------------------------------------------------------------- camera (test_camera.cpp)
def test_patch_grid():  # test_camera.cpp:37-48
    x, y = orc.patch_make((10.5, 20.0), 3, 0.25)
    assert x[0] == 9.5 and y[0] == 19.0 and x[8] == 11.5 and y[8] == 21.0 and x[4] == 10.5


def test_identity_relative_pose_exact():  # test_camera.cpp:50-60
    rng = np.random.default_rng(3)
    pose = random_pose(rng)
    x, y = orc.patch_make((100.25, 90.75), 3, 0.5)
    pts, behind = orc.reproject_patch(pose, pose, KCAM, x, y, 0.5)
    assert np.array_equal(pts[:, 0], x) and np.array_equal(pts[:, 1], y) and not behind


def test_pure_translation_parallax():  # test_camera.cpp:62-82
    b, z = 0.3, 2.5
    x, y = orc.patch_make((110.0, 95.0), 3, 1.0 / z)
    pts, _ = orc.reproject_patch(I7, [0, 0, 0, 1, -b, 0, 0], KCAM, x, y, 1.0 / z)
    assert np.allclose(pts[:, 0] - x, -KCAM[0] * b / z, rtol=1e-12)
    assert np.allclose(pts[:, 1], y, rtol=1e-12)


def test_zero_depth_kills_parallax():  # test_camera.cpp:84-95
    rot = orc.se3_exp([0, 0, 0, 0.03, -0.05, 0.02])
    wt = orc.compose([0, 0, 0, 1, 2, -1, 1], rot)
    x, y = orc.patch_make((100, 100), 3, 0.0)
    a, _ = orc.reproject_patch(I7, rot, KCAM, x, y, 0.0)
    b, _ = orc.reproject_patch(I7, wt, KCAM, x, y, 0.0)
    assert np.abs(a - b).max() < 1e-9


def test_behind_camera_flag():  # test_camera.cpp:97-104
    x, y = orc.patch_make((128, 126), 3, 0.5)
    _, behind = orc.reproject_patch(I7, [0, 0, 0, 1, 0, 0, -5], KCAM, x, y, 0.5)
    assert behind


def _random_config(rng, d):
    while True:
        pi, pj = random_pose(rng, 0.3, 0.25), random_pose(rng, 0.3, 0.25)
        x, y = orc.patch_make((rng.uniform(40, 215), rng.uniform(40, 215)), 3, d)
        j, behind = orc.reprojection_jacobians(pi, pj, KCAM, x, y, d)
        if not behind and -200 < j[0] < 500:
            return pi, pj, x, y


def test_jacobians_finite_differences():  # test_camera.cpp:116-161
    rng = np.random.default_rng(6)
    step, worst = 1e-6, 0.0
    for _ in range(100):
        d = rng.uniform(0.05, 2.0)
        pi, pj, x, y = _random_config(rng, d)
        j, _ = orc.reprojection_jacobians(pi, pj, KCAM, x, y, d)
        di, dj, dd = j[2:14].reshape(2, 6), j[14:26].reshape(2, 6), j[26:28]

        def center(a, b, dd_):
            return orc.reproject_patch(a, b, KCAM, x, y, dd_)[0][4]

        fi, fj = np.zeros((2, 6)), np.zeros((2, 6))
        for k in range(6):
            h = np.zeros(6)
            h[k] = step
            fi[:, k] = (center(orc.retract(pi, h), pj, d) - center(orc.retract(pi, -h), pj, d)) / (2 * step)
            fj[:, k] = (center(pi, orc.retract(pj, h), d) - center(pi, orc.retract(pj, -h), d)) / (2 * step)
        fd = (center(pi, pj, d + step) - center(pi, pj, d - step)) / (2 * step)
        scale = max(1.0, np.abs(di).max(), np.abs(dj).max(), np.abs(dd).max())
        worst = max(worst, max(np.abs(di - fi).max(), np.abs(dj - fj).max(), np.abs(dd - fd).max()) / scale)
    assert worst < 1e-4


def test_equal_poses_opposite_jacobians():  # test_camera.cpp:106-114
    rng = np.random.default_rng(5)
    for _ in range(20):
        pose = random_pose(rng)
        x, y = orc.patch_make((90, 140), 3, 0.4)
        j, _ = orc.reprojection_jacobians(pose, pose, KCAM, x, y, 0.4)
        assert np.abs(j[2:14] + j[14:26]).max() < 1e-9


def test_depth_column_symbolic():  # test_camera.cpp:163-180
    rng = np.random.default_rng(11)
    for _ in range(5):
        pi, pj, x, y = _random_config(rng, 0.0)
        rel = orc.compose(pj, orc.inverse(pi))
        q = np.array(orc.reproject_patch(I7, [*rel[:4], 0, 0, 0], [1, 1, 0, 0], [x[4]], [y[4]], 0.0)[0][0])
        # q = R ray via a unit-focal projection is awkward; recompute directly
        qx, qy, qw = rel[0], rel[1], rel[3]
        qz_ = rel[2]
        R = np.array([[1 - 2 * (qy * qy + qz_ * qz_), 2 * (qx * qy - qz_ * qw), 2 * (qx * qz_ + qy * qw)],
                      [2 * (qx * qy + qz_ * qw), 1 - 2 * (qx * qx + qz_ * qz_), 2 * (qy * qz_ - qx * qw)],
                      [2 * (qx * qz_ - qy * qw), 2 * (qy * qz_ + qx * qw), 1 - 2 * (qx * qx + qy * qy)]])
        ray = np.array([(x[4] - KCAM[2]) / KCAM[0], (y[4] - KCAM[3]) / KCAM[1], 1.0])
        qv = R @ ray
        t = rel[4:]
        expected = np.array([KCAM[0] * (t[0] * qv[2] - t[2] * qv[0]) / qv[2] ** 2,
                             KCAM[1] * (t[1] * qv[2] - t[2] * qv[1]) / qv[2] ** 2])
        j, _ = orc.reprojection_jacobians(pi, pj, KCAM, x, y, 0.0)
        assert np.linalg.norm(j[26:28] - expected) < 1e-9 * max(1.0, np.linalg.norm(expected))
        del q


def test_gauge_invariance():  # test_camera.cpp:182-195
    rng = np.random.default_rng(12)
    for _ in range(50):
        pi, pj, x, y = _random_config(rng, 0.5)
        g = random_pose(rng)
        a, _ = orc.reproject_patch(pi, pj, KCAM, x, y, 0.5)
        b, _ = orc.reproject_patch(orc.compose(pi, g), orc.compose(pj, g), KCAM, x, y, 0.5)
        assert np.abs(a - b).max() < 1e-9


# ---------------------------------------------------------------- correlation (test_features.cpp:144-245)
def _pyramid(seed, H=64, W=64, D=25):
    rng = np.random.default_rng(seed)
    import pvo_synth as synth

    l0 = smooth_features(rng, H, W, D)
    l1 = synth.make_level1(l0[None])[0]
    return l0, l1


def _crop(l0, l1, centroid):
    import pvo_synth as synth

    x, y = orc.patch_make(centroid, 3, 1.0)
    return (synth.crop_cubic(l0, x / 4.0, y / 4.0), synth.crop_cubic(l1, x / 16.0, y / 16.0)), np.stack([x, y], 1)


def test_self_match_peaks_at_center():  # test_features.cpp:144-169
    l0, l1 = _pyramid(17)
    rng = np.random.default_rng(13)
    for _ in range(10):
        feats, coords = _crop(l0, l1, (rng.uniform(30, 220), rng.uniform(30, 220)))
        grid = orc.correlate(feats, (l0, l1), coords)
        for v in range(3):
            for u in range(3):
                assert grid[0, v, u, 3, 3] >= grid[0, v, u].max() - 1e-6


def test_zero_map_gives_zero_grid():  # test_features.cpp:171-184
    l0, l1 = np.zeros((32, 32, 1), np.float32), np.zeros((8, 8, 1), np.float32)
    feats = (np.ones((9, 1), np.float32), np.ones((9, 1), np.float32))
    x, y = orc.patch_make((60, 60), 3, 1.0)
    grid = orc.correlate(feats, (l0, l1), np.stack([x, y], 1))
    assert not grid.any()


def test_displaced_peak_moves_opposite():  # test_features.cpp:186-217
    l0, l1 = _pyramid(23)
    feats, coords = _crop(l0, l1, (120, 132))
    rng = np.random.default_rng(14)
    for _ in range(8):
        a, b = int(rng.integers(7)) - 3, int(rng.integers(7)) - 3
        grid = orc.correlate(feats, (l0, l1), coords + np.array([4.0 * a, 4.0 * b]))
        al, be = np.unravel_index(np.argmax(grid[0, 1, 1]), (7, 7))
        assert al == 3 - b and be == 3 - a


def test_correlation_linear_in_patch_features():  # test_features.cpp:219-245
    l0, l1 = _pyramid(29)
    x, y = orc.patch_make((100, 80), 3, 1.0)
    coords = np.stack([x, y], 1)
    rng = np.random.default_rng(15)
    g1 = [rng.standard_normal((9, 25)).astype(np.float32) for _ in range(2)]
    g2 = [rng.standard_normal((9, 25)).astype(np.float32) for _ in range(2)]
    gs = [g1[i] + g2[i] for i in range(2)]
    c1, c2, cs = (orc.correlate(g, (l0, l1), coords) for g in (g1, g2, gs))
    assert np.allclose(cs, c1 + c2, rtol=1e-5, atol=1e-6)


def test_correlate_rejects_non_finite():  # correlation.cpp:43-45
    l0, l1 = _pyramid(3)
    feats, coords = _crop(l0, l1, (50, 50))
    coords[2, 0] = np.nan
    with pytest.raises(ValueError):
        orc.correlate(feats, (l0, l1), coords)


def test_correlate_at_matches_sampler_definition():  # correlation.cpp:8-23, features.cpp:9-21
    l0, _ = _pyramid(31, 16, 16, 5)
    g = np.arange(5, dtype=np.float32) - 2
    for x, y in [(3.25, 4.5), (-0.5, 2.0), (15.5, 15.5), (7.0, 7.0)]:
        v = np.array([orc.sample_zero_padded(l0, x, y, c) for c in range(5)])
        n2 = (v * v).sum()
        ref = (g * v).sum() / np.sqrt(n2) if n2 > 1e-12 else 0.0
        assert orc.correlate_at(g, l0, x, y) == pytest.approx(ref, rel=1e-12, abs=1e-15)


# ---------------------------------------------------------------- bundle adjustment (test_bundle_adjust.cpp)
KBA = np.array([160.0, 160.0, 128.0, 128.0])


def random_system(rng, num_poses, num_depths):  # test_bundle_adjust.cpp:27-53
    npp = 6 * num_poses
    hpp, hpd = np.zeros((npp, npp)), np.zeros((npp, num_depths))
    hdd, bp, bd = np.zeros(num_depths), np.zeros(npp), np.zeros(num_depths)
    for d in range(num_depths):
        for _ in range(2 + int(rng.integers(4))):
            pose = int(rng.integers(num_poses))
            jp, jd, r = rng.standard_normal((2, 6)), rng.standard_normal(2), rng.standard_normal(2)
            s = slice(6 * pose, 6 * pose + 6)
            hpp[s, s] += jp.T @ jp
            hpd[s, d] += jp.T @ jd
            hdd[d] += jd @ jd
            bp[s] -= jp.T @ r
            bd[d] -= jd @ r
    hpp[np.diag_indices(npp)] += 1e-4
    hdd += 1e-4
    return hpp, hpd, hdd, bp, bd


def two_view_problem(rng, edges, depths_free=True):  # test_bundle_adjust.cpp:57-83
    p1 = orc.compose(orc.se3_exp(random_twist(rng, 0.05, 0.05)), [0, 0, 0, 1, -0.4, 0.05, 0.02])
    px, py, d, tgt, w = [], [], [], [], []
    for _ in range(edges):
        x, y = orc.patch_make((rng.uniform(32, 223), rng.uniform(32, 223)), 3, 0.0)
        px.append(x)
        py.append(y)
        d.append(rng.uniform(0.2, 1.0))
        tgt.append([rng.uniform(32, 223), rng.uniform(32, 223)])
        w.append([0.3 + 0.4 * int(rng.integers(100)) / 100.0, 0.3 + 0.4 * int(rng.integers(100)) / 100.0])
    pr = dict(poses=np.stack([I7, p1]), fixed=np.array([1, 0], np.uint8), patch_src=np.zeros(edges, np.int32),
              patch_x=np.array(px), patch_y=np.array(py), depth=np.array(d), e_patch=np.arange(edges, dtype=np.int32),
              e_pose=np.ones(edges, np.int32), e_target=np.array(tgt), e_weight=np.array(w))
    dfree = None if depths_free else np.zeros(edges, np.uint8)
    return pr, dfree


def test_build_target_kat():  # test_bundle_adjust.cpp:91-105
    g = orc.PatchGraph(KBA, 256, 256)
    g.add_frame(0.0, I7)
    g.add_frame(0.1, I7)
    ids = g.add_patches(0, [(10, 10)], [0.5])
    g.connect(2)
    with pytest.raises(ValueError):
        g.build_target((ids[0], 1))
    g.set_revision((ids[0], 1), (0, 0), (0.5, 0.5))
    assert np.linalg.norm(g.build_target((ids[0], 1)) - [10, 10]) < 1e-12
    g.set_revision((ids[0], 1), (1, -2), (0.5, 0.5))
    assert np.linalg.norm(g.build_target((ids[0], 1)) - [11, 8]) < 1e-12


def test_zero_residual_zero_update():  # test_bundle_adjust.cpp:107-128
    rng = np.random.default_rng(31)
    pr, _ = two_view_problem(rng, 12)
    for e in range(12):
        pts, _ = orc.reproject_patch(pr["poses"][0], pr["poses"][1], KBA, pr["patch_x"][e], pr["patch_y"][e],
                                     pr["depth"][e])
        pr["e_target"][e] = pts[4]
    s = orc.gauss_newton_step(pr, KBA)
    d, ang = orc.pose_distance(s["poses"][1], pr["poses"][1])
    assert d < 1e-12 and ang < 1e-12
    assert np.abs(s["depth"] - pr["depth"]).max() < 1e-12
    assert s["residual_norms"][0] == pytest.approx(0.0)


def test_single_free_pose_matches_dense_wls():  # test_bundle_adjust.cpp:135-171
    rng = np.random.default_rng(32)
    for _ in range(5):
        pr, dfree = two_view_problem(rng, 20, depths_free=False)
        h, b = np.zeros((6, 6)), np.zeros(6)
        for e in range(20):
            j, _ = orc.reprojection_jacobians(pr["poses"][0], pr["poses"][1], KBA, pr["patch_x"][e],
                                              pr["patch_y"][e], pr["depth"][e])
            r = j[0:2] - pr["e_target"][e]
            jj = j[14:26].reshape(2, 6)
            W = np.diag(pr["e_weight"][e])
            h += jj.T @ W @ jj
            b -= jj.T @ W @ r
        h[np.diag_indices(6)] += 1e-4
        expected = scipy.linalg.lstsq(h, b)[0]
        s = orc.gauss_newton_step(pr, KBA, depth_free=dfree, debug=True)
        d, ang = orc.pose_distance(s["poses"][1], orc.retract(pr["poses"][1], expected))
        assert d < 1e-8 and ang < 1e-8
        assert s["num_free_poses"] == 1 and s["num_free_depths"] == 0
        assert np.abs(s["h"] - h).max() < 1e-9 * max(1.0, np.abs(h).max())
        assert np.abs(s["b"] - b).max() < 1e-9 * max(1.0, np.abs(b).max())
        assert np.array_equal(s["poses"][0], pr["poses"][0])


def test_normal_equations_symmetric():  # test_bundle_adjust.cpp:173-196
    rng = np.random.default_rng(33)
    pr, _ = two_view_problem(rng, 8)
    s = orc.gauss_newton_step(pr, KBA, debug=True)
    assert s["h"].shape == (14, 14)
    assert np.abs(s["h"] - s["h"].T).max() < 1e-9 * max(1.0, np.abs(s["h"]).max())


def test_schur_decoupled():  # test_bundle_adjust.cpp:198-210
    rng = np.random.default_rng(34)
    hpp, hpd, hdd, bp, bd = random_system(rng, 3, 10)
    hpd[:] = 0
    dp, dd = orc.schur_solve(hpp, hpd, hdd, bp, bd)
    assert np.abs(dp - np.linalg.solve(hpp, bp)).max() < 1e-10
    assert np.abs(dd - bd / hdd).max() < 1e-10


def test_schur_matches_dense_lu():  # test_bundle_adjust.cpp:212-236
    rng = np.random.default_rng(35)
    for _ in range(10):
        nposes, nd = 2 + int(rng.integers(5)), 10 + int(rng.integers(41))
        hpp, hpd, hdd, bp, bd = random_system(rng, nposes, nd)
        npp = 6 * nposes
        full = np.zeros((npp + nd, npp + nd))
        full[:npp, :npp], full[:npp, npp:], full[npp:, :npp] = hpp, hpd, hpd.T
        full[npp:, npp:] = np.diag(hdd)
        dense = scipy.linalg.lu_solve(scipy.linalg.lu_factor(full), np.concatenate([bp, bd]))
        dp, dd = orc.schur_solve(hpp, hpd, hdd, bp, bd)
        assert np.abs(np.concatenate([dp, dd]) - dense).max() / max(1.0, np.abs(dense).max()) < 1e-8


def test_schur_closed_form_7x7():  # test_bundle_adjust.cpp:238-252
    rng = np.random.default_rng(36)
    hpp, hpd, hdd, bp, bd = random_system(rng, 1, 1)
    full = np.zeros((7, 7))
    full[:6, :6], full[:6, 6], full[6, :6], full[6, 6] = hpp, hpd[:, 0], hpd[:, 0], hdd[0]
    dense = np.linalg.inv(full) @ np.concatenate([bp, bd])
    dp, dd = orc.schur_solve(hpp, hpd, hdd, bp, bd)
    assert np.abs(dp - dense[:6]).max() < 1e-8 and abs(dd[0] - dense[6]) < 1e-8


def test_schur_rejects_non_positive_depth_block():  # test_bundle_adjust.cpp:254-260
    rng = np.random.default_rng(37)
    hpp, hpd, hdd, bp, bd = random_system(rng, 1, 3)
    hdd[1] = 0.0
    with pytest.raises(orc.OracleDegenerate):
        orc.schur_solve(hpp, hpd, hdd, bp, bd)


def test_ldlt_restatement_matches_scipy():  # Eigen LDLT restated
    rng = np.random.default_rng(38)
    for n in (1, 6, 42, 60):
        a = rng.standard_normal((n, n))
        a = a @ a.T + 1e-3 * np.eye(n)
        rhs = rng.standard_normal(n)
        x, ok = orc.ldlt_solve(a, rhs)
        assert ok
        assert np.abs(x - scipy.linalg.solve(a, rhs, assume_a="pos")).max() < 1e-8 * max(1, np.abs(x).max())


def test_weight_damping_scale_invariance():  # test_bundle_adjust.cpp:373-389
    rng = np.random.default_rng(38)
    pr, _ = two_view_problem(rng, 16)
    pr["e_weight"] *= 0.5
    a = orc.gauss_newton_step(pr, KBA, damping=1e-4)
    pr2 = dict(pr)
    pr2["e_weight"] = pr["e_weight"] * 2.0
    b = orc.gauss_newton_step(pr2, KBA, damping=2e-4)
    d, ang = orc.pose_distance(a["poses"][1], b["poses"][1])
    assert d < 1e-9 and ang < 1e-9
    assert np.abs(a["depth"] - b["depth"]).max() < 1e-9


def test_inverse_depths_clamped_at_zero():  # test_bundle_adjust.cpp:391-406
    rng = np.random.default_rng(39)
    pr, _ = two_view_problem(rng, 6)
    pr["depth"][:] = 1e-6
    for e in range(6):
        j, _ = orc.reprojection_jacobians(pr["poses"][0], pr["poses"][1], KBA, pr["patch_x"][e], pr["patch_y"][e],
                                          pr["depth"][e])
        dd = j[26:28]
        pr["e_target"][e] = j[0:2] - 50.0 * dd / np.linalg.norm(dd)
    s = orc.gauss_newton_step(pr, KBA)
    assert (s["depth"] >= 0).all()


def test_behind_camera_edges_not_fatal():  # test_bundle_adjust.cpp:408-417
    g = orc.PatchGraph(KBA, 256, 256)
    g.add_frame(0.0, I7)
    g.add_frame(0.1, [0, 0, 0, 1, 0.01, 0, 0])
    g.add_frame(0.2, [0, 0, 0, 1, 0, 0, -10])
    g.add_patches(0, [(128, 128), (90, 110)], [0.5, 0.4])
    g.connect(3)
    kk, jj, _, _ = g.edges()
    for k, j in zip(kk, jj):
        g.set_revision((k, j), (0.1, -0.1), (0.5, 0.5))
    g.optimize_window(window=3)


def _gt_graph(seed, frames, patches, radius, noise, window, weight=0.9, graph_cls=None):
    """graph_at_ground_truth + set_oracle_revisions analogue on a synth workload
    (sim_fixtures.hpp:13-85): exact GT-pointing deltas, uniform weight."""
    import pvo_synth as synth

    w = synth.generate("c1", seed=seed, features=False, frames=frames, patches=patches)
    w.cfg["radius"] = radius
    w.cfg["window"] = window
    g = (graph_cls or orc.PatchGraph)(w.K, w.image[0], w.image[1])
    rng = np.random.default_rng(seed)
    for f in range(frames):
        g.add_frame(0.05 * f, w.gt_poses[f])
        ks = slice(f * patches, (f + 1) * patches)
        g.add_patches(f, w.centroids[ks], w.gt_depth[ks])
        g.connect(radius)
    idx, _ = g.frames()
    for f in idx[-noise[0]:]:
        if f == 0:
            continue
        tw = random_twist(rng, 1.0, 1.0)
        g.set_pose(int(f), orc.retract(w.gt_poses[f], noise[1] * tw / np.linalg.norm(tw)))
    kk, jj, _, _ = g.edges()
    gt_pts = {}
    for k, j in zip(kk, jj):
        x, y = orc.patch_make(w.centroids[k], 3, 0.0)
        gt, _ = orc.reproject_patch(w.gt_poses[w.patch_src[k]], w.gt_poses[j], w.K, x, y, w.gt_depth[k])
        ids, src, dep = None, None, None
        _, poses = g.frames()
        cur, _ = orc.reproject_patch(poses[w.patch_src[k]], poses[j], w.K, x, y, w.gt_depth[k])
        gt_pts[(k, j)] = gt[4]
        g.set_revision((k, j), gt[4] - cur[4], (weight, weight))
    return w, g, gt_pts


def test_optimize_window_recovers_ground_truth():  # test_bundle_adjust.cpp:262-288
    w, g, gt_pts = _gt_graph(101, 20, 24, 13, (10, 1e-3), 10)
    norms, ne = g.optimize_window(window=10)
    assert len(norms) == 3
    _, poses = g.frames()
    for f in range(10, 20):
        d, ang = orc.pose_distance(poses[f], w.gt_poses[f])
        assert d < 1e-4


def test_poses_outside_window_bit_exact():  # test_bundle_adjust.cpp:290-308
    w, g, _ = _gt_graph(102, 16, 12, 13, (16, 5e-3), 10, weight=0.5)
    _, before = g.frames()
    g.optimize_window(window=10)
    _, after = g.frames()
    assert np.array_equal(before[:6], after[:6])


def test_residual_non_increasing():  # test_bundle_adjust.cpp:310-334 (reduced seed count)
    failures = 0
    for seed in range(10):
        w, g, _ = _gt_graph(200 + seed, 12, 16, 8, (12, 5e-3), 12, weight=0.8)
        norms, _ = g.optimize_window(window=12)
        if norms[-1] > norms[0] + 1e-12:
            failures += 1
    assert failures <= 1


# ---------------------------------------------------------------- provider measure()
# CorrelationFlowProvider::measure (flow_provider.cpp:209-287), the "next" row of
# SURVEY.md §8f.  The reference's own tests (test_features.cpp:246-340) use its
# image feature extractor (out of scope); these ports keep their properties on
# the synthetic 128-d feature grids the rest of the suite uses.
def _measure_one(g_patch, lvl0, lvl1, center):
    pf = np.asarray(g_patch, np.float32)[None]
    d, w, fl = orc.measure_batch([0], [0], np.array([center], float), None, pf, lvl0[None], lvl1[None])
    return d[0], w[0], int(fl[0])


def _crop_patch(lvl0, lvl1, centroid):
    import pvo_synth as synth

    px, py = _patch_grid(centroid)  # Patch::make grid (camera.cpp:15-38)
    g0 = synth.crop_cubic(lvl0, px / 4.0, py / 4.0)
    g1 = synth.crop_cubic(lvl1, px / 16.0, py / 16.0)
    return np.stack([g0, g1])  # [2][9][C]


def _patch_grid(centroid):
    gx, gy = np.meshgrid(np.arange(3) - 1.0, np.arange(3) - 1.0)
    return centroid[0] + gx.ravel(), centroid[1] + gy.ravel()


def _smooth_grid(rng, H, W, D, passes=3):
    import pvo_synth as synth

    g = synth.make_level0(rng, 1, H, W, D)[0]
    for _ in range(passes - 1):  # extra blur passes: a smoother field for subpixel accuracy
        pad = np.pad(g, ((1, 1), (1, 1), (0, 0)))
        g = (pad[:-2, 1:-1] + 2 * pad[1:-1, 1:-1] + pad[2:, 1:-1]) / 4
        pad = np.pad(g, ((1, 1), (1, 1), (0, 0)))
        g = (pad[1:-1, :-2] + 2 * pad[1:-1, 1:-1] + pad[1:-1, 2:]) / 4
        g /= np.linalg.norm(g, axis=-1, keepdims=True) + 1e-12
    return np.ascontiguousarray(g, np.float32)


def _level1(g):
    import pvo_synth as synth

    return synth.make_level1(g[None])[0]


def test_measure_self_match_zero_and_confident():  # test_features.cpp:246-263
    rng = np.random.default_rng(16)
    l0 = _smooth_grid(rng, 64, 64, 32)
    l1 = _level1(l0)
    confident = 0
    for _ in range(50):
        c = rng.uniform(20.0, 235.0, 2)
        d, w, fl = _measure_one(_crop_patch(l0, l1, c), l0, l1, c)
        assert np.linalg.norm(d) < 0.05 and fl == 0
        confident += w[0] > 0.5
    assert confident > 45


def test_measure_equivariant_at_whole_cell_shifts():  # test_features.cpp:265-300 (4 px = 1 cell)
    rng = np.random.default_rng(18)
    worst = 0.0
    for _ in range(12):
        l0 = _smooth_grid(rng, 64, 64, 32)
        a, b = rng.integers(-2, 3, 2)
        t0 = np.zeros_like(l0)  # target = source moved by (a, b) cells (zero fill)
        ys, xs = slice(max(b, 0), 64 + min(b, 0)), slice(max(a, 0), 64 + min(a, 0))
        ys2, xs2 = slice(max(-b, 0), 64 + min(-b, 0)), slice(max(-a, 0), 64 + min(-a, 0))
        t0[ys, xs] = l0[ys2, xs2]
        c = rng.uniform(60.0, 190.0, 2)
        d, _, _ = _measure_one(_crop_patch(l0, _level1(l0), c), t0, _level1(t0), c)
        worst = max(worst, np.linalg.norm(d - 4.0 * np.array([a, b])))
    assert worst < 0.25


def test_measure_half_cell_shift_in_bands():  # test_features.cpp:302-322 (2 px pure-x shift)
    rng = np.random.default_rng(19)
    for _ in range(8):
        l0 = _smooth_grid(rng, 64, 64, 32)
        t0 = np.zeros_like(l0)  # target(x) = source(x - 0.5 cell): linear half-cell resample
        t0[:, 1:] = 0.5 * (l0[:, 1:] + l0[:, :-1])
        t0 /= np.linalg.norm(t0, axis=-1, keepdims=True) + 1e-12
        c = rng.uniform(60.0, 190.0, 2)
        d, _, _ = _measure_one(_crop_patch(l0, _level1(l0), c), t0, _level1(t0), c)
        assert 1.5 <= d[0] <= 2.5 and -0.5 <= d[1] <= 0.5


def test_measure_flat_region():  # test_features.cpp:324-340
    l0 = np.full((64, 64, 8), 0.5, np.float32)
    l1 = _level1(l0)
    d, w, fl = _measure_one(np.zeros((2, 9, 8), np.float32), l0, l1, (128.0, 128.0))
    assert fl & 1 and np.allclose(d, 0.0) and np.allclose(w, 0.01)


def test_measure_behind_camera_default_revision():  # flow_provider.cpp:301-302
    l0 = np.ones((8, 8, 4), np.float32)
    d, w, fl = orc.measure_batch([0], [0], np.zeros((1, 2)), np.array([1], np.uint8),
                                 np.ones((1, 2, 9, 4), np.float32), l0[None], _level1(l0)[None])
    assert fl[0] == 4 and np.allclose(d, 0) and np.allclose(w, 0.01)


# ---------------------------------------------------------------- feature extraction
# extract_features / whiten / lift / crop (features.cpp:55-235), SURVEY.md §8f row 2;
# ported from test_features.cpp:38-142 on smooth random images.
def _smooth_image(rng, h, w, blur=4):
    img = rng.standard_normal((h + 2 * blur, w + 2 * blur))
    k = np.exp(-0.5 * (np.arange(-2 * blur, 2 * blur + 1) / blur) ** 2)
    k /= k.sum()
    img = np.apply_along_axis(lambda r: np.convolve(r, k, "same"), 1, img)
    img = np.apply_along_axis(lambda c: np.convolve(c, k, "same"), 0, img)
    return img[blur:-blur, blur:-blur].astype(np.float32)


def test_constant_image_gives_zero_features():  # test_features.cpp:38-44
    l0, l1 = orc.extract_features(np.full((64, 64), 0.37, np.float32))
    assert l0.shape == (16, 16, 25) and l1.shape == (4, 4, 25)
    assert np.abs(l0).max() == 0 and np.abs(l1).max() == 0


def test_levels_pool_and_unit_descriptors():  # test_features.cpp:46-87, :126-142
    l0, l1 = orc.extract_features(_smooth_image(np.random.default_rng(5), 128, 128))
    assert l0.shape == (32, 32, 25) and l1.shape == (8, 8, 25)
    n0 = (l0.astype(np.float64) ** 2).sum(-1)
    n1 = (l1.astype(np.float64) ** 2).sum(-1)
    assert np.allclose(n0, 1.0, atol=1e-5) and np.allclose(n1, 1.0, atol=1e-5)


def test_level0_correlation_peaks_at_integer_shift():  # test_features.cpp:89-116
    rng = np.random.default_rng(9)
    big = _smooth_image(rng, 176, 176)
    a = np.ascontiguousarray(big[8:168, 8:168])
    sx, sy = 2, -1  # whole level-0 cells (4 px)
    b = np.ascontiguousarray(big[8 - 4 * sy:168 - 4 * sy, 8 - 4 * sx:168 - 4 * sx])
    fa, _ = orc.extract_features(a)
    fb, _ = orc.extract_features(b)
    best, arg = -1e30, None
    for dy in range(-4, 5):
        for dx in range(-4, 5):
            dot = (fa[8:-8, 8:-8, 12].astype(np.float64) * fb[8 + dy:fb.shape[0] - 8 + dy, 8 + dx:fb.shape[1] - 8 + dx, 12]).sum()
            if dot > best:
                best, arg = dot, (dx, dy)
    assert arg == (sx, sy)


def test_gradient_channels_appended():  # test_features.cpp:118-124
    l0, _ = orc.extract_features(_smooth_image(np.random.default_rng(11), 96, 96), base_channels=3)
    assert l0.shape[2] == 75
    d = l0[5, 5].reshape(5, 5, 3)  # (dy, dx, c) stacking, one normalisation per descriptor
    assert np.isclose(d[2, 2, 1], 0.5 * (d[2, 3, 0] - d[2, 1, 0]), atol=1e-6)


def test_crop_matches_sampler_definition():  # features.cpp:204-224 with sample_cubic (:23-52)
    rng = np.random.default_rng(12)
    l0, l1 = orc.extract_features(_smooth_image(rng, 96, 96))
    cents = np.array([[30.3, 41.7], [50.0, 20.25]])
    gx, gy = np.meshgrid(np.arange(3) - 1.0, np.arange(3) - 1.0)
    px = cents[:, :1] + gx.ravel()[None]
    py = cents[:, 1:] + gy.ravel()[None]
    out = orc.crop_patches(px, py, l0, l1)
    import pvo_synth as synth

    ref0 = synth.crop_cubic(l0, px[1] / 4.0, py[1] / 4.0)
    assert np.allclose(out[1, 0], ref0, atol=1e-6)


# ---------------------------------------------------------------- oracle provider (flow_provider.cpp:34-93)
def _gt_window(seed, frames, patches, radius):
    """graph_at_ground_truth (sim_fixtures.hpp) on a synth scene, flattened over
    every frame: the problem plus the scene poses / inverse depths per slot."""
    import pvo_synth as synth

    w = synth.generate("c1", seed=seed, features=False, frames=frames, patches=patches)
    g = orc.PatchGraph(w.K, w.image[0], w.image[1])
    for f in range(frames):
        g.add_frame(0.05 * f, w.gt_poses[f])
        ks = slice(f * patches, (f + 1) * patches)
        g.add_patches(f, w.centroids[ks], w.gt_depth[ks])
        g.connect(radius)
    kk, jj, _, _ = g.edges()
    for k, j in zip(kk, jj):  # the flattening takes edges with a revision
        g.set_revision((int(k), int(j)), (0.0, 0.0), (0.5, 0.5))
    prob = g.window_problem(frames)
    return w, prob, w.gt_poses[prob["pose_frames"]], w.gt_depth[prob["patch_ids"]]


def test_oracle_revisions_vanish_at_ground_truth():  # test_features.cpp:344-367
    w, prob, gtp, gtd = _gt_window(77, 8, 16, 4)
    delta, weight = orc.oracle_propose(prob, gtp, gtd, w.K)
    assert len(delta) == len(prob["e_patch"]) > 0
    assert np.all(np.linalg.norm(delta, axis=1) < 1e-9)
    assert np.allclose(weight, 0.99)


def test_oracle_outlier_fraction_exact():  # test_features.cpp:369-394
    w, prob, gtp, gtd = _gt_window(78, 6, 20, 4)
    E = len(prob["e_patch"])
    delta, weight = orc.oracle_propose(prob, gtp, gtd, w.K, outlier_fraction=0.1, seed=3)
    assert int(np.sum(np.isclose(weight[:, 0], 0.01))) == int(0.1 * E)
    # the outliers are uniform in [-32, 32); the rest stay at the ground truth
    out = np.isclose(weight[:, 0], 0.01)
    assert np.all(np.abs(delta[out]) <= 32.0) and np.all(np.linalg.norm(delta[~out], axis=1) < 1e-9)


def test_oracle_noise_statistics():  # flow_provider.cpp:56-66: N(0, sigma^2) per axis, weight 1/(1+sigma^2)
    w, prob, gtp, gtd = _gt_window(79, 10, 48, 4)
    sigma = 0.8
    delta, weight = orc.oracle_propose(prob, gtp, gtd, w.K, flow_sigma=sigma, seed=11)
    assert np.allclose(weight, 1.0 / (1.0 + sigma * sigma))
    assert abs(delta.std() - sigma) < 0.05 and abs(delta.mean()) < 0.05
    again, _ = orc.oracle_propose(prob, gtp, gtd, w.K, flow_sigma=sigma, seed=11)
    other, _ = orc.oracle_propose(prob, gtp, gtd, w.K, flow_sigma=sigma, seed=12)
    assert np.array_equal(delta, again) and not np.array_equal(delta, other)


def test_extra_consistent_anchor_leaves_minimizer_unchanged():  # test_bundle_adjust.cpp:334-367
    """Two fixed poses with a baseline pin the gauge (scale included): fixing a
    third, consistent pose (window 5 instead of 6 of 8 frames) must not move the
    minimizer of optimize_window(4 iterations)."""
    def solve(window):
        w, g, _ = _gt_graph(103, 8, 48, 8, (5, 1e-3), window)  # frames 3..7 perturbed
        g.optimize_window(window=window, iterations=4)
        return g.frames()[1]

    two, three = solve(6), solve(5)
    for a, b in zip(two, three):
        d, ang = orc.pose_distance(a, b)
        assert d < 1e-6 and ang < 1e-6


def test_damping_constant():  # test_bundle_adjust.cpp:130-133
    from paper_2208_04726_b200 import api

    assert api.kDefaultDamping == 1e-4 and api.BAProblem.__dataclass_fields__["damping"].default == 1e-4
