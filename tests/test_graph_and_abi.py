"""Host-side parity (CPU): the product PatchGraph / window flattening against
the oracle's std::map restatement — bit-exact, as the north star demands for
graph indexing — plus the C-ABI surface itself."""
import re
from pathlib import Path

import numpy as np
import pytest

import oracle.pyoracle as orc
from paper_2208_04726_b200 import PatchGraph
import pvo_synth as synth
from paper_2208_04726_b200 import api as pvo
from paper_2208_04726_b200._capi import SIGNATURES, lib
from tests.helpers import random_pose

ROOT = Path(__file__).resolve().parent.parent
K = np.array([160.0, 160.0, 128.0, 128.0])
I7 = np.array([0, 0, 0, 1.0, 0, 0, 0])


def _both(w=256, h=256):
    return PatchGraph(K, w, h), orc.PatchGraph(K, w, h)


def _same_edges(a, b):
    ea, eb = a.edges(), b.edges()
    for x, y in zip(ea, eb):
        assert np.array_equal(x, y)


def test_header_symbols_exported():
    header = (ROOT / "include" / "pvo_capi.h").read_text()
    declared = set(re.findall(r"\b(pvo_[a-z0-9_]+)\s*\(", header))
    assert declared == set(SIGNATURES), declared ^ set(SIGNATURES)
    for name in declared:
        assert hasattr(lib, name)


def test_status_strings():
    assert lib.pvo_status_string(0) == b"ok"
    assert lib.pvo_status_string(2) == b"degenerate_problem"


def test_host_se3_matches_oracle():
    rng = np.random.default_rng(1)
    for _ in range(200):
        a, b = random_pose(rng), random_pose(rng)
        xi = rng.standard_normal(6) * 0.3
        assert np.array_equal(pvo.compose(a, b), orc.compose(a, b)) or np.abs(
            pvo.compose(a, b) - orc.compose(a, b)).max() < 1e-14
        assert np.abs(pvo.inverse(a) - orc.inverse(a)).max() < 1e-14
        assert np.abs(pvo.se3_exp(xi) - orc.se3_exp(xi)).max() < 1e-14
        assert np.abs(pvo.retract(a, xi) - orc.retract(a, xi)).max() < 1e-13
        assert np.abs(pvo.se3_log(a) - orc.se3_log(a)).max() < 1e-9
    with pytest.raises(ArithmeticError):
        pvo.se3_log(orc.se3_exp([0, 0, 0, 0, 0, np.pi - 1e-9]))


def test_frame_indices_and_timestamps():  # test_patch_graph.cpp:28-34
    g, _ = _both()
    assert g.add_frame(0.0, I7) == 0 and g.add_frame(0.1, I7) == 1
    for ts in (0.1, 0.05):
        with pytest.raises(ValueError):
            g.add_frame(ts, I7)


def test_out_of_bounds_centroid_rejected():  # test_patch_graph.cpp:53-59
    g, _ = _both()
    g.add_frame(0.0, I7)
    with pytest.raises(ValueError):
        g.add_patches(0, [(0, 0)], [0.1])
    with pytest.raises(ValueError):
        g.add_patches(0, [(255.5, 100)], [0.1])
    g.add_patches(0, [(1, 1)], [0.1])


def test_connect_matches_brute_force_and_oracle():  # test_patch_graph.cpp:78-108
    rng = np.random.default_rng(3)
    for nf in range(1, 9):
        for r in range(1, 4):
            g, o = _both()
            ids = []
            for f in range(nf):
                c = rng.uniform(8, 247, (2, 2))
                g.add_frame(0.1 * f, I7)
                o.add_frame(0.1 * f, I7)
                ids += g.add_patches(f, c, [0.1, 0.1])
                o.add_patches(f, c, [0.1, 0.1])
                assert g.connect(r) == o.connect(r)
            _same_edges(g, o)
            kk, jj, _, _ = g.edges()
            expected = sorted((k, f) for k in ids for f in range(nf) if abs(f - k // 2) <= r - 1)
            assert list(zip(kk.tolist(), jj.tolist())) == expected


def test_random_operation_sequences_match_oracle():  # test_patch_graph.cpp:227-269
    rng = np.random.default_rng(7)
    for trial in range(12):
        g, o = _both()
        r = 1 + int(rng.integers(3))
        t = 0.0
        for _ in range(60):
            action = int(rng.integers(4))
            fi, _ = g.frames()
            if action <= 1 or len(fi) == 0:
                t += 0.1
                pose = random_pose(rng, 0.1, 0.1)
                c = rng.uniform(8, 247, (2, 2))
                f = g.add_frame(t, pose)
                assert f == o.add_frame(t, pose)
                g.add_patches(f, c, [0.1, 0.1])
                o.add_patches(f, c, [0.1, 0.1])
                g.connect(r)
                o.connect(r)
            elif action == 2 and len(fi) > 4:
                removable = [int(x) for x in fi[1:-3]]
                if removable:
                    victim = removable[int(rng.integers(len(removable)))]
                    g.remove_frame(victim)
                    o.remove_frame(victim)
            else:
                assert g.connect(r) == o.connect(r)
            _same_edges(g, o)
            kk, _, _, _ = g.edges()
            if len(kk):
                assert np.bincount(kk).max() <= 2 * r - 1


def test_newest_three_frames_not_removable():  # test_patch_graph.cpp:163-172
    g, _ = _both()
    for f in range(5):
        g.add_frame(0.1 * f, I7)
    for f in (4, 3, 2):
        with pytest.raises(ValueError):
            g.remove_frame(f)
    g.remove_frame(1)


def test_revision_validation_and_dump():  # test_patch_graph.cpp:271-301
    g, _ = _both()
    g.add_frame(0.0, I7)
    ids = g.add_patches(0, [(100, 100)], [0.2])
    g.connect(1)
    g.set_revision((ids[0], 0), (1.5, -2.0), (0.5, 0.25))
    kk, jj, rev, has = g.edges()
    assert kk[0] == ids[0] and jj[0] == 0 and list(rev[0]) == [1.5, -2.0, 0.5, 0.25] and has[0]
    for w in [(1.0, 0.5), (0.5, 0.0)]:
        with pytest.raises(ValueError):
            g.set_revision((ids[0], 0), (0, 0), w)
    with pytest.raises(ValueError):
        g.set_revision((ids[0], 5), (0, 0), (0.5, 0.5))


def test_build_target_kat_product():  # test_bundle_adjust.cpp:91-105
    g, _ = _both()
    g.add_frame(0.0, I7)
    g.add_frame(0.1, I7)
    ids = g.add_patches(0, [(10, 10)], [0.5])
    g.connect(2)
    with pytest.raises(ValueError):
        g.build_target((ids[0], 1))
    g.set_revision((ids[0], 1), (1, -2), (0.5, 0.5))
    assert np.linalg.norm(g.build_target((ids[0], 1)) - [11, 8]) < 1e-12


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_window_problem_bit_exact(name):
    w = synth.generate(name, features=False)
    g, o = synth.build_graph(w, PatchGraph), synth.build_graph(w, orc.PatchGraph)
    _same_edges(g, o)
    a, b = g.active_edges(w.cfg["window"]), o.active_edges(w.cfg["window"])
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(a[0], w.active_kk) and np.array_equal(a[1], w.active_jj)
    pa, pb = g.window_problem(w.cfg["window"]), o.window_problem(w.cfg["window"])
    for key in pa:
        assert np.array_equal(pa[key], pb[key]), key
    expected_edges = {"c1": 6144, "c2": 16800, "c3": 5376}[name]
    assert len(pa["e_patch"]) == expected_edges


def test_stress_edge_count():
    # C4 at r = 7 has exactly 404,480 active edges
    w = synth.generate("c4", features=False)
    assert w.n_edges == 404480


def test_window_problem_after_removal_matches_oracle():
    rng = np.random.default_rng(11)
    g, o = _both(640, 480)
    for f in range(14):
        pose = random_pose(rng, 0.05, 0.05)
        c = np.stack([rng.uniform(4, 635, 6), rng.uniform(4, 475, 6)], 1)
        d = rng.uniform(0.1, 1.0, 6)
        g.add_frame(0.1 * f, pose)
        o.add_frame(0.1 * f, pose)
        g.add_patches(f, c, d)
        o.add_patches(f, c, d)
        g.connect(5)
        o.connect(5)
        if f in (8, 11):
            g.remove_frame(f - 4)
            o.remove_frame(f - 4)
    kk, jj, _, _ = o.edges()
    for i, (k, j) in enumerate(zip(kk, jj)):
        if i % 3:
            dl, wt = rng.normal(0, 2, 2), rng.uniform(0.1, 0.9, 2)
            g.set_revision((k, j), dl, wt)
            o.set_revision((k, j), dl, wt)
    pa, pb = g.window_problem(6), o.window_problem(6)
    for key in pa:
        assert np.array_equal(pa[key], pb[key]), key


def test_add_patches_grid_and_radius_one_connect():  # test_patch_graph.cpp:38-51, :63-76
    rng = np.random.default_rng(2)
    for g in _both():
        g.add_frame(0.0, I7)
        g.add_frame(0.1, I7)
        c0 = rng.uniform(8, 248, (4, 2))
        c1 = rng.uniform(8, 248, (4, 2))
        g.add_patches(0, c0, [0.1] * 4)
        g.add_patches(1, c1, [0.1] * 4)
        g.connect(1)
        kk, jj, _, _ = g.edges()
        ids, src, d = g.patches()
        src_of = {int(i): int(s) for i, s in zip(ids, src)}
        assert len(kk) == 8 and len(set(int(k) for k in kk)) == 8  # one edge per patch
        assert all(src_of[int(k)] == int(j) for k, j in zip(kk, jj))  # ... onto its source frame
        assert np.all(d == 0.1)  # one shared inverse depth per patch grid


def test_removing_a_middle_frame_keeps_the_graph_consistent():  # test_patch_graph.cpp:110-140 (graph part)
    rng = np.random.default_rng(4)
    a, b = _both()
    for f in range(5):
        pose = random_pose(rng, 0.2, 0.2)
        c = rng.uniform(8, 248, (3, 2))
        for g in (a, b):
            g.add_frame(0.1 * f, pose)
            g.add_patches(f, c, [0.2] * 3)
            g.connect(3)
    for g in (a, b):
        g.remove_frame(1)
        idx, _ = g.frames()
        assert 1 not in set(int(i) for i in idx)
        kk, jj, _, _ = g.edges()
        ids, src, _ = g.patches()
        assert 1 not in set(int(j) for j in jj) and 1 not in set(int(s) for s in src)
        assert set(int(k) for k in kk) <= set(int(i) for i in ids)
        assert set(int(j) for j in jj) <= set(int(i) for i in idx)
    _same_edges(a, b)
