"""GPU parity of the reference-signature operators added for the drop-in layer.

* correlate_at / correlate_at_cubic (correlation.cpp:8-35) at free points,
  any channel count, inside / across / far outside the grid borders, against
  the oracle (FP64 both sides: 1e-12 relative);
* correlate() (correlation.cpp:37-71) at patch widths other than 3 (direct
  FP64 form) against the oracle, at the north_star tolerance 1e-4;
* the device grid cache behind the host-pyramid calls: one upload per
  pyramid, a changed pyramid is re-uploaded.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2208_04726_b200 as pvo
from tests.helpers import smooth_features

pytestmark = pytest.mark.gpu


def _points(rng, n, W, H):
    xy = np.column_stack([rng.uniform(-3, W + 2, n), rng.uniform(-3, H + 2, n)])
    xy[:8] = [[0, 0], [W - 1, H - 1], [-1.0, 3.5], [W - 0.5, 2.0], [2.25, -0.75], [1e6, 3], [-2.0, -2.0],
              [W + 0.999, H + 0.5]]
    return xy


@pytest.mark.parametrize("C", [7, 25, 128])
@pytest.mark.parametrize("cubic", [False, True])
def test_correlate_points_matches_oracle(ctx, orc, C, cubic):
    rng = np.random.default_rng(C + 100 * cubic)
    H, W = 13, 17
    grid = rng.standard_normal((H, W, C)).astype(np.float32)
    n = 300
    feats = rng.standard_normal((n, C)).astype(np.float32)
    xy = _points(rng, n, W, H)
    got = pvo.correlate_points(feats, grid, xy, cubic=cubic, ctx=ctx)
    fn = orc.correlate_at_cubic if cubic else orc.correlate_at
    ref = np.array([fn(feats[i], grid, xy[i, 0], xy[i, 1]) for i in range(n)])
    assert np.all(np.abs(got - ref) <= 1e-12 * np.maximum(1.0, np.abs(ref))), np.abs(got - ref).max()
    assert got[5] == 0.0  # far outside: only padding


def test_correlate_at_single(ctx, orc):
    rng = np.random.default_rng(5)
    grid = smooth_features(rng, 30, 40, 128)
    g = grid[10, 12].copy()
    assert abs(pvo.correlate_at(g, grid, 12.0, 10.0, ctx=ctx) - orc.correlate_at(g, grid, 12.0, 10.0)) < 1e-12
    assert abs(pvo.correlate_at(g, grid, 12.0, 10.0, ctx=ctx) - 1.0) < 1e-6  # self-match of a unit descriptor
    v = pvo.correlate_at_cubic(g, grid, 12.3, 9.6, ctx=ctx)
    assert abs(v - orc.correlate_at_cubic(g, grid, 12.3, 9.6)) < 1e-12


@pytest.mark.parametrize("p", [1, 2, 4, 5])
def test_correlate_any_patch_width(ctx, orc, p):
    rng = np.random.default_rng(p)
    C = 32
    l0 = smooth_features(rng, 30, 40, C)
    l1 = smooth_features(rng, 8, 10, C)
    pp = p * p
    g0 = rng.standard_normal((pp, C)).astype(np.float32)
    g1 = rng.standard_normal((pp, C)).astype(np.float32)
    reproj = np.column_stack([rng.uniform(-20, 180, pp), rng.uniform(-20, 140, pp)])
    got = pvo.correlate((g0, g1), (l0, l1), reproj, ctx=ctx)
    ref = orc.correlate((g0, g1), (l0, l1), reproj)
    assert got.shape == (2, p, p, 7, 7)
    gn = np.stack([np.linalg.norm(g0, axis=1), np.linalg.norm(g1, axis=1)]).reshape(2, p, p, 1, 1)
    tol = 1e-4 * np.maximum(np.abs(ref), 1e-3 * gn)
    assert np.all(np.abs(got.astype(np.float64) - ref) <= tol)


def test_host_pyramid_cache(ctx, orc):
    rng = np.random.default_rng(9)
    C = 128
    l0 = smooth_features(rng, 30, 40, C)
    l1 = smooth_features(rng, 8, 10, C)
    g0 = rng.standard_normal((9, C)).astype(np.float32)
    g1 = rng.standard_normal((9, C)).astype(np.float32)
    s0 = pvo.grid_cache_stats(ctx)
    outs = []
    for i in range(6):
        reproj = np.column_stack([rng.uniform(0, 160, 9), rng.uniform(0, 120, 9)])
        outs.append((pvo.correlate((g0, g1), (l0, l1), reproj, ctx=ctx), orc.correlate((g0, g1), (l0, l1), reproj)))
    s1 = pvo.grid_cache_stats(ctx)
    assert s1["misses"] - s0["misses"] == 2 and s1["hits"] - s0["hits"] == 10
    # the same array modified in place (different content) is uploaded again
    l0[...] = smooth_features(rng, 30, 40, C)
    reproj = np.column_stack([rng.uniform(0, 160, 9), rng.uniform(0, 120, 9)])
    got = pvo.correlate((g0, g1), (l0, l1), reproj, ctx=ctx)
    assert pvo.grid_cache_stats(ctx)["misses"] - s1["misses"] == 1
    outs.append((got, orc.correlate((g0, g1), (l0, l1), reproj)))
    for got, ref in outs:
        gn = np.stack([np.linalg.norm(g0, axis=1), np.linalg.norm(g1, axis=1)]).reshape(2, 3, 3, 1, 1)
        assert np.all(np.abs(got.astype(np.float64) - ref) <= 1e-4 * np.maximum(np.abs(ref), 1e-3 * gn))
