"""Deterministic inputs of the golden regression fixtures (tests/golden/golden_v1.npz).

The reference cannot be built in this image (Eigen3 absent) and
ships no golden vectors, so these fixtures hold the CPU restatement's outputs
(oracle/pvo_oracle.cpp, itself pinned by the reference's known-answer tests in
tests/test_oracle_pins.py) on small seeded inputs.  They freeze the oracle
(CPU suite: regenerating must reproduce them bit for bit) and let the GPU suite
check the product path against fixed numbers without the oracle in the loop.
Inputs are rebuilt from seeds here (numpy PCG64 streams are stable); their
SHA-256 is stored next to the outputs to catch any drift.
"""
from __future__ import annotations

import hashlib

import numpy as np

import pvo_synth as synth


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def corr_case():
    """2 frames of 16 x 20 level-0 cells (80 x 64 px), 128-d; 12 patches, 24 edges
    (every patch onto both frames) with reprojections displaced around the centroid,
    two of them far outside the frame (zero tiles), one straddling the border."""
    rng = np.random.default_rng(20261017)
    F, H0, W0, D = 2, 16, 20, 128
    level0 = synth.make_level0(rng, F, H0, W0, D)
    level1 = synth.make_level1(level0)
    n = 12
    cx = rng.uniform(6.0, 4 * W0 - 7.0, n)
    cy = rng.uniform(6.0, 4 * H0 - 7.0, n)
    offs = np.array([-1.0, 0.0, 1.0])
    px = (cx[:, None] + np.tile(offs, 3)[None]).reshape(n, 9)
    py = (cy[:, None] + np.repeat(offs, 3)[None]).reshape(n, 9)
    src = rng.integers(0, F, n)
    feats = np.empty((n, 2, 9, D), np.float32)
    for k in range(n):
        feats[k, 0] = synth.crop_cubic(level0[src[k]], px[k] / 4.0, py[k] / 4.0)
        feats[k, 1] = synth.crop_cubic(level1[src[k]], px[k] / 16.0, py[k] / 16.0)
    e_patch = np.repeat(np.arange(n, dtype=np.int32), 2)
    e_frame = np.tile(np.arange(F, dtype=np.int32), n)
    E = len(e_patch)
    shift = rng.normal(0.0, 3.0, (E, 1, 2))
    scale = 1.0 + rng.normal(0.0, 0.1, (E, 1, 1))
    base = np.stack([px[e_patch], py[e_patch]], -1)  # [E, 9, 2]
    centre = base[:, 4:5, :]
    coords = centre + (base - centre) * scale + shift
    coords[3] += 500.0  # far outside: every tap is zero padding
    coords[10] -= 300.0
    coords[7, :, 0] = -2.0 + (coords[7, :, 0] - coords[7, 4, 0])  # straddles the left border
    return dict(level0=level0, level1=level1, feats=feats, e_patch=e_patch, e_frame=e_frame, coords=coords)


def ba_case():
    """A 4-frame, 8-patch-per-frame window (graph radius 13, window 10): the
    flattened optimize_window problem with frozen targets."""
    import oracle.pyoracle as orc

    w = synth.generate("c1", seed=77, features=False, frames=4, patches=8)
    g = synth.build_graph(w, orc.PatchGraph)
    return w, g.window_problem(w.cfg["window"])


def features_case():
    """A smooth 64 x 96 image (base channels 1): pyramid + 5 patch crops."""
    rng = np.random.default_rng(424242)
    ih, iw = 64, 96
    yy, xx = np.mgrid[0:ih, 0:iw].astype(np.float64)
    img = np.zeros((ih, iw))
    for _ in range(6):
        fx, fy, ph = rng.uniform(0.02, 0.2), rng.uniform(0.02, 0.2), rng.uniform(0, 6.28)
        img += rng.uniform(0.2, 1.0) * np.sin(fx * xx + fy * yy + ph)
    img += 0.05 * rng.standard_normal((ih, iw))
    cents = np.stack([rng.uniform(5, iw - 6, 5), rng.uniform(5, ih - 6, 5)], 1)
    offs = np.array([-1.0, 0.0, 1.0])
    px = (cents[:, :1] + np.tile(offs, 3)[None]).reshape(-1, 9)
    py = (cents[:, 1:] + np.repeat(offs, 3)[None]).reshape(-1, 9)
    return dict(image=img.astype(np.float32), cents=cents, px=px, py=py)
