"""Correlation accuracy margin against the reference on C2 (every edge) and a
C4 sample: max |gpu - ref| / tol and tail counts (tol = 1e-4 max(|ref|, 1e-3 |g|)).
usage: [PVO_LIB=tools/lib_X.so] python tools/corr_accuracy.py [c4_sample]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle.pyoracle as orc  # noqa: E402
import paper_2208_04726_b200 as pvo  # noqa: E402
import pvo_synth as synth  # noqa: E402
from tests.test_gpu_fullsize import _coords  # noqa: E402

ctx = pvo.Context(0)
n4 = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
for cfg, nsel in (("c2", None), ("c4", n4)):
    w = synth.generate(cfg)
    F = w.cfg["frames"]
    ctx.frames_reserve(F, w.level0.shape[2], w.level0.shape[1], w.level1.shape[2], w.level1.shape[1], 128)
    for f in range(F):
        ctx.frames_upload(f, w.level0[f], w.level1[f])
    g = synth.build_graph(w, pvo.PatchGraph)
    prob = synth.window_arrays(w, g.window_problem(w.cfg["window"]))
    win = pvo.Window(ctx)
    win.load(prob, prob["pose_frames"], prob["patch_feats"], w.K, w.image)
    E = win.n_edges
    vol = win.correlate()
    sel = np.arange(E) if nsel is None else np.sort(np.random.default_rng(404).choice(E, nsel, replace=False))
    coords = _coords(prob, sel, w.K)
    frames = prob["pose_frames"][prob["e_pose"][sel]]
    ref = orc.correlate_batch(prob["e_patch"][sel], frames, coords, prob["patch_feats"], w.level0, w.level1,
                              threads=os.cpu_count())
    gn = np.linalg.norm(prob["patch_feats"][prob["e_patch"][sel]].astype(np.float64), axis=-1)[..., None, None]
    tol = 1e-4 * np.maximum(np.abs(ref), 1e-3 * gn)
    r = np.abs(vol[sel].astype(np.float64) - ref) / tol
    print(f"{cfg}: {len(sel)} edges, {r.size} outputs: max err/tol {r.max():.3f}, >1: {(r > 1).sum()}, "
          f">0.5: {(r > 0.5).sum()}, >0.25: {(r > 0.25).sum()}, mean {r.mean():.4f}", flush=True)
    win.close() if hasattr(win, "close") else None
