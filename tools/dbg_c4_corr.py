"""Print the C4 correlation entries outside tolerance with their sampling details."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle.pyoracle as orc  # noqa: E402
import paper_2208_04726_b200 as pvo  # noqa: E402
import pvo_synth as synth  # noqa: E402
from tests.test_gpu_fullsize import _coords  # noqa: E402

ctx = pvo.Context(0)
w = synth.generate("c4")
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
rng = np.random.default_rng(404)
sel = np.sort(rng.choice(E, 20000, replace=False))
coords = _coords(prob, sel, w.K)
frames = prob["pose_frames"][prob["e_pose"][sel]]
ref = orc.correlate_batch(prob["e_patch"][sel], frames, coords, prob["patch_feats"], w.level0, w.level1,
                          threads=os.cpu_count())
gn = np.linalg.norm(prob["patch_feats"][prob["e_patch"][sel]].astype(np.float64), axis=-1)[..., None, None]
tol = 1e-4 * np.maximum(np.abs(ref), 1e-3 * gn)
got = vol[sel].astype(np.float64)
bad = np.argwhere(np.abs(got - ref) > tol)
print("violations", len(bad))
for i, lv, px, a, b in bad[:20]:
    e = sel[i]
    grid = (w.level0 if lv == 0 else w.level1)[frames[i]].astype(np.float64)
    sc = 4.0 if lv == 0 else 16.0
    x = coords[i, px, 0] / sc + (b - 3)
    y = coords[i, px, 1] / sc + (a - 3)
    x0, y0 = int(np.floor(x)), int(np.floor(y))
    ax, ay = x - x0, y - y0
    H, W, C = grid.shape
    taps = []
    for (xi, yi, wt) in [(x0, y0, (1 - ax) * (1 - ay)), (x0 + 1, y0, ax * (1 - ay)), (x0, y0 + 1, (1 - ax) * ay),
                         (x0 + 1, y0 + 1, ax * ay)]:
        f = grid[yi, xi] if 0 <= xi < W and 0 <= yi < H else np.zeros(C)
        taps.append((wt, f))
    v = sum(wt * f for wt, f in taps)
    n2 = float(v @ v)
    diag = sum(wt * wt * float(f @ f) for wt, f in taps)
    gv = prob["patch_feats"][prob["e_patch"][e], lv, px].astype(np.float64)
    print(f"edge {e} lvl {lv} px {px} a {a} b {b}: got {got[i, lv, px, a, b]:.9g} ref {ref[i, lv, px, a, b]:.9g} "
          f"diff {abs(got[i, lv, px, a, b] - ref[i, lv, px, a, b]):.3g} tol {tol[i, lv, px, a, b]:.3g} "
          f"|g| {np.linalg.norm(gv):.4g} n2 {n2:.6g} diag {diag:.6g} ratio {n2 / max(diag, 1e-300):.4g} "
          f"w {[round(t[0], 4) for t in taps]} dot {float(gv @ v):.6g}")
