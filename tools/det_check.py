import sys; sys.path.insert(0, '.')
import numpy as np
import paper_2208_04726_b200 as pvo
from paper_2208_04726_b200 import synth
w = synth.generate("c1")
ctx = pvo.Context(0)
F = w.cfg["frames"]
ctx.frames_reserve(F, w.level0.shape[2], w.level0.shape[1], w.level1.shape[2], w.level1.shape[1], 128)
for f in range(F): ctx.frames_upload(f, w.level0[f], w.level1[f])
g = synth.build_graph(w, pvo.PatchGraph)
prob = synth.window_arrays(w, g.window_problem(w.cfg["window"]))
win = pvo.Window(ctx)
win.load(prob, prob["pose_frames"], prob["patch_feats"], w.K, w.image)
vols = []
for r in range(4):
    win.reset()
    vol = np.empty((win.n_edges, 2, 9, 7, 7), np.float32)
    win.iteration(2, corr_out=vol)
    vols.append(vol)
for r in range(1, 4):
    d = np.argwhere(vols[r] != vols[0])
    print(r, len(d), d[:5].tolist())
    if len(d):
        e, l, p = d[0][:3]
        print(vols[0][e, l, p].ravel()[:10], vols[r][e, l, p].ravel()[:10])
