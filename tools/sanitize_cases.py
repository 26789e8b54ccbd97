"""Small invocations of every device path, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck), numpy-only host side:

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Covers: gram_kernel, corr_prep_kernel + corr_tma_kernel (D = 128, with the
cancellation fallback triggered), corr_kernel (D = 25), ba_kernel (window,
guard), bal_* (large window: 20 free poses), ba_batch_kernel, the device
graph (connect / flatten / keyframe / remove), measure + oracle propose,
feature extraction + crop, the measurement's exact replay on tied slices, a
batch holding a window beyond 16 free poses, odd patch widths.  Prints
'sanitize cases ok'."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2208_04726_b200 as pvo  # noqa: E402
import pvo_synth as synth  # noqa: E402

ctx = pvo.Context(0)
# --- window: corr_tma (+ prep, gram) + ba_kernel -----------------------------
w = synth.generate("c1", seed=3, frames=6, patches=16)
F = w.cfg["frames"]
_, H0, W0, D = w.level0.shape
_, H1, W1, _ = w.level1.shape
l0 = w.level0.copy()
l0[2, :, 1::2] = -l0[2, :, 0:-1:2]  # anti-correlated neighbours in one frame: the exact fallback runs
ctx.frames_reserve(F, W0, H0, W1, H1, D)
for f in range(F):
    ctx.frames_upload(f, l0[f], w.level1[f])
g = synth.build_graph(w, pvo.PatchGraph)
prob = synth.window_arrays(w, g.window_problem(w.cfg["window"]))
win = pvo.Window(ctx)
win.load(prob, prob["pose_frames"], prob["patch_feats"], w.K, w.image)
vol = np.empty((win.n_edges, 2, 9, 7, 7), np.float32)
win.iteration(2, corr_out=vol)
win.read()
win.propose()
win.oracle_propose(w.poses[prob["pose_frames"]], w.depth[prob["patch_ids"]], 0.5, 0.05, seed=1)
win.ba(2)
win.read()
# --- generic correlation kernel (D = 25) + features ---------------------------
img = np.random.default_rng(0).random((64, 96)).astype(np.float32)
ctx.frames_reserve(2, 24, 16, 6, 4, 25)
ctx.frames_extract(0, img, base_channels=1)
ctx.frames_extract(1, img[:, ::-1].copy(), base_channels=1)
cents = np.array([[20.0, 20.0], [40.0, 30.0], [70.0, 40.0]])
feats = ctx.crop_patches(0, cents)
coords = np.stack([np.stack([c[0] + np.tile([-1.0, 0, 1], 3), c[1] + np.repeat([-1.0, 0, 1], 3)], 1) for c in cents])
pvo.correlate_batch(np.arange(3, dtype=np.int32), np.array([0, 1, 1], np.int32), coords, feats, ctx=ctx)
pvo.measure_batch(np.arange(3, dtype=np.int32), np.array([0, 1, 1], np.int32), coords[:, 4], feats, ctx=ctx)
# --- large window (> 16 free poses): the bal_* kernel chain ------------------
wl = synth.generate("c4", seed=4, frames=22, patches=24, features=False)
gl = synth.build_graph(wl, pvo.PatchGraph)
fl = gl.window_problem(22)
pr = pvo.BAProblem(fl["poses"], fl["fixed"].astype(bool), fl["patch_src"], fl["patch_x"], fl["patch_y"], fl["depth"],
                   fl["e_patch"], fl["e_pose"], fl["e_target"], fl["e_weight"], wl.K)
pvo.ba_window(pr, iterations=2, ctx=ctx)
# --- batch of windows ---------------------------------------------------------
ctx.frames_reserve(3 * F, W0, H0, W1, H1, D)
for s in range(3):
    for f in range(F):
        ctx.frames_upload(s * F + f, w.level0[f], w.level1[f])
bat = pvo.Batch(ctx)
bat.load([prob] * 3, [prob["pose_frames"] + s * F for s in range(3)], [prob["patch_feats"]] * 3, w.K, w.image)
bat.iteration(2)
bat.read()
# --- device graph: add / connect / flatten / keyframe / remove ----------------
ctx.frames_reserve(12, W0, H0, W1, H1, D)
wd = synth.generate("c1", seed=6, frames=10, patches=12)
dg = pvo.DeviceGraph(ctx, wd.K, wd.image[0], wd.image[1], channels=D)
M = wd.cfg["patches"]
for f in range(10):
    ctx.frames_upload(f, wd.level0[f], wd.level1[f])
    fi = dg.add_frame(0.1 * f, wd.poses[f], f)
    dg.add_patches(fi, wd.centroids[f * M:(f + 1) * M], wd.depth[f * M:(f + 1) * M], wd.patch_feats[f * M:(f + 1) * M])
    dg.connect(13)
    n = dg.load_window(10, all_active=True)
    if n[2]:
        win2 = pvo.Window(ctx)
        win2.propose(read_back=False)
        dg.store_window(revisions=True, state=False)
        dg.load_window(10)
        win2.ba(2)
        dg.store_window(revisions=False, state=True)
    if f >= 6:
        dg.keyframe(1e9)
# --- provider measurement on exact ties (stripes): the exact replay kernel runs --
Hs, Ws, Ds = 30, 40, 128
rng = np.random.default_rng(9)
row = rng.standard_normal((Hs, 1, Ds))
row /= np.linalg.norm(row, axis=-1, keepdims=True)
stripes = (row * np.where(np.arange(Ws) % 2 == 0, 1.0, -1.0)[None, :, None]).astype(np.float32)
l1s = stripes[: Hs // 4 + 1, : Ws // 4].copy()
ctx.frames_reserve(1, Ws, Hs, Ws // 4, Hs // 4 + 1, Ds)
ctx.frames_upload(0, stripes, l1s)
ns = 24
cs = np.stack([rng.uniform(8, 4 * Ws - 8, ns), rng.uniform(8, 4 * Hs - 8, ns)], 1)
fs = rng.standard_normal((ns, 2, 9, Ds)).astype(np.float32)
pvo.measure_batch(np.arange(ns, dtype=np.int32), np.zeros(ns, np.int32), cs, fs, ctx=ctx)
assert ctx.measure_replayed > 0
# --- batch with a window beyond 16 free poses (batched kernel + bal_* chain) ---
wb = synth.generate("c1", seed=8, frames=22, patches=8)
ctx.frames_reserve(22 + F, W0, H0, W1, H1, D)
for f in range(22):
    ctx.frames_upload(f, wb.level0[f], wb.level1[f])
for f in range(F):
    ctx.frames_upload(22 + f, w.level0[f], w.level1[f])
pbig = synth.window_arrays(wb, synth.build_graph(wb, pvo.PatchGraph).window_problem(20))
bat2 = pvo.Batch(ctx)
bat2.load([pbig, prob], [pbig["pose_frames"], prob["pose_frames"] + 22], [pbig["patch_feats"], prob["patch_feats"]],
          w.K, w.image)
bat2.iteration(2)
bat2.read()
# --- odd patch widths through the 3x3 stand-in ----------------------------------
g5 = synth.build_graph(synth.generate("c1", seed=10, frames=6, patches=8, features=False), pvo.PatchGraph,
                       patch_width=5)
pvo.optimize_window(g5, pvo.WindowOptions(window=6), ctx=ctx)
ctx.synchronize()
ctx.close()
print("sanitize cases ok")
