"""Debug driver: correlate_batch on the first N edges of C1 against the oracle.

python tools/dbg_corr.py [N]  (run under compute-sanitizer to localise faults)
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle.pyoracle as orc  # noqa: E402
from paper_2208_04726_b200 import api as pvo, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
w = synth.generate("c1")
ctx = pvo.Context()
F = w.cfg["frames"]
ctx.frames_reserve(F, w.level0.shape[2], w.level0.shape[1], w.level1.shape[2], w.level1.shape[1], 128)
for f in range(F):
    ctx.frames_upload(f, w.level0[f], w.level1[f])
g = synth.build_graph(w, pvo.PatchGraph)
prob = g.window_problem(w.cfg["window"])
E = min(n, len(prob["e_patch"]))
coords = np.empty((E, 9, 2))
for e in range(E):
    k = prob["e_patch"][e]
    coords[e], _ = orc.reproject_patch(prob["poses"][prob["patch_src"][k]], prob["poses"][prob["e_pose"][e]], w.K,
                                       prob["patch_x"][k], prob["patch_y"][k], prob["depth"][k])
pf = w.patch_feats[prob["patch_ids"]]
slots = prob["pose_frames"][prob["e_pose"][:E]]
ep = prob["e_patch"][:E]
out = pvo.correlate_batch(ep, slots, coords, pf, ctx=ctx)
ref = orc.correlate_batch(ep, slots, coords, pf, w.level0, w.level1, threads=8)
err = np.abs(out.astype(np.float64) - ref)
print("edges", E, "max abs err", err.max(), "argmax", np.unravel_index(err.argmax(), err.shape))
gn = np.linalg.norm(pf[ep].astype(np.float64), axis=-1)[..., None, None]
tol = 1e-4 * np.maximum(np.abs(ref), 1e-3 * gn)
viol = np.argwhere(err > tol)
print("violations", len(viol))
for v in viol[:10]:
    v = tuple(v)
    print(v, "gpu", out[v], "ref", ref[v], "tol", tol[v], "gnorm", gn[v[0], v[1], v[2], 0, 0],
          "coords", coords[v[0], v[2]], "slot", slots[v[0]])
