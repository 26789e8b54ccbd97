"""Per-patch / per-pose differences after one guarded GN step (wild-target window)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle.pyoracle as orc  # noqa: E402
import paper_2208_04726_b200 as pvo  # noqa: E402
from paper_2208_04726_b200 import synth  # noqa: E402

ctx = pvo.Context(0)
w = synth.generate("c4", features=False, frames=24, patches=12)
g = synth.build_graph(w, pvo.PatchGraph)
prob = g.window_problem(w.cfg["window"])
prob["e_target"] = prob["e_target"] + np.random.default_rng(1).normal(0, 300, prob["e_target"].shape)
for so, it in [(1, 0), (0, 1), (1, 1)]:
    ref = orc.ba_window(prob, w.K, iterations=it, structure_only=so)
    pr = pvo.BAProblem(prob["poses"], prob["fixed"].astype(bool), prob["patch_src"], prob["patch_x"],
                       prob["patch_y"], prob["depth"], prob["e_patch"], prob["e_pose"], prob["e_target"],
                       prob["e_weight"], w.K)
    sol = pvo.ba_window(pr, iterations=it, structure_only_iterations=so, ctx=ctx)
    dd = np.abs(sol.inverse_depths - ref["depth"])
    top = np.argsort(-dd)[:6]
    print("so", so, "it", it, "norms", sol.residual_norms, ref["residual_norms"])
    print("  dpose", np.abs(sol.poses - ref["poses"]).max(), "depth diffs", dd[top], "gpu", sol.inverse_depths[top],
          "ref", ref["depth"][top], "zeros gpu/ref", int((sol.inverse_depths == 0).sum()), int((ref["depth"] == 0).sum()))

# GN from the post-structure state as a fresh problem
mid = orc.ba_window(prob, w.K, iterations=0, structure_only=1)
prob2 = dict(prob)
prob2["depth"] = mid["depth"].copy()
ref = orc.ba_window(prob2, w.K, iterations=1)
pr = pvo.BAProblem(prob2["poses"], prob2["fixed"].astype(bool), prob2["patch_src"], prob2["patch_x"],
                   prob2["patch_y"], prob2["depth"], prob2["e_patch"], prob2["e_pose"], prob2["e_target"],
                   prob2["e_weight"], w.K)
sol = pvo.ba_window(pr, iterations=1, ctx=ctx)
print("fresh GN from post-structure state: norms", sol.residual_norms, ref["residual_norms"], "dpose",
      np.abs(sol.poses - ref["poses"]).max())
