"""Guard/structure-only problem (wild targets): small vs large path vs oracle."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle.pyoracle as orc  # noqa: E402
import paper_2208_04726_b200 as pvo  # noqa: E402
from paper_2208_04726_b200 import synth  # noqa: E402

ctx = pvo.Context(0)
for name, fr, pa, noise in [("c1", None, None, 300), ("c4", 24, 12, 300), ("c4", 24, 12, 30)]:
    w = synth.generate(name, features=False, frames=fr, patches=pa)
    g = synth.build_graph(w, pvo.PatchGraph)
    prob = g.window_problem(w.cfg["window"])
    prob["e_target"] = prob["e_target"] + np.random.default_rng(1).normal(0, noise, prob["e_target"].shape)
    ref = orc.ba_window(prob, w.K, iterations=2, structure_only=1)
    pr = pvo.BAProblem(prob["poses"], prob["fixed"].astype(bool), prob["patch_src"], prob["patch_x"],
                       prob["patch_y"], prob["depth"], prob["e_patch"], prob["e_pose"], prob["e_target"],
                       prob["e_weight"], w.K)
    sol = pvo.ba_window(pr, iterations=2, structure_only_iterations=1, ctx=ctx)
    print(name, fr, pa, noise, "large" if os.environ.get("PVO_BA_LARGE") else "small", "norms gpu", np.round(sol.residual_norms, 6),
          "ref", np.round(ref["residual_norms"], 6), "dpose", np.abs(sol.poses - ref["poses"]).max())
