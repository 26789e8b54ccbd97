"""Large-window BA path vs the oracle (and vs the single-kernel path) at 1 and 2
iterations; set PVO_BA_LARGE=1 to force the large path on small configs."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle.pyoracle as orc  # noqa: E402
import paper_2208_04726_b200 as pvo  # noqa: E402
from paper_2208_04726_b200 import synth  # noqa: E402

ctx = pvo.Context(0)
for name, fr, pa in [("c1", None, None), ("c4", 24, 16)]:
    w = synth.generate(name, features=False, frames=fr, patches=pa)
    g = synth.build_graph(w, pvo.PatchGraph)
    prob = g.window_problem(w.cfg["window"])
    pr = pvo.BAProblem(prob["poses"], prob["fixed"].astype(bool), prob["patch_src"], prob["patch_x"],
                       prob["patch_y"], prob["depth"], prob["e_patch"], prob["e_pose"], prob["e_target"],
                       prob["e_weight"], w.K)
    for it in (1, 2):
        ref = orc.ba_window(prob, w.K, iterations=it)
        sol = pvo.ba_window(pr, iterations=it, ctx=ctx)
        dp = np.abs(sol.poses - ref["poses"]).max()
        dd = np.abs(sol.inverse_depths - ref["depth"]).max()
        print(name, fr, pa, "it", it, "large" if os.environ.get("PVO_BA_LARGE") else "", "dpose", dp, "ddepth", dd,
              "norms", sol.residual_norms, ref["residual_norms"])
