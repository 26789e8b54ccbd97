"""Near-tie reasons of the Gram-form measurement on a config's window.

Run with a variant library built with -DPVO_MEASURE_TIE_STATS
(tools/build_variant.sh ties -DPVO_MEASURE_TIE_STATS; PVO_LIB=tools/lib_ties.so):
there a flagged edge's flags byte is 128 | reasons and the exact replay is not
launched.  Prints the per-reason counts."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
w, prob, ctx, stream, win = bench.setup(cfg, seed=0, device=0)
d, wt, fl = win.propose(read_back=True)
fl = np.asarray(fl)
tied = fl >= 128
names = ["argmax", "flat", "denom", "step", "climb", "dist"]
print(f"{cfg}: {fl.size} edges, {int(tied.sum())} flagged")
for b, n in enumerate(names):
    print(f"  {n:7s} {int(((fl & (1 << b)) != 0)[tied].sum())}")
