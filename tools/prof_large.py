"""Phase clocks of the large-window solver (config 4 by default)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
w, prob, ctx, stream, win = bench.setup(cfg, seed=0, device=0)
ctx.set_tracing(True)
with torch.cuda.stream(stream):
    for _ in range(3):
        win.reset()
        win.iteration(1)
torch.cuda.synchronize()
print("corr/ba ms", ctx.last_timing())
c = ctx.ba_phase_cycles()[14]
print({"permute": int(c[1] - c[0]), "diag": int(c[2]), "panel": int(c[3]), "trailing": int(c[4]),
       "backsub": int(c[6] - c[5]), "retract": int(c[7] - c[6]), "total": int(c[7] - c[0])})
