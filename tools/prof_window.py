"""Run a few resident-window iterations (for ncu / nsys-less profiling)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w, prob, ctx, stream, win = bench.setup(cfg, seed=0, device=0)
with torch.cuda.stream(stream):
    for _ in range(n):
        win.reset()
        ctx.frames_refresh(w.cfg["frames"] - 1)
        win.iteration(2)
torch.cuda.synchronize()
print("corr/ba ms", ctx.last_timing())
print("attempts", ctx.ba_attempts)
