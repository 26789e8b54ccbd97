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
ctx.set_tracing(True)
with torch.cuda.stream(stream):
    win.reset()
    win.iteration(1)
torch.cuda.synchronize()
c = ctx.ba_phase_cycles()
names = ["assemble", "sync1", "reduce", "sync2", "solve+retract", "update", "sync3"]
for att in range(4):
    row = c[att]
    if row[0] == 0:
        break
    print("attempt", att, {n: int(row[i + 1] - row[i]) for i, n in enumerate(names)})
print("assemble: records", int(c[15][0] - c[0][0]), "accumulate", int(c[15][1] - c[15][0]), "(last attempt's records vs first start; rerun with 1 iteration for exact)")
print("first attempt: solve", int(c[15][2] - c[0][4]), "retract+mats", int(c[0][5] - c[15][2]))
