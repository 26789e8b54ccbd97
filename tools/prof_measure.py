"""Run the resident window's propose() (flow-provider measurement) a few times (for ncu)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w, prob, ctx, stream, win = bench.setup(cfg, seed=0, device=0)
with torch.cuda.stream(stream):
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        win.propose(read_back=False)
        e1.record(stream)
        e1.synchronize()
        print("propose ms", e0.elapsed_time(e1))
