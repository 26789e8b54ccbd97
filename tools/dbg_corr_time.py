"""Correlation time + fallback count on the c2 window (PVO_LIB selects a build)."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import bench

w, prob, ctx, stream, win = bench.setup("c2", 0, 0)
E = win.n_edges
vol = torch.empty((E, 2, 9, 7, 7), dtype=torch.float32, device="cuda")
ts = []
with torch.cuda.stream(stream):
    for i in range(30):
        win.reset()
        win.iteration(2, corr_device_ptr=vol.data_ptr())
        torch.cuda.synchronize()
        ts.append(ctx.last_timing())
v = vol.cpu().numpy()
print(os.environ.get("PVO_LIB", "default"), "corr ms", np.median([t[0] for t in ts[5:]]), "ba ms",
      np.median([t[1] for t in ts[5:]]), "nan", int(np.isnan(v).sum()))
