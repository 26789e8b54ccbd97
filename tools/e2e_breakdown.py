"""Host-timed breakdown of one e2e step (bench.run_e2e) on config 2."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

w, prob, ctx, stream, win = bench.setup("c2", seed=0, device=0)
E = win.n_edges
F = w.cfg["frames"]
l0 = torch.from_numpy(w.level0[-1]).pin_memory()
l1 = torch.from_numpy(w.level1[-1]).pin_memory()
vol = torch.empty((E, 2, 9, 7, 7), dtype=torch.float32).pin_memory()
vol_np = vol.numpy()
acc = np.zeros(5)
for it in range(25):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.frames_upload(F - 1, l0.numpy(), l1.numpy())
    ctx.synchronize()
    t1 = time.perf_counter()
    win.load(prob, prob["pose_frames"], prob["patch_feats"], w.K, w.image)
    t2 = time.perf_counter()
    win.iteration(2)
    ctx.synchronize()
    t3 = time.perf_counter()
    win.correlate  # noqa: B018
    ok = win.corr_device_ptr()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    win.iteration(2, corr_out=vol_np)
    win.read()
    t5 = time.perf_counter()
    if it >= 5:
        acc += [t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4]
acc /= 20
print("ms: frame H2D %.3f | window load %.3f | iteration (device only) %.3f | - %.3f | iteration + vol D2H + read %.3f"
      % tuple(acc * 1e3))
