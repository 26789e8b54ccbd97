"""Host-timed breakdown of one e2e step (bench.run_e2e's calls, pinned host buffers) on config 2."""
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
hp = dict(prob)
for k in ("poses", "fixed", "pose_frames", "patch_src", "patch_x", "patch_y", "depth", "patch_feats", "e_patch",
          "e_pose", "e_delta", "e_weight"):
    hp[k] = torch.from_numpy(np.ascontiguousarray(prob[k])).pin_memory().numpy()
names = ["frames_upload", "window load", "iteration + volume D2H", "read"]
acc = np.zeros(len(names))
n = 40
for it in range(n + 5):
    t = [time.perf_counter()]
    ctx.frames_upload(F - 1, l0.numpy(), l1.numpy())
    ctx.synchronize()
    t.append(time.perf_counter())
    win.load(hp, hp["pose_frames"], hp["patch_feats"], w.K, w.image)
    t.append(time.perf_counter())
    win.iteration(2, corr_out=vol_np)
    ctx.synchronize()
    t.append(time.perf_counter())
    win.read()
    t.append(time.perf_counter())
    if it >= 5:
        acc += np.diff(t)
acc /= n
print(" | ".join(f"{a}: {b * 1e3:.3f} ms" for a, b in zip(names, acc)), f"| total {acc.sum() * 1e3:.3f} ms")
