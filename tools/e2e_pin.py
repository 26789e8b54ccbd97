import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench
w, prob, ctx, stream, win = bench.setup("c2", seed=0, device=0)
def pin(a):
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    return t.numpy()
keys = ["poses", "fixed", "pose_frames", "patch_src", "patch_x", "patch_y", "depth", "patch_feats", "e_patch", "e_pose", "e_delta", "e_weight"]
pp = dict(prob)
for k in keys:
    pp[k] = pin(prob[k])
for name, pr in [("pageable", prob), ("pinned", pp)]:
    for it in range(3):
        win.load(pr, pr["pose_frames"], pr["patch_feats"], w.K, w.image)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for it in range(20):
        win.load(pr, pr["pose_frames"], pr["patch_feats"], w.K, w.image)
    print(name, "load ms", (time.perf_counter() - t) / 20 * 1e3)
# host-only part: validate/plan through the oracle-free path is inside load; time a zero-feature variant
pz = dict(pp); pz["patch_feats"] = pin(np.zeros((1, 2, 9, 128), np.float32))
