"""Run optimize_window(2) on a config's window with the library PVO_LIB points at and
save the poses / depths / residual norms (bit-identity checks between solver variants).
usage: PVO_LIB=tools/lib_<V>.so python tools/ba_dump.py <cfg> <out.npz>"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

cfg, out = sys.argv[1], sys.argv[2]
w, prob, ctx, stream, win = bench.setup(cfg, seed=0, device=0)
with torch.cuda.stream(stream):
    win.reset()
    win.iteration(2)
torch.cuda.synchronize()
poses, d, norms = win.read()
np.savez(out, poses=poses, depth=d, norms=np.asarray(norms))
print(cfg, "norms", norms)
