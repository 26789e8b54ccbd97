"""Per-frame DPVO update entirely on the device (SURVEY.md §8f rows 1 + 3):
new frame pyramid -> device graph (add frame / patches, connect) -> on-device
window flatten -> propose (flow-provider measurement at the current state) ->
revisions into the graph -> optimize_window (2 GN iterations) -> write-back.

usage: python tools/pipeline_loop.py [frames=30] [config=c2] [images]
Prints the mean per-frame device time of each stage over the second half of
the sequence (CUDA events on the context stream) and the host wall time.
With "images" the frames arrive as 480x640 images and the reference's own
extractor runs on the device (features.cu: 25-d descriptors, patches cropped
from the new pyramid) — image in, poses out, only the image crossing PCIe."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2208_04726_b200 as pvo  # noqa: E402
import pvo_synth as synth  # noqa: E402

n_frames = int(sys.argv[1]) if len(sys.argv) > 1 else 30
cfg = sys.argv[2] if len(sys.argv) > 2 else "c2"
images = len(sys.argv) > 3 and sys.argv[3] == "images"
w = synth.generate(cfg, seed=5, frames=n_frames, features=not images)
F, M = w.cfg["frames"], w.cfg["patches"]
if images:  # smooth random images; the device extracts the 25-d reference pyramid
    rng = np.random.default_rng(1)
    from tests.test_oracle_pins import _smooth_image

    imgs = [torch.from_numpy(_smooth_image(rng, w.image[1], w.image[0])).pin_memory() for _ in range(F)]
    W0, H0, W1, H1, D = w.image[0] // 4, w.image[1] // 4, w.image[0] // 16, w.image[1] // 16, 25
else:
    _, H0, W0, D = w.level0.shape
    _, H1, W1, _ = w.level1.shape
ctx = pvo.Context(0)
stream = torch.cuda.Stream()
ctx.set_stream(stream.cuda_stream)
NS = 32  # frame-store ring: the window plus every frame its edges still reach
ctx.frames_reserve(NS, W0, H0, W1, H1, D)
dev = pvo.DeviceGraph(ctx, w.K, w.image[0], w.image[1], channels=D)
if "--no-reserve" not in sys.argv:  # size the graph once: no allocation inside a frame
    dev.reserve(patches=F * M, edges=F * M * (2 * w.cfg["radius"] + 1), frames=F)
if not images:
    l0 = [torch.from_numpy(w.level0[f]).pin_memory() for f in range(F)]
    l1 = [torch.from_numpy(w.level1[f]).pin_memory() for f in range(F)]
stages = ["frame (H2D/extract+Gram)", "graph add + connect", "flatten", "propose", "BA (2 it.)", "store"]
acc = {s: [] for s in stages}
walls, edges, attempts, host_ms = [], [], [], []
with torch.cuda.stream(stream):
    for f in range(F):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(stages) + 1)]
        if "--spikes" in sys.argv:
            print(f"[frame {f}]", file=sys.stderr, flush=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev[0].record(stream)
        ks = slice(f * M, (f + 1) * M)
        if images:
            ctx.frames_extract(f % NS, imgs[f].numpy(), base_channels=1)
            feats = ctx.crop_patches(f % NS, w.centroids[ks])
        else:
            ctx.frames_upload(f % NS, l0[f].numpy(), l1[f].numpy())
            feats = w.patch_feats[ks]
        ev[1].record(stream)
        th = [time.perf_counter()]
        idx = dev.add_frame(0.05 * (f + 1), w.poses[f], frame_slot=f % NS)
        dev.add_patches(idx, w.centroids[ks], w.depth[ks], feats)
        dev.connect(w.cfg["radius"])
        th.append(time.perf_counter())
        ev[2].record(stream)
        # every active edge (pipeline.cpp:164-181); after propose all of them are revised,
        # so this window is also optimize_window's problem (bundle_adjust.cpp:245)
        n = dev.load_window(w.cfg["window"], all_active=True)
        th.append(time.perf_counter())
        ev[3].record(stream)
        dev.window.propose(read_back=False)
        ev[4].record(stream)
        dev.window.ba(2)
        ev[5].record(stream)
        dev.store_window(revisions=True, state=True)
        ev[6].record(stream)
        ev[6].synchronize()
        walls.append(time.perf_counter() - t0)
        edges.append(n[2])
        attempts.append(ctx.ba_attempts)  # GN attempts of this frame's BA (guard retries included)
        host_ms.append((1e3 * (th[1] - th[0]), 1e3 * (th[2] - th[1])))
        if f >= F // 2:
            for i, s in enumerate(stages):
                acc[s].append(ev[i].elapsed_time(ev[i + 1]))
print(f"{cfg}{' (images, 25-d device features)' if images else ''}: {F} frames, {M} patches/frame, "
      f"window {w.cfg['window']}, radius {w.cfg['radius']}; "
      f"active edges at the end {edges[-1]}")
# mean and median per stage: graph admission and flatten read small counts back
# (new edge count to size the next pass, window sizes), so their event-timed
# stages include host scheduling latency, which a shared host makes spiky
tot, totm = 0.0, 0.0
for s in stages:
    m, md = float(np.mean(acc[s])), float(np.median(acc[s]))
    tot += m
    totm += md
    print(f"  {s:22s} {m:8.3f} ms   (median {md:.3f}, max {float(np.max(acc[s])):.3f})")
print(f"  divergence guard: {sum(attempts) - 2 * len(attempts)} retries over {2 * len(attempts)} GN iterations")
print(f"  {'device total':22s} {tot:8.3f} ms   (median {totm:.3f})   host wall per frame "
      f"{1e3 * np.mean(walls[F // 2:]):.3f} ms")
if "--spikes" in sys.argv:  # frames whose graph stages took > 3x the median (device events + host wall)
    half = F // 2
    for s_i, s in ((0, stages[1]), (1, stages[2])):
        med = float(np.median(acc[s]))
        for j, v in enumerate(acc[s]):
            if v > 3 * med:
                print(f"  spike: frame {half + j} {s}: {v:.3f} ms device-event span, "
                      f"{host_ms[half + j][s_i]:.3f} ms host wall in the calls")
