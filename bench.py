#!/usr/bin/env python
"""Benchmark: one DPVO corr+BA iteration (the per-frame hot path) per step.

Default workload = BASELINE config 2, the DPVO default window (96 patches /
frame, W = 10, r = 13, 22-frame span, 480x640, 128-d features): 16,800 edges.
A step is: Gram terms of the newest frame, correlation of every active edge
(coordinates reprojected on the device) and optimize_window's 2 Gauss-Newton
iterations (frozen targets, Schur, LDLT, retraction, divergence guard), all on
device-resident inputs.  With --gpus N (torchrun) each rank runs its own
independent sequence (weak scaling, no collective in the loop; a final NCCL
gather of poses and stats after the timed region).

Metric: corr+BA edge-iterations/s = E / t_step (whole job: sum over ranks of E
divided by the max-over-ranks step time).

--impl reference times the reference's own CPU implementation of the path on
the host cores: its sources compiled unmodified into oracle/_ref by
oracle/ref_build.py (the restatement oracle/pvo_oracle.cpp only if that build
is absent), every edge of the window per step, reproject_patch + correlate
split over all host threads and the reference's single-threaded
optimize_window.  Without torchrun, --gpus N > 1 relaunches itself under
torch.distributed.run (one rank per GPU, 127.0.0.1 rendezvous).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "corr+BA edge-iterations/sec and ms/iteration at DPVO default window; % roofline"


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled every 5 ms (NVML) during the timed
    region; nvidia-smi -lms 50 when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.stop_ev = threading.Event()
        self.thread = None
        self.proc = None
        self.path = None

    def _nvml_loop(self, nv, h):
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((float(sm), int(r)))
            except Exception:
                pass
            self.stop_ev.wait(0.005)

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.device]) if vis else self.device
            h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={fields}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def stop(self):
        if self.thread is not None:
            self.stop_ev.set()
            self.thread.join()
            if not self.rows:
                return None
            reasons = sorted({n for _, r in self.rows for n, bit in self.REASONS.items() if r & bit})
            return {"sm_mhz": statistics.median(sm for sm, _ in self.rows), "sm_max_mhz": self.max_mhz,
                    "reasons": reasons, "samples": len(self.rows), "source": "nvml 5 ms"}
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6 and parts[0].replace(".", "").isdigit():
                rows.append(parts)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() in ("active", "1")})
        sm = [float(r[0]) for r in rows]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows), "source": "nvidia-smi 50 ms"}


# ---------------------------------------------------------------- workload
def corr_bytes_per_edge(prob, K, level_shapes, D=128, with_fma=False):
    """Algorithmic bytes of the correlation per edge: for each
    level the union of in-bounds integer cells touched by the 3x3x7x7 bilinear
    taps x D x 4 B, + 2 x 9 x D x 4 B of patch features + 3,528 B of output.
    with_fma: also the algorithmic contraction, sum over (edge, level, pixel) of
    (in-grid cells of the pixel's 8x8 tap window) x D FMAs — the dot products
    every bilinear tap is a weighted sum of (DESIGN.md §3 K2)."""
    import oracle.pyoracle as orc  # noqa: F401  (not used: coords come from the numpy generator)
    import pvo_synth as synth

    E = len(prob["e_patch"])
    total = 0.0
    poses, src = prob["poses"], prob["patch_src"]
    per = np.empty(E)
    fma = [0]
    rel_cache = {}
    for e in range(E):
        k = prob["e_patch"][e]
        i, j = int(src[k]), int(prob["e_pose"][e])
        px, py, d = prob["patch_x"][k], prob["patch_y"][k], prob["depth"][k]
        if np.array_equal(poses[i], poses[j]):
            u, v = px, py
        else:
            if (i, j) not in rel_cache:
                rel = synth.compose(poses[j], synth.inverse(poses[i]))
                rel_cache[(i, j)] = (synth._rotmat(rel[:4]), rel[4:])
            R, t = rel_cache[(i, j)]
            ray = np.stack([(px - K[2]) / K[0], (py - K[3]) / K[1], np.ones(9)])
            q = R @ ray + (t * d)[:, None]
            z = np.maximum(q[2], 1e-6)
            u, v = K[0] * q[0] / z + K[2], K[1] * q[1] / z + K[3]
        b = 2 * 9 * D * 4 + 3528
        for lvl, (H, W) in enumerate(level_shapes):
            s = 4.0 if lvl == 0 else 16.0
            fx, fy = np.floor(u / s).astype(int), np.floor(v / s).astype(int)
            cells = set()
            for p in range(9):
                nx = max(0, min(W, fx[p] + 5) - max(0, fx[p] - 3))
                ny = max(0, min(H, fy[p] + 5) - max(0, fy[p] - 3))
                fma[0] += nx * ny * D  # <g_p, f_cell> over the pixel's in-grid 8x8 tap cells
                for yy in range(fy[p] - 3, fy[p] + 5):
                    if 0 <= yy < H:
                        for xx in range(fx[p] - 3, fx[p] + 5):
                            if 0 <= xx < W:
                                cells.add((xx, yy))
            b += len(cells) * D * 4
        per[e] = b
        total += b
    if with_fma:
        return total, per, fma[0]
    return total, per


def fp32_roofline(total_fma, corr_ms, clk):
    """The correlation's compute roofline: algorithmic FMAs (corr_bytes_per_edge
    with_fma) x 2 FLOP over the measured prep + corr time, against the FP32 CUDA-core
    peak of the clock it ran at (148 SMs x 128 FMA/clk x 2 FLOP)."""
    mhz = (clk or {}).get("sm_max_mhz") or 1965.0
    peak = 148 * 128 * 2 * mhz * 1e6 / 1e12
    ach = 2.0 * total_fma / (corr_ms * 1e-3) / 1e12
    return {"achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
            "algorithmic_fma_per_launch": float(total_fma), "peak_kind": "148 SMs x 128 FP32 FMA/clk at sm_max_mhz"}


L2_NOTE = "GPU arm: L2 flushed between steps (256 MiB write, outside the timed events); CPU arm: n/a"


def workload_config(name: str, w, E: int, world: int) -> dict:
    """The `config` object of the JSON line, identical in both arms."""
    return {"workload": name, "desc": w.cfg["desc"], "edges_per_gpu": E, "window": w.cfg["window"],
            "radius": w.cfg["radius"], "patches_per_frame": w.cfg["patches"], "channels": 128,
            "ba_iterations": 2, "sequences": world, "parallelism": f"sequence-sharded x{world}", "l2": L2_NOTE}


def batch_config(n_seq_total: int, world: int, chunk: int, n_chunks: int, E_chunk: int, distinct: int,
                 frames: int) -> dict:
    return {"workload": "c5", "desc": "batch of independent sequences at the DPVO default window, sharded by "
            "sequence", "sequences_total": n_seq_total, "sequences_per_gpu": n_seq_total // world, "chunk": chunk,
            "chunks_per_gpu": n_chunks, "edges_per_gpu": E_chunk * n_chunks, "distinct_trajectories_per_gpu": distinct,
            "frames_per_sequence": frames, "parallelism": f"sequence-sharded x{world}",
            "l2": f"inputs ({chunk * frames * 10.4 / 1024:.1f} GB frame store per chunk) far larger than L2"}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def setup(config: str, seed: int, device: int):
    import torch

    import paper_2208_04726_b200 as pvo
    import pvo_synth as synth

    w = synth.generate(config, seed=seed)
    g = synth.build_graph(w, pvo.PatchGraph)
    prob = synth.window_arrays(w, g.window_problem(w.cfg["window"]))
    ctx = pvo.Context(device)
    stream = torch.cuda.Stream(device=device)
    ctx.set_stream(stream.cuda_stream)
    F = w.cfg["frames"]
    _, H0, W0, D = w.level0.shape
    _, H1, W1, _ = w.level1.shape
    ctx.frames_reserve(F, W0, H0, W1, H1, D)
    for f in range(F):
        ctx.frames_upload(f, w.level0[f], w.level1[f])
    win = pvo.Window(ctx)
    win.load(prob, prob["pose_frames"], prob["patch_feats"], w.K, w.image)
    ctx.synchronize()
    return w, prob, ctx, stream, win


# ---------------------------------------------------------------- reference arm
def _ref_inputs(config: str):
    import oracle.pyoracle as orc
    import pvo_synth as synth

    w = synth.generate("c2" if config == "c5" else config, seed=0)
    og = synth.build_graph(w, orc.PatchGraph)
    prob = og.window_problem(w.cfg["window"])
    pf = w.patch_feats[prob["patch_ids"]]
    frames = prob["pose_frames"][prob["e_pose"]]
    return w, og, prob, pf, frames


def _ref_step(orc, w, og, prob, pf, frames, threads, edges=None):
    """One iteration of the reference's per-frame hot path over the window:
    reproject_patch + correlate for every edge (or the given edge slice), then
    optimize_window(2 iterations).  Seconds (corr, BA), measured in C++."""
    sub = prob
    if edges is not None:
        sub = dict(prob)
        for k in ("e_patch", "e_pose", "e_target", "e_weight"):
            sub[k] = prob[k][edges]
    t_corr = orc.bench_corr(sub, w.K, frames if edges is None else frames[edges], pf, w.level0, w.level1,
                            threads=threads)
    t_ba = orc.bench_optimize_window(og, window=w.cfg["window"], iterations=2)
    return t_corr, t_ba


def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle.pyoracle as orc

    w, og, prob, pf, frames = _ref_inputs(args.config)
    E = len(prob["e_patch"])
    threads = os.cpu_count() or 1
    kind = "reference" if orc.lib_ref is not None else "port"
    # every step is the whole window unless K steps of it would not finish in a
    # few minutes: then each step takes the next contiguous slice of the edges
    # (the slices cycle through all edges) and the full BA
    probe_c, probe_b = _ref_step(orc, w, og, prob, pf, frames, threads)
    budget_s = 240.0
    n_slices = max(1, int(np.ceil((args.steps + args.warmup) * (probe_c + probe_b) / budget_s)))
    bounds = np.linspace(0, E, n_slices + 1).astype(int)
    times = []
    for i in range(args.warmup + args.steps):
        sl = i % n_slices
        edges = None if n_slices == 1 else np.arange(bounds[sl], bounds[sl + 1])
        tc, tb = _ref_step(orc, w, og, prob, pf, frames, threads, edges)
        if i >= args.warmup:
            n_e = E if edges is None else len(edges)
            times.append((tc / n_e, tb))
    per_edge_corr = float(np.mean([a for a, _ in times]))
    t_ba = float(np.mean([b for _, b in times]))
    if args.config == "c5":
        # a batch of independent sequences: one sequence per host core, so the
        # single-threaded BA of each sequence overlaps the others'
        step_s = per_edge_corr * E + t_ba / threads
        how = (f"c5 = independent c2 sequences over {threads} host threads: corr of every edge of a c2 window "
               f"split over the threads, BA time / {threads} (one sequence per core)")
    else:
        step_s = per_edge_corr * E + t_ba
        how = (f"reproject_patch + correlate over every edge of the {args.config} window on {threads} threads, "
               f"then the reference's single-threaded optimize_window(2)")
    if n_slices > 1:
        how += f"; each step one of {n_slices} contiguous edge slices (cycling through all {E} edges)"
    value = E / step_s
    if args.config == "c5":  # the GPU arm's batch layout (run_batch), for an identical config
        n_seq = args.sequences // world
        chunk = min(n_seq, args.chunk)
        cfg = batch_config(n_seq * world, world, chunk, -(-n_seq // chunk), E * chunk, min(args.distinct, chunk),
                           w.cfg["frames"])
    else:
        cfg = workload_config(args.config, w, E, world)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "edge-iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64 (f32 feature storage)", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": "edge-iterations/s", "cores": threads, "kind": kind,
                         "cpu": cpu_model(), "sample": how,
                         "build": "oracle/_ref: /root/reference/proj/src compiled unmodified, -O3 -DNDEBUG"
                         if kind == "reference" else "oracle/pvo_oracle.cpp -O3 -DNDEBUG (restatement)"},
        "e2e": {"value": value, "unit": "edge-iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "corr_ms": per_edge_corr * E * 1e3, "ba_ms": t_ba * 1e3,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(w, prob):
    """The reference's CPU path on ONE host core over the whole window (no
    extrapolation): reproject_patch + correlate for every edge, then
    optimize_window(2) on the same graph."""
    import oracle.pyoracle as orc
    import pvo_synth as synth

    og = synth.build_graph(w, orc.PatchGraph)
    frames = prob["pose_frames"][prob["e_pose"]]
    E = len(prob["e_patch"])
    t_corr = orc.bench_corr(prob, w.K, frames, prob["patch_feats"], w.level0, w.level1, threads=1)
    t_ba = orc.bench_optimize_window(og, window=w.cfg["window"], iterations=2)
    kind = "reference" if orc.lib_ref is not None else "port"
    return {"value": E / (t_corr + t_ba), "unit": "edge-iterations/s", "cores": 1, "kind": kind,
            "cpu": cpu_model(),
            "sample": f"one full iteration on 1 core: reproject_patch + correlate over all {E} edges "
                      f"({t_corr * 1e3:.0f} ms) + optimize_window(2) ({t_ba * 1e3:.0f} ms)"}


# ---------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    w, prob, ctx, stream, win = setup(args.config, seed=rank, device=local_rank)
    E = win.n_edges
    F = w.cfg["frames"]
    newest = F - 1
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local_rank}")

    def step():  # the timed work: the newest frame's Gram terms + corr + 2 GN iterations
        ctx.frames_refresh(newest)
        win.iteration(2)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            flush.zero_()
            win.reset()
            step()
    torch.cuda.synchronize()
    # the step's launches captured once into a CUDA graph and replayed per step
    # (same kernels, same arguments; the window is fixed, as within one frame of
    # the reference's loop): removes the host launch gaps between the kernels
    eager_step, graph, per_step_launches = step, None, 0
    split_step = eager_step
    if not args.no_graph:
        try:
            win.reset()
            l0 = ctx.kernel_launches
            # the timed graph carries no timing events (event nodes add device time)
            ctx.set_timing(False)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream, capture_error_mode="relaxed"):
                eager_step()
            per_step_launches = ctx.kernel_launches - l0
            ctx.set_timing(True)
            # a second capture with the library's corr | BA events, for the split pass
            split_graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(split_graph, stream=stream, capture_error_mode="relaxed"):
                eager_step()
            torch.cuda.synchronize()
            step, split_step = graph.replay, split_graph.replay
        except Exception as ex:  # capture unsupported here: time the eager launches
            print(f"bench: CUDA graph capture failed ({type(ex).__name__}: {ex}); eager steps", file=sys.stderr)
            ctx.set_timing(True)
            graph, step, split_step = None, eager_step, eager_step
            torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                flush.zero_()
                win.reset()
                step()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    launches0 = ctx.kernel_launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    t_wall = time.perf_counter()
    # the steps are enqueued back to back (no host sync inside the loop, so host
    # launch latency never idles the device inside a step); each step is timed
    # on the device by its own pair of events
    with torch.cuda.stream(stream):
        for i in range(args.steps):
            flush.zero_()  # L2 flush between steps, outside the timed events
            win.reset()  # every step starts from the same window state (harness, untimed)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    # graph replays do not pass through the library's host-side launch counter
    launches = per_step_launches * args.steps if graph is not None else ctx.kernel_launches - launches0
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    mean_ms = float(np.mean(step_ms))
    # the step's split (correlation incl. tile preparation | BA) from the library's
    # per-iteration events (captured into the graph as event nodes, so a replay
    # records them with no host launch latency inside), read back after each of a
    # few more flushed steps
    kt = []
    with torch.cuda.stream(stream):
        for i in range(min(args.steps, 50)):
            flush.zero_()
            win.reset()
            split_step()
            kt.append(ctx.last_timing())
    corr_ms = float(np.mean([k[0] for k in kt]))
    ba_ms = float(np.mean([k[1] for k in kt]))

    # the flow provider's propose() over the same window (not part of the
    # corr+BA step the metric is defined on): device ms per call
    prop_ms = []
    with torch.cuda.stream(stream):
        for i in range(6):
            win.reset()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            win.propose(read_back=False)
            e1.record(stream)
            e1.synchronize()
            if i:
                prop_ms.append(e0.elapsed_time(e1))
    prop_replayed = ctx.measure_replayed  # edges re-measured exactly (near-tie decisions)
    win.load(prob, prob["pose_frames"], prob["patch_feats"], w.K, w.image)  # restore the revisions

    # max over ranks (the job's clock)
    from paper_2208_04726_b200.dist import gather_poses, max_over_ranks

    dev = f"cuda:{local_rank}"
    mean_ms, corr_ms_max, ba_ms_max = max_over_ranks([mean_ms, corr_ms, ba_ms], device=dev).tolist()

    # e2e through the public API with host buffers (our own sequence, rank-local)
    e2e = run_e2e(args, w, prob, ctx, stream, win)
    e2e["ms"] = float(max_over_ranks([e2e["ms"]], device=dev)[0])

    # final gather of poses (the only data collective, after the timed region)
    poses, depth, norms = win.read()
    gathered = gather_poses(poses, device=dev)
    assert len(gathered) == world

    if rank != 0:
        return
    hbm, peak_kind = load_peaks()
    total_b, _, total_fma = corr_bytes_per_edge(prob, w.K, [w.level0.shape[1:3], w.level1.shape[1:3]],
                                                 with_fma=True)
    achieved = total_b / (corr_ms * 1e-3) / 1e9
    prof = ROOT / "profiles" / "corr_traffic.json"
    traffic, counters = None, None
    if prof.exists():
        pj = json.loads(prof.read_text())
        traffic = pj.get(args.config)
        counters = pj.get("counters", {}).get(args.config)
    fp32 = fp32_roofline(total_fma, corr_ms, clk)
    cpu = cpu_baseline(w, prob) if (world == 1 and not args.no_cpu) else None
    value = E * world / (mean_ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": "edge-iterations/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": mean_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 corr (f64 coords/weights), f64 BA", "data": "synthetic",
        "config": workload_config(args.config, w, E, world),
        "timing": {"state": "window state restored before every step (outside the timed events)",
                   "launch": "CUDA graph of the step's launches, replayed" if graph is not None else "eager launches"},
        "corr_ms": corr_ms_max, "ba_ms": ba_ms_max, "propose_ms": float(np.mean(prop_ms)), "propose_replayed_edges": prop_replayed,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "kernel": "corr_tma_kernel", "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": total_b, "fp32": fp32, "ncu": counters,
                     "note": "achieved = algorithmic gather bytes / (prep + corr time); the kernel is bound by FP32 "
                             "FMA issue + shared-memory wavefronts, not DRAM (see fp32 and ncu)"},
        "e2e": {"value": E * world / (e2e["ms"] * 1e-3), "unit": "edge-iterations/s",
                "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"], "ms_per_step": e2e["ms"]},
        "gpu_launches": int(launches),
        "clocks": clk,
        "wall_s_timed_region": t_wall,
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def run_batch(args, rank, world, local_rank):
    """Config 5: a batch of independent sequences at the DPVO default window,
    sharded by sequence across ranks (weak scaling, no collective in the loop).
    Each rank runs its 1024 / N sequences in chunks that fit HBM (frame store of
    a chunk = chunk x 22 frames x 10.4 MB); a step = one corr + 2-GN-iteration
    pass over all of the rank's sequences.  Inputs: `distinct` synthetic C2
    trajectories (geometry + patch descriptors) replicated over the chunk,
    frame features generated on the device per chunk (unit-norm random cells,
    distinct for every sequence), so the frames read by the correlation are
    never shared between sequences."""
    import torch

    import paper_2208_04726_b200 as pvo
    import pvo_synth as synth
    from paper_2208_04726_b200.dist import gather_poses, max_over_ranks

    torch.cuda.set_device(local_rank)
    dev = f"cuda:{local_rank}"
    n_seq = args.sequences // world
    chunk = min(n_seq, args.chunk)
    n_chunks = (n_seq + chunk - 1) // chunk
    geos = []
    for gi in range(min(args.distinct, chunk)):
        w = synth.generate("c2", seed=10_000 * rank + gi, features=False)
        g = synth.build_graph(w, pvo.PatchGraph)
        prob = synth.window_arrays(w, g.window_problem(w.cfg["window"]))
        rng = np.random.default_rng(77 + gi)
        pf = rng.standard_normal((len(prob["depth"]), 2, 9, 128)).astype(np.float32)
        pf /= np.linalg.norm(pf, axis=-1, keepdims=True)
        geos.append((w, prob, pf))
    w0 = geos[0][0]
    F = w0.cfg["frames"]
    H0, W0i = w0.image[1] // 4, w0.image[0] // 4
    H1, W1i = H0 // 4, W0i // 4
    D = 128
    ctx = pvo.Context(local_rank)
    stream = torch.cuda.Stream(device=local_rank)
    ctx.set_stream(stream.cuda_stream)
    ctx.frames_reserve(chunk * F, W0i, H0, W1i, H1, D)
    probs, slots, feats = [], [], []
    for i in range(chunk):
        _, prob, pf = geos[i % len(geos)]
        probs.append(prob)
        slots.append(prob["pose_frames"] + i * F)
        feats.append(pf)
    bat = pvo.Batch(ctx)
    bat.load(probs, slots, feats, w0.K, w0.image)
    E_chunk = bat.n_edges
    newest = [i * F + int(p["pose_frames"].max()) for i, p in enumerate(probs)]

    def fill(c):  # device-generated frame features of chunk c (untimed)
        gen = torch.Generator(device=dev)
        gen.manual_seed(1_000_003 * rank + c)
        with torch.cuda.stream(stream):
            for s0 in range(0, chunk * F, 64):
                k = min(64, chunk * F - s0)
                l0 = torch.randn((k, H0, W0i, D), device=dev, generator=gen)
                l0 /= l0.norm(dim=-1, keepdim=True)
                l1 = l0.view(k, H1, 4, W1i, 4, D).mean(dim=(2, 4))
                l1 /= l1.norm(dim=-1, keepdim=True).clamp_min(1e-12)
                l1 = l1.contiguous()
                for j in range(k):
                    ctx.frames_upload(s0 + j, l0[j], l1[j], device=True)
                del l0, l1
        torch.cuda.synchronize()

    timed_launches = [0]

    def step():  # one corr + BA pass over all of the rank's sequences: device ms
        tot = 0.0
        for c in range(n_chunks):
            fill(c)
            bat.reset()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            l0 = ctx.kernel_launches
            with torch.cuda.stream(stream):
                ev0.record(stream)
                for sl in newest:
                    ctx.frames_refresh(sl)
                bat.iteration(2)
                ev1.record(stream)
            timed_launches[0] += ctx.kernel_launches - l0
            ev1.synchronize()
            tot += ev0.elapsed_time(ev1)
        return tot

    for _ in range(args.warmup):
        step()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    timed_launches[0] = 0
    t_wall = time.perf_counter()
    ms = [step() for _ in range(args.steps)]
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    clk = clocks.stop()
    launches = timed_launches[0]
    corr_ms, ba_ms = ctx.last_timing()
    mean_ms = float(np.mean(ms))
    mean_ms = float(max_over_ranks([mean_ms], device=dev)[0])

    # e2e through the public API with host buffers: per chunk, the newest frame
    # of every sequence from pinned host memory + the iteration + poses/depths back
    frame0 = torch.randn((H0, W0i, D)).pin_memory()
    frame0 /= frame0.norm(dim=-1, keepdim=True)
    frame1 = frame0.view(H1, 4, W1i, 4, D).mean(dim=(1, 3)).contiguous().pin_memory()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n_e2e = max(1, min(args.steps, 2))
    for _ in range(n_e2e):
        for c in range(n_chunks):
            bat.reset()
            for sl in newest:
                ctx.frames_upload(sl, frame0.numpy(), frame1.numpy())
            bat.iteration(2)
            bat.read()
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) / n_e2e * 1e3
    e2e_ms = float(max_over_ranks([e2e_ms], device=dev)[0])
    h2d = n_chunks * chunk * (frame0.numel() + frame1.numel()) * 4
    d2h = n_chunks * (bat.n_poses * 7 * 8 + bat.n_patches * 8 + chunk * (66 * 8 + 4))
    res = bat.read()
    gathered = gather_poses(np.concatenate([r[0] for r in res]), device=dev)
    assert len(gathered) == world
    if rank != 0:
        return
    E_total = E_chunk * n_chunks * world
    # roofline of the correlation launch of the last chunk: algorithmic bytes of every
    # distinct trajectory's edges (the chunk replicates them) over the launch time
    hbm, peak_kind = load_peaks()
    level_shapes = [(H0, W0i), (H1, W1i)]
    sampled = geos[: min(4, len(geos))]  # exact per-edge bytes of 4 trajectories, scaled to the chunk
    per_edge = sum(corr_bytes_per_edge(p, w0.K, level_shapes)[0] for _, p, _ in sampled) / sum(
        len(p["e_patch"]) for _, p, _ in sampled)
    chunk_bytes = per_edge * E_chunk
    achieved = chunk_bytes / (corr_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": E_total / (mean_ms * 1e-3), "unit": "edge-iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 corr (f64 coords/weights), f64 BA", "data": "synthetic",
        "config": batch_config(n_seq * world, world, chunk, n_chunks, E_chunk, len(geos), F),
        "last_chunk_corr_ms": corr_ms, "last_chunk_ba_ms": ba_ms,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": None, "kernel": "corr_tma_kernel", "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": chunk_bytes,
                     "bytes_note": f"per-edge bytes measured on {len(sampled)} of the {len(geos)} trajectories"},
        "e2e": {"value": E_total / (e2e_ms * 1e-3), "unit": "edge-iterations/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms},
        "gpu_launches": int(launches), "clocks": clk, "wall_s_timed_region": t_wall,
    }
    print(json.dumps(line), flush=True)


def run_e2e(args, w, prob, ctx, stream, win):
    """Same step through the public API with HOST buffers: upload the newest
    frame's pyramid and the window state, run, read back the corr volume and
    the BA result — copies inside the timed region."""
    import torch

    E = win.n_edges
    l0 = torch.from_numpy(w.level0[-1]).pin_memory()
    l1 = torch.from_numpy(w.level1[-1]).pin_memory()
    vol = torch.empty((E, 2, 9, 7, 7), dtype=torch.float32).pin_memory()
    vol_np = vol.numpy()
    F = w.cfg["frames"]
    arrays = [prob["poses"], prob["fixed"], prob["pose_frames"], prob["patch_src"], prob["patch_x"],
              prob["patch_y"], prob["depth"], prob["patch_feats"], prob["e_patch"], prob["e_pose"], prob["e_delta"],
              prob["e_weight"]]
    h2d = l0.numel() * 4 + l1.numel() * 4 + sum(np.asarray(a).nbytes for a in arrays)
    d2h = vol.numel() * 4 + prob["poses"].nbytes + prob["depth"].nbytes + 8 * 3

    def pinned(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

    hp = dict(prob)  # the step's host inputs live in pinned memory (DMA straight from the caller's arrays)
    for k in ("poses", "fixed", "pose_frames", "patch_src", "patch_x", "patch_y", "depth", "patch_feats",
              "e_patch", "e_pose", "e_delta", "e_weight"):
        hp[k] = pinned(prob[k])

    def one():
        ctx.frames_upload(F - 1, l0.numpy(), l1.numpy())
        win.load(hp, hp["pose_frames"], hp["patch_feats"], w.K, w.image)
        win.iteration(2, corr_out=vol_np)
        return win.read()

    for _ in range(max(1, args.warmup)):
        one()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = max(1, min(args.steps, 50))
    for _ in range(n):
        one()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / n * 1e3
    return {"ms": ms, "h2d": int(h2d), "d2h": int(d2h)}


def relaunch(n: int) -> None:
    """`python bench.py --gpus N` without torchrun: run this script under
    torch.distributed.run with N ranks (one per GPU, rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--sequences", type=int, default=1024, help="c5: sequences in the whole job")
    ap.add_argument("--chunk", type=int, default=256, help="c5: sequences per device launch")
    ap.add_argument("--distinct", type=int, default=32, help="c5: distinct trajectories per rank")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of a captured step")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        relaunch(args.gpus)  # does not return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" in os.environ and args.gpus != world:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    try:
        if args.config == "c5":
            run_batch(args, rank, world, local_rank)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
