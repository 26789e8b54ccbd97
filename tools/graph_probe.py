import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
w, prob, ctx, stream, win = bench.setup("c2", seed=0, device=0)
F = w.cfg["frames"]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda:0")
def step():
    ctx.frames_refresh(F - 1)
    win.iteration(2)
with torch.cuda.stream(stream):
    for _ in range(5):
        win.reset(); step()
torch.cuda.synchronize()
def timed(fn, n=300):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    with torch.cuda.stream(stream):
        for i in range(n):
            flush.zero_(); win.reset()
            ev[i][0].record(stream); fn(); ev[i][1].record(stream)
    torch.cuda.synchronize()
    return np.mean([a.elapsed_time(b) for a, b in ev])
print("eager ms", timed(step))
g = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(g, stream=stream, capture_error_mode="relaxed"):
        step()
    torch.cuda.synchronize()
    print("captured")
    print("graph ms", timed(g.replay))
    # check the graph result equals eager
    win.reset(); 
    with torch.cuda.stream(stream): g.replay()
    torch.cuda.synchronize(); pg, dg, ng = win.read()
    win.reset()
    with torch.cuda.stream(stream): step()
    torch.cuda.synchronize(); pe, de, ne = win.read()
    print("equal", np.array_equal(pg, pe), np.array_equal(dg, de))
except Exception as ex:
    print("capture failed:", type(ex).__name__, ex)
