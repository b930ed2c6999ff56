"""Internal graph (ws_estimate_ranked_async per step) vs the same call captured once in a caller's
CUDA graph and replayed: device time per step over 500 back-to-back steps, and host time per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2204_14242_b200 import Context, config_array

s = torch.cuda.Stream()
ctx = Context(0, s.cuda_stream)
kid, gid = ctx.describe_kernel(W.k25(512)), ctx.describe_gpu(W.gpu_a100())
a = config_array(kid, gid, W.space_stencil_paper())
n = len(a)
dc = torch.from_numpy(a.view(np.uint8).copy()).cuda()
do = torch.empty(n * 336, dtype=torch.uint8, device="cuda")
top = torch.zeros(10, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
def run(fn, reps=500):
    for _ in range(5): fn()
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    for _ in range(reps): fn()
    e1.record(s)
    t1 = time.perf_counter()
    s.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3, (t1 - t0) / reps * 1e6
f1 = lambda: ctx.estimate_ranked_async(dc.data_ptr(), n, do.data_ptr(), 10, top.data_ptr())
d, h = run(f1); print(f"internal graph: device {d:.1f} us/step, host {h:.1f} us/call")
f2 = lambda: ctx.estimate_async(dc.data_ptr(), n, do.data_ptr())
d, h = run(f2); print(f"estimate_async: device {d:.1f} us/step, host {h:.1f} us/call")
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    f1()
def rep():
    with torch.cuda.stream(s):
        g.replay()
d, h = run(rep); print(f"caller graph:   device {d:.1f} us/step, host {h:.1f} us/call")
