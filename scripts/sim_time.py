"""ws_simulate wall / device time of the bench's NEXT-1 workload (168 configs at 128^3 x 16 capacities)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_2204_14242_b200 import Context, config_array
ctx = Context(0)
k, g = W.k25(128), W.gpu_a100()
cf = config_array(ctx.describe_kernel(k), ctx.describe_gpu(g), W.space_stencil_paper())
caps = [int(g["l2_bytes"] // 2 * 2 ** (e / 2)) for e in range(-12, 4)]
ctx.simulate(cf[:4], caps)
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.simulate(cf, caps)
    torch.cuda.synchronize()
    print(f"simulate: {(time.perf_counter() - t0) * 1e3:.1f} ms wall")
