"""NEXT-1 probe: device time of ws_simulate on the 25pt paper space at n^3 (A100) x capacities."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2204_14242_b200 import Context, config_array

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ncap = int(sys.argv[2]) if len(sys.argv) > 2 else 16
ctx = Context(0, torch.cuda.current_stream().cuda_stream)
k, g = W.k25(n), W.gpu_a100()
kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(g)
cf = config_array(kid, gid, W.space_stencil_paper())
caps = [int(g["l2_bytes"] // 2 * 2 ** (e / 2)) for e in range(-ncap + 4, 4)]
ctx.profile_enable(True)
for it in range(3):
    t = time.time()
    r = ctx.simulate(cf, caps)
    dt = time.time() - t
    prof = ctx.profile_read()
    print(f"n={n} wall {dt*1e3:.1f} ms", {k: round(v[0], 3) for k, v in prof.items() if v[1]})
req = sum(row[0]["l1_requests"] + row[0]["st_requests"] for row in r)
print("l1+st requests", req)
