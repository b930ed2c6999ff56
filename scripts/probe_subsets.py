"""k_sclass / k_rows device time per subset of the extended space (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2204_14242_b200 import Context, config_array, result_dicts
ctx = Context(0, torch.cuda.current_stream().cuda_stream)
k, g = W.k25(512), W.gpu_a100()
kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(g)
sp = W.space_extended()
groups = {}
for c in sp:
    T = c[0][0] * c[0][1] * c[0][2]
    groups.setdefault((T, c[1]), []).append(c)
for key in sorted(groups):
    cf = config_array(kid, gid, groups[key])
    ctx.estimate(cf)
    ctx.profile_enable(True)
    r = ctx.estimate(cf)
    ctx.profile_enable(False)
    p = ctx.profile_read()
    rr = result_dicts(r)
    print(key, len(cf), "k", sorted({x["k"] for x in rr}), "sclass %.3f rows %.3f warp %.3f" % (p["k_sclass"][0], p["k_rows"][0], p["k_wclass"][0]), flush=True)
