"""One workload's estimate launches for ncu (development profiling target).

Runs 3 estimates of BJ configs[1] (168 configs, 3D-25pt 512^3, A100); profile the third:
  ncu --set full -k regex:"k_" -s 18 -c 9 python scripts/ncu_target.py [lbm15|lbm27|k7]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2204_14242_b200 import Context, config_array

which = sys.argv[1] if len(sys.argv) > 1 else "k25"
k, g, space = {
    "k25": (W.k25(512), W.gpu_a100(), W.space_stencil_paper()),
    "lbm15": (W.lbm15(256), W.gpu_a100(), W.space_lbm()),
    "lbm27": (W.lbm27(256), W.gpu_a100(), W.space_lbm()),
    "k7": (W.k7(64), W.gpu_v100(), W.space_k7()),
}[which]
ctx = Context(0, torch.cuda.current_stream().cuda_stream)
kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(g)
a = config_array(kid, gid, space)
n = len(a)
dc = torch.from_numpy(a.view(np.uint8)).cuda()
do = torch.empty(n * 336, dtype=torch.uint8, device="cuda")
for _ in range(3):
    ctx.estimate_async(dc.data_ptr(), n, do.data_ptr())
    torch.cuda.synchronize()
print("ok", n)
