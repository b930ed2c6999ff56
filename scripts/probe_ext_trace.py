"""Extended 1890-config space, one estimate (development probe for the k_sclass trace build)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2204_14242_b200 import Context, config_array
ctx = Context(0, torch.cuda.current_stream().cuda_stream)
k, g = W.k25(512), W.gpu_a100()
kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(g)
a = config_array(kid, gid, W.space_extended())
dc = torch.from_numpy(a.view(np.uint8)).cuda()
do = torch.empty(len(a) * 336, dtype=torch.uint8, device="cuda")
ctx.estimate_async(dc.data_ptr(), len(a), do.data_ptr())
torch.cuda.synchronize()
print("done", len(a))
