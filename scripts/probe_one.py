"""Per-kernel device times for single configurations vs the whole configs[1] batch (development probe):
is a kernel bound by its slowest item (single-configuration time close to the batch time) or by the
whole batch's throughput?"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import workloads as W
from paper_2204_14242_b200 import Context, config_array

ctx = Context(0, torch.cuda.current_stream().cuda_stream)
k, g = W.k25(512), W.gpu_a100()
kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(g)
space = W.space_stencil_paper()


def prof(cfgs, reps=10):
    a = config_array(kid, gid, cfgs)
    dc = torch.from_numpy(a.view(np.uint8)).cuda()
    do = torch.empty(len(a) * 336, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        ctx.estimate_async(dc.data_ptr(), len(a), do.data_ptr())
    torch.cuda.synchronize()
    ctx.profile_enable(True)
    for _ in range(reps):
        ctx.estimate_async(dc.data_ptr(), len(a), do.data_ptr())
    torch.cuda.synchronize()
    ctx.profile_enable(False)
    p = ctx.profile_read()
    return {kk: v[0] / v[1] * 1e3 for kk, v in p.items() if v[1]}


full = prof(space)
print("all 168:", {kk: round(v, 1) for kk, v in full.items()})
picks = [i for i, c in enumerate(space) if c[0] in ((1, 16, 64), (2, 8, 64), (16, 2, 32), (1024, 1, 1), (32, 32, 1),
                                                     (8, 8, 16), (64, 4, 4))]
for i in picks:
    r = prof([space[i]])
    print(space[i], {kk: round(v, 1) for kk, v in r.items() if kk in ("k_plan", "k_rows", "k_fold", "k_smset",
                                                                       "k_sclass", "k_warp", "k_wclass", "k_instr")})
