"""Per-kernel device ms of one estimate of the 168-config 512^3 space per variant / parameter set
(WS_SERIAL=1 gives uncontended kernel times)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2204_14242_b200 import Context, config_array

ctx = Context(0, torch.cuda.current_stream().cuda_stream)
k = W.k25(512)
for gname, g in [("A100", W.gpu_a100()), ("B200", W.with_outlook(W.gpu_b200_like()))]:
    for var in (0, 1, 2, 4, 7):
        kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(g)
        cf = config_array(kid, gid, [c + (var,) for c in W.space_stencil_paper()])
        n = len(cf)
        d_cfg = torch.from_numpy(cf.view(np.uint8).copy()).cuda()
        d_out = torch.empty(n * 336, dtype=torch.uint8, device="cuda")
        for _ in range(2):
            ctx.estimate_async(d_cfg.data_ptr(), n, d_out.data_ptr())
        torch.cuda.synchronize()
        ctx.profile_enable(True)
        for _ in range(3):
            ctx.estimate_async(d_cfg.data_ptr(), n, d_out.data_ptr())
        torch.cuda.synchronize()
        ctx.profile_enable(False)
        p = ctx.profile_read()
        print(gname, var, {kk: round(v[0] / 3, 3) for kk, v in p.items() if v[1]}, flush=True)
