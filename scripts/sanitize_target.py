"""Tiny workload for compute-sanitizer (memcheck / racecheck / synccheck): every kernel of the
library runs once on small inputs -- estimate (all variants, outlook metrics), rank, simulate,
fit, the validation stencil."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2204_14242_b200 import Context, config_array  # noqa: E402

ctx = Context(0)
k = W.stencil_star(20, 12, 10, 4, regs=64)
g = W.with_outlook(dict(W.gpu_a100(), n_sm=6), page_bytes=4096, link_bw=1e12)
kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(g)
cfgs = [((8, 2, 2), (1, 1, 1), 1, v) for v in (0, 1, 2, 4, 8, 15)] + [((4, 4, 4), (1, 2, 1), 2, 0),
                                                                      ((32, 1, 1), (1, 1, 2), 0, 6)]
a = config_array(kid, gid, cfgs)
res = ctx.estimate(a)
ctx.rank(res, 4)
kl = ctx.describe_kernel(W.lbm15(6))
ctx.estimate(config_array(kl, gid, [((4, 2, 2), (1, 1, 1), 1, 0), ((2, 2, 2), (2, 1, 1), 0, 9)]))
rows = ctx.simulate(config_array(kid, gid, [c[:3] for c in cfgs[:3]]), [1 << 20, 8192, 1024])
ctx.fit_gompertz([0.1 * i for i in range(12)], [1.0 / (1 + 0.1 * i * i) for i in range(12)])
src = torch.rand((18, 18, 20), dtype=torch.float64, device="cuda")
dst = torch.zeros_like(src)
ctx.validate_stencil25(src.data_ptr(), dst.data_ptr(), (12, 10, 10), (8, 2, 2), (1, 1, 2), reps=1)
torch.cuda.synchronize()
print("sanitize target ok", len(res), len(rows))
