"""Bounds-check workload (tests/test_bounds_check.py): run under WS_LIB=libwsb200_check.so, every
estimate-chain kernel on the paper's workloads at full size and on small edge cases, then print
the device-side bounds-check counters (ws_check_read)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2204_14242_b200 import Context, config_array  # noqa: E402

ctx = Context(0)
flag = ctx.check_read()
assert flag[0] == 1, "not the bounds-check build"
gid = ctx.describe_gpu(W.gpu_a100())
gb = ctx.describe_gpu(W.with_outlook(W.gpu_b200_like(), page_bytes=1 << 21, link_bw=1e13))
runs = [
    (W.k25(512), gid, W.space_stencil_paper(), "configs[1] 512^3"),
    (W.k25(512), gb, [c[:3] + (7,) for c in W.space_stencil_paper()], "variants + outlook 512^3"),
    (W.lbm15(256), gid, W.space_lbm(), "LBM15 256^3"),
    (W.lbm27(256), gid, W.space_lbm(), "LBM27 256^3"),
    (W.k25(96), gid, W.space_extended(), "extended 96^3"),
    (W.k25(64), gid, W.space_stencil_paper()[::11], "configs[0]-like 64^3"),
    (W.k7(64), ctx.describe_gpu(W.gpu_v100()), W.space_k7(), "7pt V100"),
]
for k, g, space, name in runs:
    kid = ctx.describe_kernel(k)
    res = ctx.estimate(config_array(kid, g, space))
    ctx.rank(res, 10)
    chk = ctx.check_read()
    print(f"{name}: {len(res)} configs, status ok {int((res['status'] == 0).sum())}, check {chk}")
    assert chk[1] == 0, (name, chk)
# the fused model + rank path and the multi-hardware fan-out
kid = ctx.describe_kernel(W.k25(128))
a = config_array(kid, gid, W.space_stencil_paper())
dc = torch.from_numpy(a.view(np.uint8).copy()).cuda()
do = torch.zeros(len(a) * 336, dtype=torch.uint8, device="cuda")
top = torch.zeros(10, dtype=torch.int32, device="cuda")
ctx.estimate_ranked_async(dc.data_ptr(), len(a), do.data_ptr(), 10, top.data_ptr())
torch.cuda.synchronize()
sets = [gid, gb, ctx.describe_gpu(W.gpu_v100())]
ctx.estimate_multi(a, sets)
ctx.simulate(config_array(kid, gid, W.space_stencil_paper()[:6]), [1 << 16, 1 << 20])
chk = ctx.check_read()
print(f"ranked / multi / simulate: check {chk}")
assert chk[1] == 0, chk
print("bounds check target ok")
