"""ws_rank_async on synthetic records (development profiling target): device us per call for n in argv."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2204_14242_b200 import Context
from paper_2204_14242_b200.ws import RESULT_DTYPE

ctx = Context(0, torch.cuda.current_stream().cuda_stream)
for n in [int(a) for a in sys.argv[1:]] or [168, 8232, 100000]:
    rng = np.random.default_rng(1)
    r = np.zeros(n, dtype=RESULT_DTYPE)
    r["t_pred"] = rng.random(n)
    d = torch.from_numpy(r.view(np.uint8).copy()).cuda()
    top = torch.zeros(10, dtype=torch.int32, device="cuda")
    for _ in range(3):
        ctx.rank_async(d.data_ptr(), n, 10, top.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        ctx.rank_async(d.data_ptr(), n, 10, top.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    print(f"rank n={n}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per ws_rank_async ({ctx.last_launch_count()} launches)")
