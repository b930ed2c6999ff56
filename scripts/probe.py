"""Per-kernel device times of one workload (development probe)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2204_14242_b200 import Context, config_array, result_dicts

def run(name, k, g, cfgs, reps=20):
    ctx = Context(0, torch.cuda.current_stream().cuda_stream)
    kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(g)
    a = config_array(kid, gid, cfgs)
    n = len(a)
    dc = torch.from_numpy(a.view(np.uint8)).cuda()
    do = torch.empty(n * 336, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        ctx.estimate_async(dc.data_ptr(), n, do.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ctx.estimate_async(dc.data_ptr(), n, do.data_ptr())
    e1.record(); torch.cuda.synchronize()
    tot = e0.elapsed_time(e1) / reps
    ctx.profile_enable(True)
    e0.record()
    for _ in range(reps):
        ctx.estimate_async(dc.data_ptr(), n, do.data_ptr())
    e1.record(); torch.cuda.synchronize()
    ctx.profile_enable(False)
    prof = ctx.profile_read()
    totp = e0.elapsed_time(e1) / reps
    print(f"{name}: n={n} step {tot:.3f} ms (profiled {totp:.3f}) -> {n/tot*1e3:.0f} configs/s")
    for kname, (ms, cnt) in prof.items():
        if cnt: print(f"   {kname:8s} {ms/cnt:9.4f} ms")

WORK = {
    "configs1": ("configs1 K25 512^3 A100 168", lambda: (W.k25(512), W.gpu_a100(), W.space_stencil_paper()), 20),
    "lbm15": ("configs2 LBM15 256^3 A100 49", lambda: (W.lbm15(256), W.gpu_a100(), W.space_lbm()), 20),
    "lbm27": ("configs2 LBM27 256^3 A100 49", lambda: (W.lbm27(256), W.gpu_a100(), W.space_lbm()), 20),
    "configs0": ("configs0 K7 64^3 V100 16", lambda: (W.k7(64), W.gpu_v100(), W.space_k7()), 20),
    "extended": ("extended K25 512^3 A100", lambda: (W.k25(512), W.gpu_a100(), W.space_extended()), 3),
}
# python scripts/probe.py [name ...]  (default: all)
if __name__ == "__main__":
    for name in (sys.argv[1:] or list(WORK)):
        label, mk, reps = WORK[name]
        run(label, *mk(), reps=reps)
