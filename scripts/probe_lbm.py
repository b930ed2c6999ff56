"""Per-kernel device times of BJ configs[2] (LBM15 / LBM27 at 256^3, 49 configs, A100)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "probe.py")).read()
exec(src[:src.index('run("configs1')])
run("LBM15 256^3", W.lbm15(256), W.gpu_a100(), W.space_lbm())
run("LBM27 256^3", W.lbm27(256), W.gpu_a100(), W.space_lbm())
