"""Per-kernel device times of the extended 1890-config space at 512^3, A100."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "probe.py")).read()
exec(src[:src.index('run("configs1')])
run("extended K25 512^3 A100", W.k25(512), W.gpu_a100(), W.space_extended(), reps=3)
