"""Per-kernel device times of the 168-config 25pt space at n^3 (A100 parameters), WS_SERIAL optional."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv += [] if len(sys.argv) > 1 else ["64"]
import importlib.util
spec = importlib.util.spec_from_file_location("probe", os.path.join(os.path.dirname(os.path.abspath(__file__)), "probe.py"))
import workloads as W
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "probe.py")).read()
src = src[:src.index('run("configs1')]
exec(src)
for n in [int(a) for a in sys.argv[1:]]:
    run(f"k25 {n}^3", W.k25(n), W.gpu_a100(), W.space_stencil_paper())
