"""One ws_simulate call of the 25pt space at n^3 x 16 capacities (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from paper_2204_14242_b200 import Context, config_array
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ctx = Context(0)
k, g = W.k25(n), W.gpu_a100()
cf = config_array(ctx.describe_kernel(k), ctx.describe_gpu(g), W.space_stencil_paper())
caps = [int(g["l2_bytes"] // 2 * 2 ** (e / 2)) for e in range(-12, 4)]
ctx.simulate(cf, caps)
