"""Parity of the estimator's alternate launch paths (run in a subprocess by test_modes.py with
WS_FOLD_MODE / WS_SERIAL / WS_GRAPH set): the fold by CTA or by warp, all chains on one stream,
eager launches instead of graph replay -- every count against the oracle."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import workloads as W  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2204_14242_b200 import Context, config_array, result_dicts  # noqa: E402
from parity_util import compare  # noqa: E402

NT = max(1, min(32, os.cpu_count() or 1))
ctx = Context(0)
cases = [
    (W.k25(48), dict(W.gpu_a100(), n_sm=24), W.space_stencil_paper()[::5]),
    (W.lbm15(8), dict(W.gpu_a100(), n_sm=3), [((4, 2, 2), (1, 1, 1), 1), ((8, 1, 1), (1, 1, 1), 0),
                                              ((2, 2, 2), (2, 1, 1), 0, 3)]),
    (W.stencil_star(40, 36, 44, 4, regs=64), dict(W.gpu_a100(), n_sm=24),
     [c for c in W.space_extended() if c[0][0] * c[0][1] * c[0][2] <= 512][::40]),
]
errs, n = [], 0
for i, (k, g, cf) in enumerate(cases):
    kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(g)
    for rep in range(2):  # the second call replays the captured graph (unless WS_GRAPH=0)
        res = result_dicts(ctx.estimate(config_array(kid, gid, cf)))
        ora = O.estimate_batch(k, g, cf, NT) if rep == 0 else ora
        for j, (a, b) in enumerate(zip(res, ora)):
            errs += compare(a, b, f"case{i} rep{rep} [{j}] {cf[j]}")
        n += len(cf)
if errs:
    print("\n".join(errs[:40]))
    sys.exit(1)
print("mode target ok", n)
