import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import workloads as W
from oracle import oracle as O
from paper_2204_14242_b200 import Context, config_array, result_dicts
ctx = Context(0)
k, g = W.k7(12), W.gpu_v100()
cf = [((32, 2, 1), (1, 1, 1), 0), ((32, 1, 1), (1, 1, 1), 0), ((32, 4, 2), (1, 1, 1), 0)]
o = O.estimate_batch(k, g, cf, 4)
kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(g)
for rep in range(5):
    r = result_dicts(ctx.estimate(config_array(kid, gid, cf)))
    print(rep, [(x['sm_ld_sectors'], x['sm_ld_lines']) for x in r], 'oracle', [(x['sm_ld_sectors'], x['sm_ld_lines']) for x in o], [x['k'] for x in r])
