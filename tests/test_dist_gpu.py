"""Rank-count invariance of the sharded sweep with the real estimator (SURVEY §4 layer 4, §8(e)):
two processes on one GPU (gloo over host copies) run `ShardedSweep` over the configs[3]-shaped
space (168 configurations x the 51 configs[3] hardware sets, 3D-25pt at 64^3) with the device-
derived cost plan broadcast from rank 0; the gathered, ranked records must be byte-identical to a
single rank's `ws_estimate_multi` + `ws_rank` of the same space."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    import workloads as W
    from paper_2204_14242_b200 import Context, config_array
    ctx = Context(0)
    kid = ctx.describe_kernel(W.k25(64))
    gids = [ctx.describe_gpu(g) for g in W.hw_grid_configs3()]
    return ctx, config_array(kid, 0, W.space_stencil_paper()), gids


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2204_14242_b200 import dist as D
    ctx, cf, gids = _setup()
    obj = [D.device_costs(ctx, cf, gids) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    sw = D.ShardedSweep(ctx, cf, gids, obj[0], device=torch.device("cuda", 0))
    res = sw.step()
    torch.cuda.synchronize()
    out[rank] = (res.cpu().numpy().tobytes(), [len(s) for s in sw.shards])
    dist.barrier()
    dist.destroy_process_group()
    ctx.close()


def _single(out):
    ctx, cf, gids = _setup()
    from paper_2204_14242_b200.ws import RESULT_DTYPE
    r = ctx.estimate_multi(cf, gids).reshape(-1)
    ctx.rank(r, 10)
    out["single"] = r.tobytes()
    ctx.close()


def test_sharded_sweep_world2_byte_identical():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    ctx_mp = mp.get_context("spawn")
    mgr = ctx_mp.Manager()
    out = mgr.dict()
    p = ctx_mp.Process(target=_single, args=(out,))
    p.start()
    p.join()
    assert p.exitcode == 0
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    b0, sh0 = out[0]
    b1, sh1 = out[1]
    assert sh0 == sh1 and sum(sh0) == 168 and min(sh0) > 0
    assert b0 == b1 == out["single"]
