"""Multi-process host logic of the sharded sweep on CPU with gloo,
world size 2: shard plans partition the batch deterministically and balance it, and the
gathered result records come back in global order, byte-identical on every rank."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W
from paper_2204_14242_b200 import dist as D


def test_shard_plan_partition_and_balance():
    cfgs = W.space_stencil_paper()
    costs = [D.proxy_cost(c) for c in cfgs]
    for world in (1, 2, 3, 4, 8):
        sh = D.shard_plan(costs, world)
        flat = sorted(i for s in sh for i in s)
        assert flat == list(range(len(cfgs)))
        loads = [sum(costs[i] for i in s) for s in sh]
        assert max(loads) - min(loads) <= max(costs)          # LPT bound
        assert sh == D.shard_plan(costs, world)                # deterministic


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_record(g, i):
    b = bytearray(D.RECORD_BYTES)
    b[0:8] = int(i * 7919 + 3 + g * 104729).to_bytes(8, "little")
    b[100:108] = int(i).to_bytes(8, "little")
    b[200:204] = int(g).to_bytes(4, "little")
    return bytes(b)


def _cfg_records(n):
    from paper_2204_14242_b200.ws import CONFIG_DTYPE
    import numpy as np
    r = np.zeros(n, dtype=CONFIG_DTYPE)
    r["kernel_id"] = np.arange(n)          # the fake estimator reads the global index from here
    return r


def _fake_estimate(H):
    def est(local_cfg, out):
        m = len(local_cfg)
        for g in range(H):
            for j in range(m):
                out[g * m + j] = torch.tensor(list(_fake_record(g, int(local_cfg[j]["kernel_id"]))), dtype=torch.uint8)
    return est


def _worker(rank, world, port, n, H, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    costs = [float((i * 37) % 11 + 1) for i in range(n)]
    sw = D.ShardedSweep(None, _cfg_records(n), list(range(H)), costs, device=torch.device("cpu"),
                        estimate=_fake_estimate(H))
    g = sw.step()
    out[rank] = g.numpy().tobytes()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,H", [(1, 1), (7, 3), (168, 2), (3, 4)])
def test_sharded_sweep_gather_gloo_world2(n, H):
    """The real ShardedSweep gather path (padding, one all-gather, the precomputed permutation to
    the canonical [hardware set][configuration] order) with a fake estimator, world size 2."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, H, out), nprocs=world, join=True)
    expect = b"".join(_fake_record(g, i) for g in range(H) for i in range(n))
    assert out[0] == expect
    assert out[1] == expect


def test_sharded_sweep_single_rank_matches_canonical():
    costs = [1.0] * 5
    sw = D.ShardedSweep(None, _cfg_records(5), [0, 1], costs, device=torch.device("cpu"), estimate=_fake_estimate(2))
    assert sw.step().numpy().tobytes() == b"".join(_fake_record(g, i) for g in range(2) for i in range(5))
