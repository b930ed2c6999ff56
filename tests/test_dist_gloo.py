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


def _fake_record(i):
    b = bytearray(D.RECORD_BYTES)
    b[0:8] = int(i * 7919 + 3).to_bytes(8, "little")
    b[100:108] = int(i).to_bytes(8, "little")
    return bytes(b)


def _worker(rank, world, port, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    costs = [float((i * 37) % 11 + 1) for i in range(n)]
    shards = D.shard_plan(costs, world)
    mine = shards[rank]
    local = torch.tensor([list(_fake_record(i)) for i in mine], dtype=torch.uint8).view(-1, D.RECORD_BYTES) \
        if mine else torch.zeros((0, D.RECORD_BYTES), dtype=torch.uint8)
    g = D.gather_records(local, shards)
    out[rank] = g.numpy().tobytes()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [1, 7, 168])
def test_gather_records_gloo_world2(n):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, out), nprocs=world, join=True)
    expect = b"".join(_fake_record(i) for i in range(n))
    assert out[0] == expect
    assert out[1] == expect
