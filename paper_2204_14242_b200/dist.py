"""Multi-GPU plumbing: configurations are independent, so a sweep is
sharded over ranks (one process per GPU) and the only exchange is one all-gather of
the fixed-size result records (336 B, include/ws.h `ws_result`) over NCCL; every rank
then ranks the gathered set with the library's `ws_rank_async` and holds identical bytes.

This module holds host logic only (shard assignment, padding, gather, reordering);
every estimator step runs in libwsb200.so.
"""
from __future__ import annotations

import heapq

import torch
import torch.distributed as dist

RECORD_BYTES = 336


def proxy_cost(config) -> float:
    """Scheduling heuristic (not part of any result): the work of a configuration grows with
    the depth of its block layer (the L_z layer set spans one block layer) plus the
    halo; (block, fold, k) as in workloads."""
    (bx, by, bz), (fx, fy, fz) = config[0], config[1]   # (block, fold, k[, variant])
    return float(bz * fz + 8)


def shard_plan(costs, world: int):
    """Longest-processing-time-first assignment of items to `world` ranks.

    Deterministic (ties broken by item index, then rank).  Returns one ascending list of item
    indices per rank; together they partition range(len(costs))."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0.0, r) for r in range(world)]
    heapq.heapify(heap)
    shards = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        shards[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(s) for s in shards]


def gather_records(local: torch.Tensor, shards, group=None) -> torch.Tensor:
    """All-gather every rank's result records and return them in global item order.

    local: uint8 tensor (len(shards[rank]), RECORD_BYTES) on this rank's device (CPU for gloo).
    Returns a uint8 tensor (n_items, RECORD_BYTES), identical on every rank."""
    world = len(shards)
    m = max(len(s) for s in shards)
    padded = torch.zeros((m, RECORD_BYTES), dtype=torch.uint8, device=local.device)
    padded[: local.shape[0]] = local
    if world == 1:
        gathered = padded.unsqueeze(0)
    elif dist.get_backend(group) == "nccl":
        gathered = torch.empty((world, m, RECORD_BYTES), dtype=torch.uint8, device=local.device)
        dist.all_gather_into_tensor(gathered.view(-1), padded.view(-1), group=group)
    else:
        parts = [torch.empty_like(padded) for _ in range(world)]
        dist.all_gather(parts, padded, group=group)
        gathered = torch.stack(parts)
    n = sum(len(s) for s in shards)
    src = torch.empty(n, dtype=torch.long)
    for r, s in enumerate(shards):
        for j, i in enumerate(s):
            src[i] = r * m + j
    return gathered.view(world * m, RECORD_BYTES).index_select(0, src.to(local.device))


def estimate_sharded(ctx, cfg_records, group=None, k_top: int = 10):
    """Shard a batch of ws_config records (numpy CONFIG_DTYPE) over the ranks of `group`,
    estimate locally on this rank's GPU, all-gather, rank the full set on every rank.

    Returns (results uint8 tensor (n, 336) on this rank's GPU, top-k indices tensor)."""
    from .ws import CONFIG_DTYPE, RESULT_DTYPE
    import numpy as np
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = len(cfg_records)
    cfgs = [((int(c["block"][0]), int(c["block"][1]), int(c["block"][2])),
             (int(c["fold"][0]), int(c["fold"][1]), int(c["fold"][2])), int(c["blocks_per_sm"]))
            for c in cfg_records]
    shards = shard_plan([proxy_cost(c) for c in cfgs], world)
    mine = np.ascontiguousarray(cfg_records[shards[rank]], dtype=CONFIG_DTYPE)
    dev = torch.device("cuda", torch.cuda.current_device())
    d_cfg = torch.from_numpy(mine.view(np.uint8).copy()).to(dev)
    d_out = torch.empty((len(mine), RESULT_DTYPE.itemsize), dtype=torch.uint8, device=dev)
    if len(mine):
        ctx.estimate_async(d_cfg.data_ptr(), len(mine), d_out.data_ptr())
    allres = gather_records(d_out, shards, group) if world > 1 else d_out
    top = torch.empty(max(1, k_top), dtype=torch.int32, device=dev)
    ctx.rank_async(allres.data_ptr(), n, k_top, top.data_ptr())
    return allres, top[: min(k_top, n)]
