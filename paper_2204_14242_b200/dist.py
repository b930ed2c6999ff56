"""Multi-GPU plumbing: configurations are independent, so a sweep is sharded
over ranks (one process per GPU) and the only exchange is one all-gather of the fixed-size
result records (336 B, include/ws.h `ws_result`) over NCCL; every rank then ranks the gathered
set with the library's `ws_rank_async` and holds identical bytes.

This module holds host logic only (cost model for the shard plan, shard assignment, padding,
the gather permutation); every estimator step runs in libwsb200.so.

`ShardedSweep` is the BJ configs[3] path: a configuration space x a list of hardware sets
(`ws_estimate_multi`), sharded by configuration.  Everything that does not change between sweeps
(shard plan, per-rank device buffers, the permutation from the gathered layout to the canonical
`[hardware set][configuration]` order) is built once, outside any timed region; a step is
estimate -> one all-gather -> one index_select -> rank.
"""
from __future__ import annotations

import heapq

import numpy as np
import torch
import torch.distributed as dist

RECORD_BYTES = 336


def proxy_cost(config) -> float:
    """Device-free fallback cost (tests without a GPU): the work of a configuration grows with
    the depth of its block layer (the L_z layer set spans one block layer)."""
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


def device_costs(ctx, cfg_records, gpu_ids) -> list:
    """Per-configuration device cost (ms) of `ws_estimate_multi` over `gpu_ids`, derived on the
    device: one profiled pass of the whole batch gives each kernel's milliseconds per algorithmic
    work unit (`ws_profile_read` / `ws_work_read`); one work-count pass per configuration gives its
    units per kernel.  cost_i = sum_k ms_k / U_k * u_k,i + (time of the kernels without work
    counters) / n.  Deterministic given the measured rates; compute on one rank and broadcast."""
    n = len(cfg_records)
    ctx.estimate_multi(cfg_records, gpu_ids)              # warm-up (graph capture)
    ctx.profile_enable(True)
    ctx.estimate_multi(cfg_records, gpu_ids)
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    total = ctx.work_read()
    rate = {k: prof[k][0] / total[k] for k in total if total[k] > 0 and k in prof and prof[k][1] > 0}
    fixed = sum(v[0] for k, v in prof.items() if k not in rate)
    costs = []
    for i in range(n):
        ctx.estimate_multi(cfg_records[i:i + 1], gpu_ids)
        u = ctx.work_read()
        costs.append(fixed / n + sum(rate[k] * u.get(k, 0) for k in rate))
    return costs


class ShardedSweep:
    """`n` configurations x `len(gpu_ids)` hardware sets, sharded by configuration over the ranks
    of `group` (world 1 without torch.distributed).

    costs:    per-configuration costs for the LPT plan (identical on every rank: `device_costs` on
              rank 0, then broadcast).
    estimate: optional callable (local config records, out tensor) used instead of the library
              (the CPU tests plug a fake estimator in; the gather logic is the same).
    Backend nccl: records stay on the device.  Backend gloo: host copies around the all-gather.
    Result of `step()`: a uint8 tensor (n_gpu * n, 336) in canonical order `g * n + i`, ranked on
    every rank; byte-identical for every world size."""

    def __init__(self, ctx, cfg_records, gpu_ids, costs, group=None, device=None, k_top=10, estimate=None):
        from .ws import CONFIG_DTYPE
        self.ctx, self.group, self.k_top = ctx, group, k_top
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        self.backend = dist.get_backend(group) if self.world > 1 else "none"
        self.dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.n, self.H = len(cfg_records), len(gpu_ids)
        self.gpu_ids = [int(g) for g in gpu_ids]
        self.shards = shard_plan(costs, self.world)
        self.m = max(len(s) for s in self.shards)
        mine = np.ascontiguousarray(cfg_records[self.shards[self.rank]], dtype=CONFIG_DTYPE)
        self.n_local = len(mine)
        self.local_cfg = mine
        self.d_cfg = torch.from_numpy(mine.view(np.uint8).copy()).to(self.dev) if self.n_local else None
        # this rank's records [g][j], padded at the tail to H * m (padding: status = WS_EINVAL)
        self.d_out = torch.zeros((self.H * self.m, RECORD_BYTES), dtype=torch.uint8, device=self.dev)
        self.d_out[self.H * self.n_local:, 0] = 1
        on_host = self.backend == "gloo"
        gdev = torch.device("cpu") if on_host else self.dev
        self.gathered = torch.empty((self.world * self.H * self.m, RECORD_BYTES), dtype=torch.uint8, device=gdev)
        self.h_out = torch.empty((self.H * self.m, RECORD_BYTES), dtype=torch.uint8) if on_host else None
        # canonical position g * n + i  <-  gathered row r * H * m + g * n_r + j (shards[r][j] = i)
        src = np.empty(self.H * self.n, dtype=np.int64)
        for r, s in enumerate(self.shards):
            nr = len(s)
            for j, i in enumerate(s):
                src[np.arange(self.H) * self.n + i] = r * self.H * self.m + np.arange(self.H) * nr + j
        self.perm = torch.from_numpy(src).to(gdev)
        self.result = torch.empty((self.H * self.n, RECORD_BYTES), dtype=torch.uint8, device=self.dev)
        self.top = torch.empty(max(1, k_top), dtype=torch.int32, device=self.dev)
        self.estimate = estimate
        self.est_launches, self.est_groups = 0, 0

    def step(self):
        if self.n_local:
            if self.estimate is not None:
                self.estimate(self.local_cfg, self.d_out[: self.H * self.n_local])
            else:
                self.ctx.estimate_multi_async(self.d_cfg.data_ptr(), self.n_local, self.gpu_ids, self.d_out.data_ptr())
                self.est_launches = self.ctx.last_launch_count()
                self.est_groups = self.ctx.last_group_count()
        nvtx = torch.cuda.nvtx if self.dev.type == "cuda" else None
        if nvtx:
            nvtx.range_push("ShardedSweep.gather")
        if self.world == 1:
            torch.index_select(self.d_out, 0, self.perm, out=self.result)
        elif self.backend == "nccl":
            dist.all_gather_into_tensor(self.gathered, self.d_out, group=self.group)
            torch.index_select(self.gathered, 0, self.perm, out=self.result)
        else:
            self.h_out.copy_(self.d_out)
            dist.all_gather_into_tensor(self.gathered, self.h_out, group=self.group)
            self.result.copy_(torch.index_select(self.gathered, 0, self.perm))
        if nvtx:
            nvtx.range_pop()
        if self.ctx is not None:
            self.ctx.rank_async(self.result.data_ptr(), self.H * self.n, self.k_top, self.top.data_ptr())
        return self.result


def estimate_sharded(ctx, cfg_records, group=None, k_top: int = 10, costs=None):
    """One sweep of a batch of ws_config records over the ranks of `group` (each record with its
    own gpu_id): returns (results uint8 tensor (n, 336) on this rank's GPU, top-k indices)."""
    cfgs = [((int(c["block"][0]), int(c["block"][1]), int(c["block"][2])),
             (int(c["fold"][0]), int(c["fold"][1]), int(c["fold"][2])), int(c["blocks_per_sm"]))
            for c in cfg_records]
    costs = costs if costs is not None else [proxy_cost(c) for c in cfgs]
    gids = np.unique(cfg_records["gpu_id"])
    if len(gids) != 1:
        raise ValueError("estimate_sharded: one gpu_id per batch (use ShardedSweep for several)")
    sw = ShardedSweep(ctx, cfg_records, [int(gids[0])], costs, group=group, k_top=k_top)
    res = sw.step()
    return res, sw.top[: min(k_top, len(cfg_records))]
