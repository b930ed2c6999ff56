#!/usr/bin/env python3
"""bench.py -- configs estimated/s of the B200-native Warpspeed hot path.

Workload (BASELINE.json configs[1]): range-4 3D-25pt double stencil on 512^3,
the paper's full block-shape x thread-folding space (56 shapes x {none, 2y, 2z}
= 168 configurations), A100 parameters with the split-L2 halving.
One step = the whole hot path (a1-a8: plan, warp-instruction, SM-set, wave and
layer-set scopes, model, ranking) over that batch.  At N GPUs every rank
evaluates the same 168-config space on its own hardware parameter set
(architecture exploration, BJ configs[3]: rank 0 = A100, then B200-like, V100
and a hypothetical grid), the results are all-gathered over NCCL and every rank
ranks the gathered set: per-GPU work is fixed -> "scaling": "weak".  The same run
also measures BJ configs[3] with a fixed total (`configs3_strong`: 217 configs x 51
hardware sets sharded by configuration over the ranks, one all-gather).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]

`--gpus N` without a launcher starts N ranks itself (torch.distributed.run, one per
GPU); under a launcher WORLD_SIZE must equal N.  Rank 0 prints one JSON line.
`--impl reference` times the plain CPU oracle (oracle/) on the host cores instead
(this tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "configs estimated/sec (8×B200, device-timed) + bit-exact volume match vs CPU"
UNIT = "configs/s"
WORKLOAD = ("BJ configs[1]: 3D-25pt r4 double stencil, grid 512^3, 168 configs "
            "(56 block shapes x {none,2y,2z} folding), A100 parameters (split L2)")
TOPK = 10
# algorithmic integer lane-ops per work unit
OPS_PER_UNIT = {"k_warp": 12, "k_wclass": 12, "k_smset": 16, "k_sclass": 16, "k_rows": 1, "k_plan": 8}


def peaks():
    p = {}
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    return p


def alu_peak_gops(sm_max_mhz):
    """Issue-limited integer lane-op peak: 148 SMs x 4 SMSPs x 1 warp-instruction/clk x 32 lanes."""
    return 148 * 4 * 32 * sm_max_mhz * 1e6 / 1e9


def hw_sets(world):
    pk = peaks()
    sets = [W.gpu_a100(), W.gpu_b200_like(pk.get("hbm_gbs", 6546.2)), W.gpu_v100()]
    for l1 in (128, 256):
        for l2 in (20, 40, 64):
            for nsm in (108, 148):
                sets.append(W.gpu_hypothetical(l1, l2, nsm))
    while len(sets) < world:
        sets.append(W.gpu_hypothetical(192, 32 + len(sets), 132))
    return sets[:max(1, world)]


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.rows, self.proc, self.t = device, [], None, None
        self.marks = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def mark(self, tag):
        self.marks.append((tag, time.time()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()
        if self.t:
            self.t.join(2)

    def summary(self, t0, t1):
        inside = [r for t, r in self.rows if t0 <= t <= t1]
        note = "samples inside the timed region"
        if len(inside) < 3:
            inside = [r for _, r in self.rows]
            note = "timed region shorter than the sampling interval: samples over warm-up + timed region"
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "note": "nvidia-smi unavailable"}
        sm = [float(r[0]) for r in inside if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in inside if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in inside for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside), "note": note}


# ------------------------------------------------------------------ CPU oracle (baseline / reference arm)
def host_info():
    """CPU model, logical CPUs and RAM of the host the oracle runs on."""
    model, mem = "unknown", 0
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
        mem = int(open("/proc/meminfo").readline().split()[1]) // (1024 * 1024)
    except OSError:
        pass
    return {"cpu": model, "nproc": os.cpu_count(), "ram_gib": mem}


def stratified_sample(plans, cfgs, max_evals=1.0e8, stride=6):
    """Configurations spread over the space's cost distribution: every `stride`-th configuration
    in cost order among those the oracle finishes in about half a minute (<= max_evals address
    evaluations, one host thread each) -- shallow and deep blocks, folded and unfolded."""
    order = sorted(range(len(cfgs)), key=lambda i: plans[i]["addr_evals"])
    ok = [i for i in order if plans[i]["status"] == 0 and plans[i]["addr_evals"] <= max_evals]
    return [cfgs[i] for i in ok[::stride]]


def full_space_timing():
    """The measured single-thread oracle seconds of every configuration of configs[1] (written by
    scripts/oracle_golden.py when it generated tests/golden/full_c1_k25_512_a100.json)."""
    try:
        doc = json.load(open(os.path.join(ROOT, "tests", "golden", "full_c1_k25_512_a100.json")))
    except Exception:
        return None
    sec = doc.get("oracle_seconds") or []
    if not sec:
        return None
    tot = sum(sec)
    return {"configs": len(sec), "thread_seconds": tot, "configs_per_s_one_thread": len(sec) / tot,
            "max_config_s": max(sec), "host": doc.get("host"),
            "note": "measured: every configuration of the space once, one host thread each "
                    "(scripts/oracle_golden.py), on the host named here (not the GPU box)"}


def oracle_sample(kernel, gpu, cfgs, threads):
    """The plain CPU oracle on a bounded, stratified sample of the workload on all host threads,
    extrapolated to configs/s of the whole space by the oracle's own work measure (addr_evals,
    the plain definition's address evaluations): value = evals/s / mean evals per configuration."""
    from oracle import oracle as O
    plans = [O.plan(kernel, gpu, c) for c in cfgs]
    mean_evals = statistics.mean(p["addr_evals"] for p in plans if p["status"] == 0)
    sample = stratified_sample(plans, cfgs)
    t0 = time.perf_counter()
    res = O.estimate_batch(kernel, gpu, sample, threads)
    dt = time.perf_counter() - t0
    ev = sum(r["addr_evals"] for r in res)
    rate = ev / dt
    out = {"value": rate / mean_evals, "unit": UNIT, "cores": min(threads, len(sample)), "kind": "oracle",
           "estimated": True,
           "sample": (f"{len(sample)} of {len(cfgs)} configs (stratified over the cost distribution, <= 1e8 "
                      f"address evaluations each) on {min(threads, len(sample))} host threads: {dt:.2f} s wall, "
                      f"{ev:.3e} address evaluations -> {rate:.3e} evals/s, extrapolated by the space's mean "
                      f"{mean_evals:.3e} evals/config"),
           "sample_configs_per_s": len(sample) / dt, "evals_per_s": rate, "wall_s": dt, "host": host_info()}
    fs = full_space_timing()
    if fs is not None:
        out["full_space_measured"] = fs
    return out


def run_reference(args, rank, world):
    """The reference arm: the plain CPU oracle as it stands, on the host cores, on this arm's
    configuration and metric.  Each step: one configuration per host thread, taken in turn from
    the stratified sample of the space (cycled), timed; value = address evaluations per second
    over the steps / the space's mean evaluations per configuration."""
    if rank != 0:
        return
    kernel, gpu, cfgs = W.k25(512), W.gpu_a100(), W.space_stencil_paper()
    threads = os.cpu_count() or 1
    from oracle import oracle as O
    O.build()
    plans = [O.plan(kernel, gpu, c) for c in cfgs]
    mean_evals = statistics.mean(p["addr_evals"] for p in plans if p["status"] == 0)
    # a step is bounded: configurations of <= 3e7 evaluations (~10 s on one thread)
    sample = stratified_sample(plans, cfgs, max_evals=3e7, stride=2)
    pos = 0

    def take():
        nonlocal pos
        out = [sample[(pos + j) % len(sample)] for j in range(threads)]
        pos += threads
        return out

    for _ in range(max(0, args.warmup)):
        O.estimate_batch(kernel, gpu, take()[:1], 1)
    tot_dt, tot_ev, tot_n = 0.0, 0, 0
    for _ in range(args.steps):
        batch = take()
        t0 = time.perf_counter()
        res = O.estimate_batch(kernel, gpu, batch, threads)
        tot_dt += time.perf_counter() - t0
        tot_ev += sum(r["addr_evals"] for r in res)
        tot_n += len(batch)
    rate = tot_ev / tot_dt
    value = rate / mean_evals
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic", "config": {"workload": WORKLOAD, "global_batch": len(cfgs), "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "estimated": True,
                         "host": host_info(),
                         "sample": (f"each step: {threads} configs (one per host thread) cycled from a stratified "
                                    f"sample of {len(sample)} of the 168 (<= 3e7 evaluations each); throughput "
                                    f"{rate:.3e} address evals/s extrapolated by the space's mean {mean_evals:.3e} "
                                    f"evals/config")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    fs = full_space_timing()
    if fs is not None:
        line["cpu_baseline"]["full_space_measured"] = fs
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ native arm
def run_native(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2204_14242_b200 import Context, config_array, result_dicts
    from paper_2204_14242_b200.ws import RESULT_DTYPE

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()
    ctx = Context(local, stream.cuda_stream)
    kernel = W.k25(512)
    gpu = hw_sets(world)[rank]
    space = W.space_stencil_paper()
    kid, gid = ctx.describe_kernel(kernel), ctx.describe_gpu(gpu)
    host_cfg = config_array(kid, gid, space)
    n = len(host_cfg)
    rb = RESULT_DTYPE.itemsize
    d_cfg = torch.from_numpy(host_cfg.view(np.uint8).copy()).to(dev)
    d_out = torch.empty(n * rb, dtype=torch.uint8, device=dev)
    gathered = torch.empty(world * n * rb, dtype=torch.uint8, device=dev) if world > 1 else d_out
    d_top = torch.empty(TOPK, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    # rank r evaluates the space on hardware set r: the gathered buffer [r][i] is already in
    # canonical order (equal shards), so a step is estimate -> one all-gather -> rank
    # one rank: ws_estimate_ranked_async (the model and the ranking fused into the chain's last
    # kernel); several: estimate -> all-gather -> rank of the gathered set
    def step():
        if world == 1:
            ctx.estimate_ranked_async(d_cfg.data_ptr(), n, d_out.data_ptr(), TOPK, d_top.data_ptr())
            return
        ctx.estimate_async(d_cfg.data_ptr(), n, d_out.data_ptr())
        dist.all_gather_into_tensor(gathered, d_out)
        ctx.rank_async(gathered.data_ptr(), world * n, TOPK, d_top.data_ptr())

    launches_per_step = None
    for _ in range(max(args.warmup, 0)):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    if world == 1:
        step()
        launches_per_step = ctx.last_launch_count()
    else:
        ctx.estimate_async(d_cfg.data_ptr(), n, d_out.data_ptr())
        launches_per_step = ctx.last_launch_count() + 1
    work = ctx.work_read()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_wall0 = time.time()
    for i in range(args.steps):
        flush.zero_()                       # L2 flushed between timed steps (outside the events)
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.time()
    if world > 1:
        dist.barrier()
    ms_total = sum(a.elapsed_time(b) for a, b in evs)
    # per-kernel durations (CUDA events on each kernel's own stream) from a separate pass of
    # the same steps: event recording disables the graph replay of the timed loop
    ctx.profile_enable(True)
    for i in range(args.steps):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    ctx.profile_enable(False)
    prof = ctx.profile_read()
    time.sleep(0.2)
    sampler.stop()
    clocks = sampler.summary(t_wall0, t_wall1)
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * n * args.steps / (ms_max / 1e3)

    # correctness guard on the timed output (no silently empty work)
    res = np.frombuffer(gathered.cpu().numpy().tobytes(), dtype=RESULT_DTYPE)
    assert (res["status"] == 0).all() and (res["lup_wave"] > 0).all()
    addr_evals = int(res["addr_evals"][:n].sum())

    # ---- e2e through the public API with host buffers
    e2e = e2e_measure(ctx, host_cfg, n, world, dev, stream, args, rb)

    # ---- roofline: k_rows (the kernel VERDICT r01 names; the row chain's critical path), and
    # the executed issue rate of every kernel against the MEASURED integer issue peak
    kern = {k: v for k, v in prof.items() if v[1] > 0}
    dom = "k_rows" if "k_rows" in kern else max(kern, key=lambda k: kern[k][0])
    longest = max(kern, key=lambda k: kern[k][0] / kern[k][1])
    dom_ms = kern[dom][0] / kern[dom][1]
    pk = peaks()
    sm_max = pk.get("sm_max_mhz", 1965.0)
    ipk = {}
    try:
        ipk = json.load(open(os.path.join(ROOT, "profiles", "r02_int_peak.json")))
    except Exception:
        pass
    issue_peak_nominal = 148 * 4 * sm_max * 1e6
    issue_peak = ipk.get("issue_peak_measured_warp_inst_per_s") or issue_peak_nominal
    peak = issue_peak * 32 / 1e9          # lane-ops/s (Gop/s)
    peak_note = (f"measured: {issue_peak:.4g} warp-instructions/s x 32 lanes (profiles/r02_int_peak.json, "
                 f"scripts/int_peak.cu: integer ALU+FMA+SHFL mix at {ipk.get('issue_active_pct_mix_shfl', 0):.0f} % "
                 f"issue-active; nominal 148 SMs x 4 SMSPs x 1/clk x {sm_max:.0f} MHz = {issue_peak_nominal:.4g})"
                 if ipk else f"nominal: 148 SMs x 4 SMSP x 32 lanes x {sm_max:.0f} MHz (issue-limited int lane-ops)")
    units = work.get(dom, 0)
    ops = units * OPS_PER_UNIT.get(dom, 0)
    achieved = ops / (dom_ms / 1e3) / 1e9 if dom_ms > 0 else 0.0
    nt = {}
    try:
        nt = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except Exception:
        pass
    traffic = nt.get(dom)
    share = {k: round(v[0] / sum(x[0] for x in kern.values()), 4) for k, v in kern.items()}
    # executed instruction mix (with row spans the roofline is recomputed for the
    # executed mix): the committed ncu capture's warp instructions per launch over the kernel's
    # live launch time in this run, against the measured issue peak
    warp_inst = nt.get(dom + ":warp_inst")
    executed = ({"warp_inst_per_launch": warp_inst, "issue_rate_per_s": warp_inst / (dom_ms / 1e3),
                 "issue_peak_per_s": issue_peak, "issue_frac": warp_inst / (dom_ms / 1e3) / issue_peak,
                 "source": "profiles/ncu_traffic.json (ncu --set full, smsp__inst_executed.sum)"}
                if warp_inst and dom_ms > 0 else None)
    # a profile bucket (CUDA events around a group of launches) against the warp instructions of
    # every kernel in it
    bucket = {"k_smset": ["k_scan", "k_spairs", "k_smset"],
              "k_sclass": ["k_cplan", "k_cplanes", "k_cfold", "k_sclass", "k_sshare"]}
    def bucket_inst(k):
        parts = [nt.get(x + ":warp_inst") for x in bucket.get(k, [k])]
        return sum(x for x in parts if x) if any(parts) else None
    issue_by_kernel = {k: round(bucket_inst(k) / (v[0] / v[1] / 1e3) / issue_peak, 4)
                       for k, v in kern.items() if bucket_inst(k) and v[0] > 0}

    strong = configs3_strong_measure(ctx, stream, args, rank, world, dev)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(kernel, gpu, space, os.cpu_count() or 1)
    nxt = None
    if rank == 0 and not args.no_next:
        nxt = next_rows_measure(ctx, stream, args, world == 1 and not args.no_cpu_baseline)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (analytic kernel descriptions shaped like the paper's; no datasets or weights)",
            "config": {"workload": WORKLOAD, "global_batch": world * n, "per_gpu_batch": n,
                       "hardware_sets": [hw_sets(world)[r]["name"] for r in range(world)],
                       "parallelism": f"dp{world} over configurations (one NCCL all-gather of results)",
                       "l2": "flushed between timed steps (256 MiB write, outside the events)"},
            "addresses_per_s_equiv": world * addr_evals * args.steps / (ms_max / 1e3),
            "roofline": {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "Gop/s",
                         "frac": achieved / peak if peak else None, "traffic": traffic,
                         "units_per_launch": units, "ops_per_unit": OPS_PER_UNIT.get(dom),
                         "avg_launch_ms": dom_ms,
                         "peak_note": peak_note, "executed": executed,
                         "kernel_choice": "k_rows: the kernel VERDICT r01 names (row chain, critical path); "
                                          f"longest average launch this run: {longest}",
                         "issue_frac_by_kernel": issue_by_kernel},
            "kernel_ms_per_step": {k: v[0] / args.steps for k, v in kern.items()},
            "kernel_share": share,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if nxt is not None:
            line["next_rows"] = nxt
        line["configs3_strong"] = strong
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def configs3_strong_measure(ctx, stream, args, rank, world, dev):
    """BJ configs[3] with a fixed total (strong scaling): configs[1] u configs[2] (the 168-config
    3D-25pt 512^3 space and the 49 LBM15 256^3 configurations) x the 51 configs[3] hardware sets
    (V100, A100, B200-like, 48 hypothetical; workloads.hw_grid_configs3) = 11067 (configuration,
    hardware set) estimates, sharded by configuration over the ranks (LPT on device-derived per-configuration
    costs computed on rank 0 and broadcast), ws_estimate_multi per rank (integer stages once per
    SM-count group, model fanned out), one all-gather, the canonical permutation, ws_rank of the
    whole set on every rank.  Timed like the headline: barrier + synchronize around K steps,
    CUDA events on the context stream, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2204_14242_b200 import config_array, dist as D
    sets = W.hw_grid_configs3(peaks().get("hbm_gbs", 6546.2))
    import numpy as np
    k25, klbm = ctx.describe_kernel(W.k25(512)), ctx.describe_kernel(W.lbm15(256))
    gids = [ctx.describe_gpu(g) for g in sets]
    cf = np.concatenate([config_array(k25, 0, W.space_stencil_paper()), config_array(klbm, 0, W.space_lbm())])
    costs = [D.device_costs(ctx, cf, gids) if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(costs, src=0)
    sw = D.ShardedSweep(ctx, cf, gids, costs[0], device=dev)
    for _ in range(max(3, args.warmup)):
        sw.step()
    torch.cuda.synchronize()
    groups, launches = sw.est_groups, sw.est_launches
    steps = max(20, min(args.steps, 200))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        sw.step()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / steps
    total = len(cf) * len(gids)
    import numpy as np
    from paper_2204_14242_b200.ws import RESULT_DTYPE
    res = np.frombuffer(sw.result.cpu().numpy().tobytes(), dtype=RESULT_DTYPE)
    assert (res["status"] == 0).all() and len(res) == total
    loads = [sum(costs[0][i] for i in s) for s in sw.shards]
    return {"workload": f"BJ configs[3]: (3D-25pt r4 512^3, 168 configs) u (LBM15 256^3, 49 configs) x {len(gids)} "
                        "hardware sets (V100, A100, B200-like + hypothetical grid L1 x L2 x SM count), fixed total",
            "value": total / (ms / 1e3), "unit": "configs/s", "metric_unit_note": "one config = one (configuration, "
            "hardware set) estimate", "n_gpus": world, "scaling": "strong", "steps": steps, "ms_per_step": ms,
            "integer_groups_per_rank": groups, "gpu_launches_per_step": launches + 1,
            "shard_sizes": [len(s) for s in sw.shards],
            "shard_cost_imbalance": max(loads) / (sum(loads) / len(loads)) if loads else None,
            "timing": "barrier + synchronize around the K steps, CUDA events on the context stream, max over ranks; "
                      "no L2 flush (working set of a step is re-read from HBM-resident descriptors)"}


def next_rows_measure(ctx, stream, args, cpu_baseline):
    """SURVEY 8(f) rows beyond the headline path, measured on the same context (rank 0):
    NEXT-3/4 -- the 168-config 512^3 space with every WS_VAR_* bit and the outlook metrics on
    (B200-like parameters: TLB pages, section link); NEXT-1 -- LRU-simulated hit-rate samples
    (ws_simulate) of the 168-config space at 40^3 x 8 capacities, device-timed per kernel, with
    the plain CPU oracle timed on one configuration of it."""
    import numpy as np
    import torch
    from paper_2204_14242_b200 import config_array
    out = {}
    # ---- NEXT-3/4: variants + outlook metrics through the same estimate path
    k, g = W.k25(512), W.with_outlook(W.gpu_b200_like(peaks().get("hbm_gbs", 6546.2)))
    kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(g)
    cf = config_array(kid, gid, [c + (7,) for c in W.space_stencil_paper()])
    n = len(cf)
    d_cfg = torch.from_numpy(cf.view(np.uint8).copy()).cuda()
    d_out = torch.empty(n * 336, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ctx.estimate_async(d_cfg.data_ptr(), n, d_out.data_ptr())
    torch.cuda.synchronize()
    steps = max(10, min(args.steps, 100))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        ctx.estimate_async(d_cfg.data_ptr(), n, d_out.data_ptr())
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ctx.profile_enable(True)
    ctx.estimate_async(d_cfg.data_ptr(), n, d_out.data_ptr())
    torch.cuda.synchronize()
    ctx.profile_enable(False)
    sect_ms = ctx.profile_read().get("k_sect", (0.0, 0))[0]
    out["next3_4_variants"] = {
        "workload": "3D-25pt r4 512^3, 168 configs, variant bits 7 (multidimensional space + previous-wave reuse "
                    "+ duplication-based L2 capacity), B200-like parameters with 2 MiB pages and a 10 TB/s "
                    "section link (k_sect active)",
        "value": n / (ms / 1e3), "unit": "configs/s", "ms_per_step": ms, "k_sect_ms": sect_ms,
        "data": "synthetic", "timing": "CUDA events on the context stream, graph replay, no L2 flush"}
    # ---- the extended throughput space: 1890 configs (power-of-two shapes with
    # 64..1024 threads x (fy, fz) in {1,2,4}^2) of the same 512^3 stencil, A100 parameters
    k, g = W.k25(512), W.gpu_a100()
    kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(g)
    cf = config_array(kid, gid, W.space_extended())
    n = len(cf)
    d_cfg = torch.from_numpy(cf.view(np.uint8).copy()).cuda()
    d_out = torch.empty(n * 336, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        ctx.estimate_async(d_cfg.data_ptr(), n, d_out.data_ptr())
    torch.cuda.synchronize()
    steps_x = 10
    e0.record(stream)
    for _ in range(steps_x):
        ctx.estimate_async(d_cfg.data_ptr(), n, d_out.data_ptr())
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps_x
    out["extended_space"] = {"workload": f"3D-25pt r4 512^3, extended space (SURVEY Q34), {n} configs, A100 parameters",
                             "value": n / (ms / 1e3), "unit": "configs/s", "ms_per_step": ms, "data": "synthetic",
                             "timing": "CUDA events on the context stream, graph replay, no L2 flush"}
    # ---- BJ configs[2]: the LBM kernels (LBM15 = the paper's D3Q15 + phase field, LBM27 = D3Q27
    # with the D3Q27 phase-field stencil), 256^3, the 49 shapes of 512 threads, A100 parameters
    for name, kk in (("configs2_lbm15", W.lbm15(256)), ("configs2_lbm27", W.lbm27(256))):
        kid, gid = ctx.describe_kernel(kk), ctx.describe_gpu(W.gpu_a100())
        cf = config_array(kid, gid, W.space_lbm())
        n = len(cf)
        d_cfg = torch.from_numpy(cf.view(np.uint8).copy()).cuda()
        d_out = torch.empty(n * 336, dtype=torch.uint8, device="cuda")
        for _ in range(2):
            ctx.estimate_async(d_cfg.data_ptr(), n, d_out.data_ptr())
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(20):
            ctx.estimate_async(d_cfg.data_ptr(), n, d_out.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        out[name] = {"workload": f"{name[9:].upper()} 256^3, 49 configs (P:730), A100 parameters", "value": n / (ms / 1e3),
                     "unit": "configs/s", "ms_per_step": ms, "data": "synthetic",
                     "timing": "CUDA events on the context stream, graph replay, no L2 flush"}
    # ---- NEXT-1: simulated hit-rate samples
    k, g = W.k25(128), W.gpu_a100()
    kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(g)
    space = W.space_stencil_paper()
    cf = config_array(kid, gid, space)
    caps = [int(g["l2_bytes"] // 2 * 2 ** (e / 2)) for e in range(-24, 8)][::2]
    ctx.simulate(cf, caps)                          # warm-up: the grow-only buffers reach full size
    ctx.profile_enable(True)
    reps = 3
    t0 = time.perf_counter()
    for _ in range(reps):
        rows = ctx.simulate(cf, caps)
    wall = (time.perf_counter() - t0) / reps
    ctx.profile_enable(False)
    prof = ctx.profile_read()
    dev_ms = (prof.get("k_simgen", (0, 0))[0] + prof.get("k_simrun", (0, 0))[0]) / reps
    req = sum(r[0]["l1_requests"] + r[0]["st_requests"] for r in rows)
    sim = {"workload": f"3D-25pt r4 128^3, 168 configs x {len(caps)} capacities (A100 L2/2 x 2^-12..2^3), "
                       "L1 / store / layer-set streams", "value": len(space) * len(caps) / (wall), "unit": "samples/s",
           "wall_ms_per_call": wall * 1e3, "device_ms_per_call": dev_ms,
           "kernel_ms_per_call": {k: v[0] / reps for k, v in prof.items() if v[1]},
           "l1_plus_store_requests": req, "data": "synthetic",
           "timing": "wall clock around the synchronous ws_simulate (includes the host sizing; buffers kept from "
                     "a full-size warm-up call); device ms from CUDA events on the stream"}
    if cpu_baseline:
        from oracle import oracle as O
        one = [c for c in space if c[0] in ((1024, 1, 1), (512, 2, 1)) and c[1] == (1, 1, 1)]
        t0 = time.perf_counter()
        O.simulate_batch(k, g, one, caps, 2)
        dt = time.perf_counter() - t0
        sim["cpu_baseline"] = {"value": len(one) * len(caps) / dt, "unit": "samples/s", "cores": 2, "kind": "oracle",
                               "sample": f"{len(one)} of the 168 configs x {len(caps)} capacities on 2 host threads "
                                         f"({dt:.1f} s): direct LRU simulation per capacity"}
    out["next1_simulate"] = sim
    return out


def e2e_measure(ctx, host_cfg, n, world, dev, stream, args, rb):
    """Same metric end to end: pinned host configs -> device -> whole path -> results + top-k
    back in pinned host memory, every step."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2204_14242_b200.ws import RESULT_DTYPE
    h_cfg = torch.from_numpy(host_cfg.view(np.uint8).copy()).pin_memory()
    h_res = torch.empty(world * n * rb, dtype=torch.uint8).pin_memory()
    h_top = torch.empty(TOPK, dtype=torch.int32).pin_memory()
    d_cfg = torch.empty_like(h_cfg, device=dev)
    d_out = torch.empty(n * rb, dtype=torch.uint8, device=dev)
    gathered = torch.empty(world * n * rb, dtype=torch.uint8, device=dev) if world > 1 else d_out
    d_top = torch.empty(TOPK, dtype=torch.int32, device=dev)

    def one():
        d_cfg.copy_(h_cfg, non_blocking=True)
        if world == 1:
            ctx.estimate_ranked_async(d_cfg.data_ptr(), n, d_out.data_ptr(), TOPK, d_top.data_ptr())
        else:
            ctx.estimate_async(d_cfg.data_ptr(), n, d_out.data_ptr())
            dist.all_gather_into_tensor(gathered, d_out)
            ctx.rank_async(gathered.data_ptr(), world * n, TOPK, d_top.data_ptr())
        h_res.copy_(gathered, non_blocking=True)
        h_top.copy_(d_top, non_blocking=True)
        stream.synchronize()

    for _ in range(max(1, args.warmup)):
        one()
    # one rank: two steps in flight (double-buffered pinned result buffers): step i+1 is enqueued
    # (H2D, ranked estimate, D2H) before the host waits for step i's results and reads them, so the
    # device does not idle through the host's synchronisation; every step still copies its
    # configurations in and its records + top-k out, and the host reads each step's top-1
    pipelined = world == 1
    if pipelined:
        hb = [(h_res, h_top), (torch.empty_like(h_res).pin_memory(), torch.empty_like(h_top).pin_memory())]
        evs = [torch.cuda.Event(), torch.cuda.Event()]
        tops = []

        def enqueue(b):
            d_cfg.copy_(h_cfg, non_blocking=True)
            ctx.estimate_ranked_async(d_cfg.data_ptr(), n, d_out.data_ptr(), TOPK, d_top.data_ptr())
            hb[b][0].copy_(d_out, non_blocking=True)
            hb[b][1].copy_(d_top, non_blocking=True)
            evs[b].record(stream)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    if pipelined:
        for i in range(args.steps):
            enqueue(i & 1)
            if i >= 1:
                evs[(i - 1) & 1].synchronize()
                tops.append(int(hb[(i - 1) & 1][1][0]))
        evs[(args.steps - 1) & 1].synchronize()
        tops.append(int(hb[(args.steps - 1) & 1][1][0]))
    else:
        for _ in range(args.steps):
            one()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    res = np.frombuffer(h_res.numpy().tobytes(), dtype=RESULT_DTYPE)
    assert (res["status"] == 0).all()
    if pipelined:   # every step's top-1 read on the host, and the records of both buffers agree
        assert len(tops) == args.steps and len(set(tops)) == 1
        assert hb[1][0].numpy().tobytes() == h_res.numpy().tobytes()
    return {"value": world * n * args.steps / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": int(h_cfg.numel()), "d2h_bytes_per_step": int(h_res.numel() + h_top.numel() * 4),
            "api": ("pinned host configs -> ws_estimate_ranked_async -> pinned host results (two steps in flight, "
                    "double-buffered results; the host reads every step's top-1)" if world == 1 else
                    "pinned host configs -> ws_estimate_async -> all-gather -> ws_rank_async -> pinned host results")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # native: 1500 timed steps (>= ~0.3 s: clock samples inside the timed region); reference
    # arm (the slow CPU oracle, seconds per step): 3 unless given
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-next", action="store_true", help="skip the NEXT-1/3/4 measurements")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 3 if args.impl == "reference" else 1500
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without a launcher: start N ranks (one per GPU) ourselves
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: the launcher and the flag disagree")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_native(args, rank, world, local)


if __name__ == "__main__":
    main()
