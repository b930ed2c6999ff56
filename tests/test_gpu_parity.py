"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by element,
on the same seeded inputs (integers bit-exact, doubles within 1e-9 relative)."""
import os
import random

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O
from parity_util import check_ranking, compare

pytestmark = pytest.mark.gpu

NT = max(1, min(32, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2204_14242_b200 import Context
    return Context(0)


def run_gpu(ctx, kernel, gpu, configs):
    from paper_2204_14242_b200 import config_array, result_dicts
    kid = ctx.describe_kernel(kernel)
    gid = ctx.describe_gpu(gpu)
    res = ctx.estimate(config_array(kid, gid, configs))
    return result_dicts(res), res


def assert_parity(ctx, kernel, gpu, configs, label):
    g, _ = run_gpu(ctx, kernel, gpu, configs)
    o = O.estimate_batch(kernel, gpu, configs, NT)
    errs = []
    for i, (a, b) in enumerate(zip(g, o)):
        errs += compare(a, b, f"{label}[{i}] {configs[i]}")
    assert not errs, "\n".join(errs[:40])
    return g, o


def test_configs0_k7_v100(ctx):
    """BJ configs[0]: 7pt 64^3, 16 shapes on V100 (incl. the invalid 2048-thread block)."""
    g, o = assert_parity(ctx, W.k7(64), W.gpu_v100(), W.space_k7(), "cfg0")
    assert sum(r["status"] != 0 for r in g) == 1


def test_small_cases(ctx):
    cases = [
        (W.k7(12), W.gpu_v100(), [((32, 2, 1), (1, 1, 1), 0), ((32, 8, 8), (1, 1, 1), 0)]),
        (W.stencil_star(20, 10, 12, 4, regs=64), dict(W.gpu_a100(), n_sm=6),
         [((8, 4, 2), (1, 1, 2), 1), ((4, 2, 4), (1, 2, 1), 2), ((1, 1, 1), (1, 1, 1), 1)]),
        (W.lbm15(6), dict(W.gpu_a100(), n_sm=3), [((4, 2, 2), (1, 1, 1), 1), ((2, 2, 2), (2, 1, 1), 0)]),
    ]
    for i, (k, gp, cf) in enumerate(cases):
        assert_parity(ctx, k, gp, cf, f"small{i}")


def test_stencil25_paper_space_64(ctx):
    """Full 168-config paper space on a 64^3 grid, A100 parameters."""
    assert_parity(ctx, W.k25(64), W.gpu_a100(), W.space_stencil_paper(), "k25_64")


def test_stencil25_ragged(ctx):
    """Ragged domain (not divisible by any block), several tiles and a tail."""
    k = W.stencil_star(75, 37, 29, 4, regs=64)
    g = dict(W.gpu_a100(), n_sm=20)
    cf = [((32, 4, 2), (1, 1, 1), 0), ((16, 2, 8), (1, 1, 2), 0), ((64, 1, 4), (1, 2, 1), 0),
          ((1, 16, 4), (1, 1, 1), 0), ((128, 2, 1), (1, 1, 1), 0), ((1024, 1, 1), (1, 1, 1), 0)]
    assert_parity(ctx, k, g, cf, "ragged")


def test_lbm_spaces_small(ctx):
    """LBM15 / LBM27 (Q23) on 40^3 with 16 SMs: 49 shapes."""
    g = dict(W.gpu_a100(), n_sm=16)
    assert_parity(ctx, W.lbm15(40), g, W.space_lbm(), "lbm15")
    sub = W.space_lbm()[::4]
    assert_parity(ctx, W.lbm27(24), dict(W.gpu_a100(), n_sm=8), sub, "lbm27")


@pytest.mark.parametrize("seed", range(40))
def test_random_kernels(ctx, seed):
    k, gp = W.random_kernel(seed), W.random_gpu(seed)
    rng = random.Random(seed)
    cf = [W.random_config(seed * 10 + j) for j in range(4)]
    assert_parity(ctx, k, gp, cf, f"rand{seed}")


def test_edge_cases(ctx):
    # single block grid: wave = whole grid, empty layer sets
    k = W.stencil_star(8, 8, 8, 1, regs=0)
    assert_parity(ctx, k, W.gpu_v100(), [((8, 8, 8), (1, 1, 1), 0), ((16, 16, 4), (1, 1, 2), 0)], "single")
    # negative alignment (P:540 uses -1 element), 4- and 16-byte elements
    k2 = W.stencil_star(16, 8, 8, 1, regs=0)
    k2["fields"][0] = dict(k2["fields"][0], align=-8)
    k2["fields"][1] = dict(k2["fields"][1], align=-120, elem=8)
    assert_parity(ctx, k2, dict(W.gpu_v100(), n_sm=4), [((8, 2, 2), (1, 1, 1), 0), ((4, 4, 1), (2, 1, 1), 1)], "neg")
    k3 = W.stencil_star(16, 8, 8, 1, regs=0)
    k3["fields"][0] = dict(k3["fields"][0], elem=4, align=4)
    k3["fields"][1] = dict(k3["fields"][1], elem=16, align=16)
    assert_parity(ctx, k3, dict(W.gpu_v100(), n_sm=4), [((8, 2, 2), (1, 1, 1), 0), ((32, 1, 1), (1, 1, 1), 1)], "elem")
    # per-config errors: zero block, fold cube > 64, T > max threads, k override
    assert_parity(ctx, k, W.gpu_v100(),
                  [((0, 1, 1), (1, 1, 1), 0), ((8, 8, 8), (8, 8, 2), 0), ((64, 32, 1), (1, 1, 1), 0),
                   ((8, 1, 1), (1, 1, 1), 3)], "errors")


def test_unknown_ids_and_empty_batch(ctx):
    from paper_2204_14242_b200 import config_array, result_dicts
    kid = ctx.describe_kernel(W.k7(8))
    gid = ctx.describe_gpu(W.gpu_v100())
    a = config_array(kid, gid, [((32, 1, 1), (1, 1, 1), 0)] * 2)
    a[1]["kernel_id"] = 999
    r = result_dicts(ctx.estimate(a))
    assert r[0]["status"] == 0 and r[1]["status"] == 6 and r[1]["t_pred"] == 0.0
    assert len(ctx.estimate(a[:0])) == 0


def test_rank_parity_and_determinism(ctx):
    k, gp, cf = W.k25(64), W.gpu_a100(), W.space_stencil_paper()
    g, res = run_gpu(ctx, k, gp, cf)
    _, res2 = run_gpu(ctx, k, gp, cf)
    assert res.tobytes() == res2.tobytes()
    o = O.estimate_batch(k, gp, cf, NT)
    top = ctx.rank(res, 10)
    ranks = [int(r) for r in res["rank"]]
    check_ranking(ranks, o)
    assert [int(t) for t in top] == sorted(range(len(cf)), key=lambda i: ranks[i])[:10]


def test_describe_errors(ctx):
    from paper_2204_14242_b200 import WSError
    bad = W.k7(8)
    bad["accesses"] = bad["accesses"] + [(0, 0, (3, 0, 0))]
    with pytest.raises(WSError) as e:
        ctx.describe_kernel(bad)
    assert e.value.status == 3
    bad2 = W.k7(8)
    bad2["fields"][0] = dict(bad2["fields"][0], pitch=(1, 5, 100))
    with pytest.raises(WSError) as e:
        ctx.describe_kernel(bad2)
    assert e.value.status == 1
    g = W.gpu_v100()
    g["sector_bytes"] = 24
    with pytest.raises(WSError):
        ctx.describe_gpu(g)
    g = W.gpu_v100()
    g["line_bytes"] = 8192                       # 32-bit plane-relative unit arithmetic limit
    with pytest.raises(WSError) as e:
        ctx.describe_gpu(g)
    assert e.value.status == 2
    big = W.k7(8)                                # z-plane of 2 GiB (pitch[2] * 8 B = 2^31)
    big["fields"][0] = dict(big["fields"][0], extent=(1 << 14, 1 << 14, 4), pitch=(1, 1 << 14, 1 << 28))
    with pytest.raises(WSError) as e:
        ctx.describe_kernel(big)
    assert e.value.status == 2


# ----------------------------------------------------------------- full size (bench launch configuration)
def test_full_size_configs1_sampled(ctx):
    """BJ configs[1]: 25pt 512^3 A100, the whole 168-config batch in one launch (as bench.py
    times it); sampled configurations recomputed one by one by the oracle."""
    k, gp, cf = W.k25(512), W.gpu_a100(), W.space_stencil_paper()
    g, _ = run_gpu(ctx, k, gp, cf)
    assert all(r["status"] == 0 for r in g)
    # samples with small layer sets so the oracle finishes in seconds each (plus one deep one)
    idx = [i for i, c in enumerate(cf) if c[0] in ((1024, 1, 1), (512, 2, 1), (32, 32, 1), (256, 4, 1))
           and c[1] == (1, 1, 1)]
    idx += [i for i, c in enumerate(cf) if c[0] == (64, 4, 4) and c[1] == (1, 1, 2)]
    o = O.estimate_batch(k, gp, [cf[i] for i in idx], NT)
    errs = []
    for j, i in enumerate(idx):
        errs += compare(g[i], o[j], f"full[{i}] {cf[i]}")
    assert not errs, "\n".join(errs)
    # properties that hold at any size
    for r in g:
        assert r["sm_ld_lines"] <= r["sm_ld_sectors"] <= 4 * r["sm_ld_lines"]
        assert r["wave_ld_sectors"] <= r["sm_ld_sectors"] <= r["l1_req_ld_sectors"]
        assert r["ov_y"] <= r["ov_z"] <= r["wave_ld_sectors"]
        assert r["dram_ld_Bpl"] >= 8.0 - 1e-9 and r["dram_st_Bpl"] >= 8.0 - 1e-9


def test_full_size_lbm15_sampled(ctx):
    """BJ configs[2]: LBM15 256^3 A100 (49 shapes) in one launch; two sampled configs."""
    k, gp, cf = W.lbm15(256), W.gpu_a100(), W.space_lbm()
    g, _ = run_gpu(ctx, k, gp, cf)
    idx = [i for i, c in enumerate(cf) if c[0] in ((512, 1, 1), (64, 8, 1))]
    o = O.estimate_batch(k, gp, [cf[i] for i in idx], NT)
    errs = []
    for j, i in enumerate(idx):
        errs += compare(g[i], o[j], f"lbm[{i}] {cf[i]}")
    assert not errs, "\n".join(errs)
    for r in g:
        assert r["dram_ld_Bpl"] >= 120.0 and r["dram_ld_Bpl"] + r["dram_st_Bpl"] >= 240.0


def test_sharded_single_rank_matches(ctx):
    """dist.estimate_sharded on one rank = the direct batch (record bytes identical)."""
    import torch
    from paper_2204_14242_b200 import config_array, dist as D
    k, gp = W.k25(64), W.gpu_a100()
    kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(gp)
    a = config_array(kid, gid, W.space_stencil_paper())
    ref = ctx.estimate(a)
    ctx.rank(ref, 10)
    res, top = D.estimate_sharded(ctx, a, k_top=10)
    torch.cuda.synchronize()
    assert res.cpu().numpy().tobytes() == ref.tobytes()


@pytest.mark.parametrize("seed", range(8))
def test_random_medium_domains(ctx, seed):
    """Medium domains (24-56 cells per dim) with deep / folded blocks and occupancy > 1:
    exercises the derived planes, multi-block SM sets and multi-component row unions."""
    rng = random.Random(1000 + seed)
    k = W.random_kernel(500 + seed, max_fields=2, max_acc=10, max_dom=56)
    gp = dict(W.random_gpu(seed), n_sm=rng.choice([4, 6, 9, 16]))
    cf = []
    for _ in range(5):
        b = (rng.choice([1, 2, 4, 8, 16, 32]), rng.choice([1, 2, 4, 8]), rng.choice([1, 2, 4, 8, 16]))
        while b[0] * b[1] * b[2] > 256:
            b = (b[0], b[1], max(1, b[2] // 2))
        f = (rng.choice([1, 1, 2]), rng.choice([1, 2]), rng.choice([1, 2, 4]))
        cf.append((b, f, rng.choice([0, 1, 2, 3])))
    assert_parity(ctx, k, gp, cf, f"med{seed}")


def test_grid_sweep_sizes_sampled(ctx):
    """BJ configs[4]: the 25pt space at 32^3 and 96^3 (every config; oracle in seconds)."""
    for n in (32, 96):
        cf = W.space_stencil_paper()[::3]
        assert_parity(ctx, W.k25(n), W.gpu_a100(), cf, f"sweep{n}")


def test_full_size_lbm27_sampled(ctx):
    """BJ configs[2] LBM27 (58 arrays) 256^3: whole space in one launch, one sampled config."""
    k, gp, cf = W.lbm27(256), W.gpu_a100(), W.space_lbm()
    g, _ = run_gpu(ctx, k, gp, cf)
    idx = [i for i, c in enumerate(cf) if c[0] == (64, 8, 1)]
    o = O.estimate_batch(k, gp, [cf[i] for i in idx], NT)
    errs = []
    for j, i in enumerate(idx):
        errs += compare(g[i], o[j], f"lbm27[{i}] {cf[i]}")
    assert not errs, "\n".join(errs)


def test_architecture_exploration_sampled(ctx):
    """BJ configs[3]: the 25pt space on the B200-like set and hypothetical GPUs (varied L1,
    effective L2, SM count) at 128^3, every 7th configuration, plus LBM15 with folds."""
    k = W.k25(128)
    cf = W.space_stencil_paper()[::7]
    for gp in [W.with_outlook(W.gpu_b200_like()), W.gpu_hypothetical(128, 20, 148), W.gpu_hypothetical(256, 64, 80)]:
        assert_parity(ctx, k, gp, cf, gp["name"])
    assert_parity(ctx, W.lbm15(48), dict(W.gpu_a100(), n_sm=24), W.space_lbm(folds=True)[::5], "lbm15folds")


def test_full_size_b200_like_sampled(ctx):
    """configs[3] at full size: 25pt 512^3 on the B200-like parameters (148 SMs), whole space in
    one launch, three sampled configurations recomputed by the oracle."""
    k, gp, cf = W.k25(512), W.with_outlook(W.gpu_b200_like()), W.space_stencil_paper()
    g, _ = run_gpu(ctx, k, gp, cf)
    idx = [i for i, c in enumerate(cf) if c[0] in ((512, 2, 1), (128, 8, 1)) and c[1] == (1, 1, 1)]
    idx += [i for i, c in enumerate(cf) if c[0] == (32, 32, 1) and c[1] == (1, 2, 1)]
    o = O.estimate_batch(k, gp, [cf[i] for i in idx], NT)
    errs = []
    for j, i in enumerate(idx):
        errs += compare(g[i], o[j], f"b200[{i}] {cf[i]}")
    assert not errs, "\n".join(errs)


# ----------------------------------------------------------------- NEXT-3 / NEXT-4 variants + outlook metrics
def test_variants_paper_space_64(ctx):
    """Every other configuration of the 168-config space on 64^3 with each WS_VAR_* combination
    (multidimensional address space, previous-wave reuse, duplication-based L2 capacity), TLB
    pages and the L2 section link limiter on."""
    gp = dict(W.gpu_a100(), page_bytes=64 * 1024, link_bw=2e12)
    cf = [c + (1 + i % 15,) for i, c in enumerate(W.space_stencil_paper()[::2])]
    g, _ = assert_parity(ctx, W.k25(64), gp, cf, "var64")
    assert any(r["l2_link_sectors"] > 0 for r in g) and all(r["wave_pages"] > 0 for r in g)


def test_variants_lbm_and_sections(ctx):
    """LBM15 (32 arrays) with 3 and 4 L2 sections, 4 KiB pages, every variant."""
    for S in (3, 4):
        gp = dict(W.gpu_a100(), n_sm=12, l2_sections=S, page_bytes=4096, link_bw=5e11)
        cf = [c + (v,) for c in W.space_lbm()[::6] for v in (0, 5, 6, 8, 14)]
        assert_parity(ctx, W.lbm15(20), gp, cf, f"lbmS{S}")


def test_mdim_paper_example_gpu(ctx):
    """P:557-562 through the GPU path: 128 multidimensional vs 129 linear sectors."""
    k = {"fields": [{"extent": (256, 4, 1), "pitch": (1, 256, 1024), "align": -8, "elem": 8}],
         "accesses": [(0, 0, (0, 1, 0))], "dom_lo": (0, 0, 0), "dom_hi": (256, 2, 1), "regs": 0, "flops": 0.0}
    gp = dict(W.gpu_a100(), n_sm=1)
    g, _ = assert_parity(ctx, k, gp, [((256, 2, 1), (1, 1, 1), 1, 1), ((256, 2, 1), (1, 1, 1), 1, 0)], "mdim")
    assert g[0]["wave_ld_sectors"] == 128 and g[1]["wave_ld_sectors"] == 129


def test_variant_errors(ctx):
    from paper_2204_14242_b200 import WSError, config_array, result_dicts
    kid, gid = ctx.describe_kernel(W.k7(8)), ctx.describe_gpu(W.gpu_v100())
    r = result_dicts(ctx.estimate(config_array(kid, gid, [((32, 1, 1), (1, 1, 1), 0, 16)])))
    assert r[0]["status"] == 1
    for bad, st in [(dict(W.gpu_a100(), l2_sections=5), 2), (dict(W.gpu_a100(), page_bytes=100), 1),
                    (dict(W.gpu_a100(), page_bytes=64), 1), (dict(W.gpu_a100(), link_bw=-1.0), 1)]:
        with pytest.raises(WSError) as e:
            ctx.describe_gpu(bad)
        assert e.value.status == st


def test_full_size_variants_sampled(ctx):
    """configs[1] at 512^3 with variant bits 7 and the link limiter: whole space in one launch,
    three configurations recomputed by the oracle."""
    k, cf = W.k25(512), [c + (15,) for c in W.space_stencil_paper()]
    gp = dict(W.gpu_a100(), page_bytes=2 * 1024 * 1024, link_bw=2e12)
    g, _ = run_gpu(ctx, k, gp, cf)
    idx = [i for i, c in enumerate(cf) if c[0] in ((512, 2, 1), (32, 32, 1)) and c[1] == (1, 1, 1)]
    idx += [i for i, c in enumerate(cf) if c[0] == (64, 4, 4) and c[1] == (1, 1, 2)]
    o = O.estimate_batch(k, gp, [cf[i] for i in idx], NT)
    errs = []
    for j, i in enumerate(idx):
        errs += compare(g[i], o[j], f"fullvar[{i}] {cf[i]}")
    assert not errs, "\n".join(errs)
    for r in g:
        assert r["ov_y"] == r["ov_z"] and r["wave_pages"] > 0
        assert 0 < r["l2_eff_bytes"] <= gp["l2_bytes"]


# ----------------------------------------------------------------- NEXT-1: simulated hit rates
SIM_KEYS_INT = ["status", "capacity_bytes", "l1_requests", "l1_compulsory", "l1_misses", "st_requests",
                "st_compulsory", "st_misses", "ov_y", "y_resident", "ov_z_only", "z_resident"]
SIM_KEYS_FP = ["O_l1", "R_l1", "O_y", "R_y", "O_z", "R_z", "O_st", "R_st"]


def sim_parity(ctx, kernel, gpu, configs, caps, label):
    from paper_2204_14242_b200 import config_array
    from parity_util import close
    kid, gid = ctx.describe_kernel(kernel), ctx.describe_gpu(gpu)
    g = ctx.simulate(config_array(kid, gid, configs), caps)
    o = O.simulate_batch(kernel, gpu, configs, caps, NT)
    errs = []
    for i in range(len(configs)):
        for k in range(len(caps)):
            a, b = g[i][k], o[i][k]
            for key in SIM_KEYS_INT:
                if a[key] != b[key]:
                    errs.append(f"{label}[{i},{k}] {configs[i]} cap {caps[k]} {key}: gpu {a[key]} oracle {b[key]}")
            if b["status"] == 0:
                for key in SIM_KEYS_FP:
                    if not close(a[key], b[key]):
                        errs.append(f"{label}[{i},{k}] {key}: gpu {a[key]!r} oracle {b[key]!r}")
    assert not errs, "\n".join(errs[:40])
    return g


CAPS = [1 << 40, 1 << 20, 262144, 65536, 16384, 4096, 1024, 128]


def test_sim_small_cases(ctx):
    cases = [
        (W.stencil_star(24, 12, 12, 4, regs=64), dict(W.gpu_a100(), n_sm=6),
         [((8, 2, 2), (1, 1, 1), 1), ((16, 4, 1), (1, 1, 2), 0), ((4, 4, 4), (1, 2, 1), 2), ((32, 1, 1), (1, 1, 1), 1, 2)]),
        (W.stencil_star(20, 10, 12, 1, regs=0), dict(W.gpu_a100(), n_sm=4), [((4, 4, 2), (1, 1, 2), 2)]),
        (W.lbm15(8), dict(W.gpu_a100(), n_sm=3), [((4, 2, 2), (1, 1, 1), 1), ((8, 1, 1), (1, 1, 1), 0)]),
    ]
    for i, (k, gp, cf) in enumerate(cases):
        sim_parity(ctx, k, gp, cf, CAPS, f"simsmall{i}")


@pytest.mark.parametrize("seed", range(10))
def test_sim_random(ctx, seed):
    k, gp = W.random_kernel(seed, max_dom=12), W.random_gpu(seed)
    cf = [W.random_config(seed * 10 + j) for j in range(3)]
    sim_parity(ctx, k, gp, cf, [1 << 30, 8192, 2048, 512, 128], f"simrand{seed}")


def test_sim_paper_space_48(ctx):
    """Every 4th configuration of the 168-config 25pt space on 48^3 (A100 with 24 SMs), eight
    capacities from 128 B to 1 TiB; then the device fit of the z-layer samples against the oracle's."""
    k, gp = W.k25(48), dict(W.gpu_a100(), n_sm=24)
    cf = W.space_stencil_paper()[::4]
    g = sim_parity(ctx, k, gp, cf, CAPS, "sim48")
    Os = [r["O_z"] for row in g for r in row if r["status"] == 0 and r["ov_z_only"] > 0]
    Rs = [r["R_z"] for row in g for r in row if r["status"] == 0 and r["ov_z_only"] > 0]
    (a, b, c), rss = ctx.fit_gompertz(Os, Rs)
    (oa, ob, oc), orss = O.fit_gompertz(Os, Rs)
    assert rss == pytest.approx(orss, rel=1e-6, abs=1e-12)
    assert (a, b, c) == pytest.approx((oa, ob, oc), rel=1e-4)


def test_fit_known_curves(ctx):
    Os = [0.05 * i for i in range(60)]
    for abc in ([1.0, 5.0, -2.0], [0.95, 0.02, -3.0], list(W.HIT_ABC_DEFAULT[2])):
        Rs = [O.hit_rate(abc, o) for o in Os]
        (a, b, c), rss = ctx.fit_gompertz(Os, Rs)
        (oa, ob, oc), orss = O.fit_gompertz(Os, Rs)
        assert (a, b, c) == pytest.approx((oa, ob, oc), rel=1e-6)
        assert (a, b, c) == pytest.approx(tuple(abc), rel=1e-6)


def test_sim_buffer_cache(ctx):
    """ws_simulate keeps its device buffers between calls (grow-only slots): a small call after a
    large one, after a forced parallel-path call, and after ws_sim_release all match the oracle."""
    small = (W.stencil_star(20, 10, 12, 1, regs=0), dict(W.gpu_a100(), n_sm=4), [((4, 4, 2), (1, 1, 2), 2)])
    large = (W.k25(48), dict(W.gpu_a100(), n_sm=24), W.space_stencil_paper()[::21])
    sim_parity(ctx, *large, CAPS, "cache-large")
    sim_parity(ctx, *small, CAPS, "cache-small")
    os.environ["WS_SIM_PAR"] = "all"
    try:
        sim_parity(ctx, *large, CAPS, "cache-large-par")
    finally:
        os.environ.pop("WS_SIM_PAR", None)
    sim_parity(ctx, *small, CAPS, "cache-small2")
    ctx.sim_release()
    ctx.sim_release()
    sim_parity(ctx, *small, CAPS, "cache-small3")


def test_sim_errors(ctx):
    from paper_2204_14242_b200 import config_array
    kid, gid = ctx.describe_kernel(W.k7(8)), ctx.describe_gpu(dict(W.gpu_v100(), n_sm=4))
    r = ctx.simulate(config_array(kid, gid, [((32, 1, 1), (1, 1, 1), 0, 1), ((32, 1, 1), (1, 1, 1), 0)]), [0, 4096])
    assert r[0][0]["status"] == 1 and r[0][1]["status"] == 1      # multidimensional variant
    assert r[1][0]["status"] == 1 and r[1][1]["status"] == 0      # capacity 0


def test_sim_full_size_sampled(ctx):
    """25pt 512^3 A100 (BJ configs[1] size): three configurations through the whole simulation at
    the A100's L1 and effective L2 capacities (and 1/4, 4x), against the oracle."""
    k, gp = W.k25(512), W.gpu_a100()
    cf = [((512, 2, 1), (1, 1, 1), 0), ((32, 32, 1), (1, 1, 1), 0), ((256, 4, 1), (1, 1, 1), 0)]
    caps = [gp["l1_bytes"], gp["l2_bytes"] // 8, gp["l2_bytes"] // 2, 2 * gp["l2_bytes"]]
    sim_parity(ctx, k, gp, cf, caps, "simfull")


def test_sim_full_space_512_properties(ctx):
    """The whole 168-config space at 512^3 (the NEXT-1 calibration size; memory-bounded batches
    of the parallel path) x 4 capacities: LRU inclusion (misses never grow with the capacity),
    compulsory <= misses <= requests, residency <= overlap, hit rates in [0, 1]."""
    from paper_2204_14242_b200 import config_array
    k, gp = W.k25(512), W.gpu_a100()
    kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(gp)
    caps = [gp["l1_bytes"], gp["l2_bytes"] // 8, gp["l2_bytes"] // 2, 2 * gp["l2_bytes"]]
    rows = ctx.simulate(config_array(kid, gid, W.space_stencil_paper()), caps)
    for i, row in enumerate(rows):
        assert all(r["status"] == 0 for r in row), i
        for key in ("l1", "st"):
            m = [r[f"{key}_misses"] for r in row]
            assert all(a >= b for a, b in zip(m, m[1:])), (i, key, m)
            assert row[0][f"{key}_compulsory"] <= m[-1] and m[0] <= row[0][f"{key}_requests"], (i, key)
        for a, b in zip(row, row[1:]):
            assert b["y_resident"] >= a["y_resident"] and b["z_resident"] >= a["z_resident"], i
        for r in row:
            assert r["y_resident"] <= r["ov_y"] and r["z_resident"] <= r["ov_z_only"], i
            for f in ("R_l1", "R_y", "R_z", "R_st"):
                assert 0.0 <= r[f] <= 1.0 + 1e-12, (i, f, r[f])
    ctx.sim_release()


# ----------------------------------------------------------------- NEXT-2: validation kernel
def _st_run(ctx, n, block, fold, seed=0):
    import torch
    from oracle import stencil as ST
    g = torch.Generator().manual_seed(seed)
    src = torch.rand((n[2] + 8, n[1] + 8, n[0] + 8), dtype=torch.float64, generator=g)
    d_src = src.cuda()
    d_dst = torch.zeros_like(d_src)
    ctx.validate_stencil25(d_src.data_ptr(), d_dst.data_ptr(), n, block, fold, reps=1)
    torch.cuda.synchronize()
    return src.numpy(), d_dst.cpu().numpy(), ST


@pytest.mark.parametrize("fold", [(1, 1, 1), (1, 2, 1), (1, 1, 2)])
def test_validation_stencil_small(ctx, fold):
    """The NEXT-2 kernel against the plain numpy definition on ragged domains (partial blocks and
    partially active folded threads): FP64 within 1e-13 (FMA contraction only)."""
    for n, block in [((20, 12, 16), (8, 4, 2)), ((37, 11, 9), (16, 2, 4)), ((9, 9, 9), (32, 1, 1))]:
        src, dst, ST = _st_run(ctx, n, block, fold)
        ref = ST.stencil25(src, n)
        assert np.allclose(dst, ref, rtol=1e-13, atol=1e-13), (n, block, fold)


def test_validation_stencil_full_size_sampled(ctx):
    """512^3 (the bench / validation size), (16,2,32) with 2z folding: 2000 sampled cells."""
    import torch
    from oracle import stencil as ST
    n = (512, 512, 512)
    d_src = torch.rand((520, 520, 520), dtype=torch.float64, device="cuda")
    d_dst = torch.zeros_like(d_src)
    ctx.validate_stencil25(d_src.data_ptr(), d_dst.data_ptr(), n, (16, 2, 32), (1, 1, 2), reps=1)
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    pts = rng.integers(4, 516, size=(2000, 3))
    src = d_src.cpu().numpy()
    dst = d_dst.cpu().numpy()
    for z, y, x in pts:
        sub = src[z - 4:z + 5, y - 4:y + 5, x - 4:x + 5]
        ref = ST.stencil25(np.pad(sub, 0), (1, 1, 1))[4, 4, 4]
        assert abs(dst[z, y, x] - ref) <= 1e-13 * max(1.0, abs(ref))


def test_validation_lbm15_small(ctx):
    """The LBM15 validation kernel against the plain numpy definition (ragged blocks)."""
    import torch
    from oracle import stencil as ST
    for n, block in [((10, 8, 6), (4, 2, 2)), ((13, 7, 5), (8, 4, 1)), ((6, 6, 6), (1, 8, 8))]:
        g = torch.Generator().manual_seed(sum(n))
        shp = (n[2] + 2, n[1] + 2, n[0] + 2)
        src = torch.rand((15,) + shp, dtype=torch.float64, generator=g)
        phi = torch.rand(shp, dtype=torch.float64, generator=g)
        d_src, d_phi = src.cuda(), phi.cuda()
        d_dst, d_fd = torch.zeros_like(d_src), torch.zeros_like(d_phi)
        ctx.validate_lbm15(d_src.data_ptr(), d_dst.data_ptr(), d_phi.data_ptr(), d_fd.data_ptr(), n, block)
        torch.cuda.synchronize()
        dst, fd = ST.lbm15(src.numpy(), phi.numpy(), n)
        assert np.allclose(d_dst.cpu().numpy(), dst, rtol=1e-12, atol=1e-12), (n, block)
        assert np.allclose(d_fd.cpu().numpy(), fd, rtol=1e-12, atol=1e-12), (n, block)


def test_extended_space_multiblock_sets(ctx):
    """The extended space with 64-512-thread blocks: several blocks per SM
    (k = 2..16), so multi-block SM sets whose members are split into translation classes
    when their footprints cannot share a line (k_smset) -- every configuration against the
    oracle on 48^3 and a ragged 40x36x44 domain."""
    sp = [c for c in W.space_extended() if c[0][0] * c[0][1] * c[0][2] <= 512][::9]
    for k in (W.k25(48), W.stencil_star(40, 36, 44, 4, regs=64)):
        assert_parity(ctx, k, dict(W.gpu_a100(), n_sm=24), sp, "ext")


def test_extended_space_grouped_sets_full_a100(ctx):
    """Extended-space configurations with 64-256-thread blocks on 96^3 with the full A100 (108
    SMs, k up to 16 blocks per SM): multi-block SM sets grouped by translation in k_smset (group
    sizes > 1) and fetched dynamically by k_sclass -- every count against the oracle."""
    sp = [c for c in W.space_extended() if c[0][0] * c[0][1] * c[0][2] <= 256][::60][:6]
    assert_parity(ctx, W.k25(96), W.gpu_a100(), sp, "ext96")


@pytest.mark.parametrize("mode", ["all", "0"])
def test_sim_parallel_path_matches_oracle(ctx, mode):
    """The parallel offline path (wavelet-matrix stack distances) forced on every stream, and the
    warp path forced on every stream, both against the oracle (WS_SIM_PAR)."""
    os.environ["WS_SIM_PAR"] = mode
    try:
        cases = [
            (W.stencil_star(24, 12, 12, 4, regs=64), dict(W.gpu_a100(), n_sm=6),
             [((8, 2, 2), (1, 1, 1), 1), ((16, 4, 1), (1, 1, 2), 0), ((4, 4, 4), (1, 2, 1), 2)]),
            (W.lbm15(8), dict(W.gpu_a100(), n_sm=3), [((4, 2, 2), (1, 1, 1), 1), ((8, 1, 1), (1, 1, 1), 0)]),
        ]
        for i, (k, gp, cf) in enumerate(cases):
            sim_parity(ctx, k, gp, cf, CAPS, f"par{mode}{i}")
        for seed in range(4):
            k, gp = W.random_kernel(seed, max_dom=12), W.random_gpu(seed)
            cf = [W.random_config(seed * 10 + j) for j in range(3)]
            sim_parity(ctx, k, gp, cf, [1 << 30, 8192, 2048, 512, 128], f"par{mode}r{seed}")
    finally:
        os.environ.pop("WS_SIM_PAR", None)
