"""GPU tests of the round-2 boundary additions, through the C ABI:

* ws_rank at scale: the one-CTA shared-memory sort (n <= 16384) and the radix path (larger n)
  against a plain numpy lexsort of (t_pred, index), with ties and failed records;
* describe-time errors of SURVEY 8(b): alignment not a multiple of the element size, more than 16
  distinct x-offset runs in a field;
* ws_estimate_multi (BJ configs[3]): byte-identical to one ws_estimate per hardware set, and
  against the oracle on sampled (configuration, hardware set) pairs.
"""
import os

import numpy as np
import pytest

import workloads as W
from oracle import oracle as O
from parity_util import compare

pytestmark = pytest.mark.gpu
NT = max(1, min(32, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2204_14242_b200 import Context
    c = Context(0)
    yield c
    c.close()


def _synthetic_results(n, seed):
    from paper_2204_14242_b200.ws import RESULT_DTYPE
    rng = np.random.default_rng(seed)
    r = np.zeros(n, dtype=RESULT_DTYPE)
    r["t_pred"] = rng.choice(rng.random(max(2, n // 7)) * 1e-3, n)      # many exact ties
    r["status"] = np.where(rng.random(n) < 0.03, 2, 0)
    return r


def _expected_order(r):
    key = np.where(r["status"] == 0, r["t_pred"], np.inf)
    return np.lexsort((np.arange(len(r)), key))


@pytest.mark.parametrize("n", [1, 2, 168, 2048, 2049, 5000, 8232, 32768, 32769, 100000, 262144, 300001])
def test_rank_sort_paths(ctx, n):
    r = _synthetic_results(n, n)
    top = ctx.rank(r, 10)
    order = _expected_order(r)
    assert np.array_equal(r["rank"][order], np.arange(n))
    assert list(top) == list(order[:10])


def test_rank_async_device_time(ctx):
    """Radix path on 10^5 device-resident records: time per ws_rank_async (CUDA events)."""
    import torch
    from paper_2204_14242_b200.ws import RESULT_DTYPE
    n = 100000
    r = _synthetic_results(n, 7)
    d = torch.from_numpy(r.view(np.uint8).copy()).cuda()
    top = torch.zeros(10, dtype=torch.int32, device="cuda")
    for _ in range(3):
        ctx.rank_async(d.data_ptr(), n, 10, top.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        ctx.rank_async(d.data_ptr(), n, 10, top.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"ws_rank_async n={n}: {ms * 1e3:.1f} us")
    back = np.frombuffer(d.cpu().numpy().tobytes(), dtype=RESULT_DTYPE)
    assert np.array_equal(back["rank"][_expected_order(r)], np.arange(n))
    assert ms < 1.0


def test_describe_alignment_and_run_limits(ctx):
    from paper_2204_14242_b200 import WSError
    k = W.k7(8)
    k["fields"][0] = dict(k["fields"][0], align=4)           # 8 B elements at a 4 B alignment
    with pytest.raises(WSError) as e:
        ctx.describe_kernel(k)
    assert e.value.status == 1
    k["fields"][0] = dict(k["fields"][0], align=-8)
    ctx.describe_kernel(k)                                   # negative multiples are valid
    # 17 distinct x-offset runs in one field: loads at x offsets {0}, {2}, ... {32} (isolated)
    runs = W.stencil_star(40, 4, 4, 1, regs=0)
    f0 = dict(runs["fields"][0])
    f0["extent"] = (80, f0["extent"][1], f0["extent"][2])
    f0["pitch"] = (1, 80, 80 * f0["extent"][1])
    runs["fields"] = [f0, dict(f0)]
    runs["accesses"] = [(0, 0, (2 * i, 0, 0)) for i in range(17)] + [(1, 1, (0, 0, 0))]
    with pytest.raises(WSError) as e:
        ctx.describe_kernel(runs)
    assert e.value.status == 2
    runs["accesses"] = [(0, 0, (2 * i, 0, 0)) for i in range(16)] + [(1, 1, (0, 0, 0))]
    ctx.describe_kernel(runs)


def test_estimate_multi_byte_identical(ctx):
    """configs[3]: [1] u [2] (the 168-config 25pt space and the 49 LBM15 configurations, two
    kernels in one batch) at small sizes x the 51 configs[3] hardware sets in one call == one
    ws_estimate per set (every byte of every record); six integer-stage groups."""
    from paper_2204_14242_b200 import config_array
    sets = W.hw_grid_configs3()
    k1, k2 = ctx.describe_kernel(W.k25(96)), ctx.describe_kernel(W.lbm15(24))
    gids = [ctx.describe_gpu(g) for g in sets]
    cf = np.concatenate([config_array(k1, 0, W.space_stencil_paper()), config_array(k2, 0, W.space_lbm())])
    multi = ctx.estimate_multi(cf, gids)
    assert ctx.last_group_count() == 6
    for g, gid in enumerate(gids):
        cf["gpu_id"] = gid
        one = ctx.estimate(cf)
        assert multi[g].tobytes() == one.tobytes(), sets[g]["name"]
    multi2 = ctx.estimate_multi(cf, gids)          # graph replay
    assert multi2.tobytes() == multi.tobytes()


def test_estimate_multi_vs_oracle_sampled(ctx):
    """configs[3] at the full sizes: the 25pt 512^3 space and LBM15 256^3 x the 51 hardware sets in
    one call; sampled (configuration, set) pairs recomputed by the oracle."""
    from paper_2204_14242_b200 import config_array, result_dicts
    sets = W.hw_grid_configs3()
    kern = [W.k25(512), W.lbm15(256)]
    kids = [ctx.describe_kernel(k) for k in kern]
    gids = [ctx.describe_gpu(g) for g in sets]
    s25, slbm = W.space_stencil_paper(), W.space_lbm()
    cf = np.concatenate([config_array(kids[0], 0, s25), config_array(kids[1], 0, slbm)])
    which = [(0, c) for c in s25] + [(1, c) for c in slbm]
    multi = ctx.estimate_multi(cf, gids)
    assert (multi["status"] == 0).all()
    cheap = [i for i, (ki, c) in enumerate(which) if c[0][2] == 1 and c[1][2] == 1 and (ki == 0 or c[0][0] >= 64)]
    picks = [(g, cheap[(5 * g) % len(cheap)]) for g in (0, 1, 2, 7, 13, 26, 40, 50)]
    picks += [(2, len(s25) + 2), (30, len(s25) + 40)]      # LBM15 configurations
    errs = []
    for g, i in picks:
        ki, c = which[i]
        o = O.estimate(kern[ki], sets[g], c)
        a = result_dicts(multi[g][i:i + 1])[0]
        errs += compare(a, o, f"set{g} cfg{i} {c}")
    assert not errs, "\n".join(errs)


@pytest.mark.parametrize("case", ["c0_16", "c1_168", "ext_1024", "ext_1025", "one"])
def test_estimate_ranked_byte_identical(ctx, case):
    """ws_estimate_ranked_async (model + rank fused into one CTA for n <= 1024) = ws_estimate_async
    followed by ws_rank_async, record bytes and top-k, over graph capture and replays."""
    import torch
    from paper_2204_14242_b200 import config_array
    from paper_2204_14242_b200.ws import RESULT_DTYPE
    k, space = {
        "c0_16": (W.k25(64), W.space_stencil_paper()[::11]),
        "c1_168": (W.k25(96), W.space_stencil_paper()),
        "ext_1024": (W.k25(48), W.space_extended()[:1024]),
        "ext_1025": (W.k25(48), W.space_extended()[:1025]),
        "one": (W.k25(32), W.space_stencil_paper()[5:6]),
    }[case]
    kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(W.gpu_a100())
    a = config_array(kid, gid, space)
    n, kt = len(a), min(10, len(a))
    dc = torch.from_numpy(a.view(np.uint8).copy()).cuda()
    ref = torch.zeros(n * RESULT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    rtop = torch.zeros(kt, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    ctx.estimate_async(dc.data_ptr(), n, ref.data_ptr())
    ctx.rank_async(ref.data_ptr(), n, kt, rtop.data_ptr())
    torch.cuda.synchronize()
    out = torch.zeros_like(ref)
    top = torch.zeros_like(rtop)
    for rep in range(3):
        out.zero_()
        top.zero_()
        torch.cuda.synchronize()
        ctx.estimate_ranked_async(dc.data_ptr(), n, out.data_ptr(), kt, top.data_ptr())
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == ref.cpu().numpy().tobytes(), (case, rep)
        assert top.cpu().tolist() == rtop.cpu().tolist(), (case, rep)
    r = np.frombuffer(ref.cpu().numpy().tobytes(), dtype=RESULT_DTYPE)
    assert sorted(r["rank"].tolist()) == list(range(n))


def test_graph_cache_alternating_buffers(ctx):
    """Double-buffered callers: ws_estimate_ranked_async alternating between two input / output
    buffer pairs (the context keeps a captured graph per key) gives the same records every call."""
    import torch
    from paper_2204_14242_b200 import config_array
    from paper_2204_14242_b200.ws import RESULT_DTYPE
    kid, gid = ctx.describe_kernel(W.k25(80)), ctx.describe_gpu(W.gpu_a100())
    a = config_array(kid, gid, W.space_stencil_paper()[::3])
    n = len(a)
    ref = ctx.estimate(a)
    ctx.rank(ref, 5)
    dc = [torch.from_numpy(a.view(np.uint8).copy()).cuda() for _ in range(2)]
    do = [torch.zeros(n * RESULT_DTYPE.itemsize, dtype=torch.uint8, device="cuda") for _ in range(2)]
    tp = [torch.zeros(5, dtype=torch.int32, device="cuda") for _ in range(2)]
    for it in range(6):
        b = it & 1
        do[b].zero_()
        torch.cuda.synchronize()
        ctx.estimate_ranked_async(dc[b].data_ptr(), n, do[b].data_ptr(), 5, tp[b].data_ptr())
        torch.cuda.synchronize()
        assert do[b].cpu().numpy().tobytes() == ref.tobytes(), it
