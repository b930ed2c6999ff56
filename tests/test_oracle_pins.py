"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test names the passage it pins.  None of these expected values comes
from the CUDA path; they are the paper's printed numbers
(tests/golden/paper_values.json), closed forms derived in DESIGN.md, or an
independent brute-force implementation (tests/indep_model.py).
"""
import json
import math

import numpy as np
import os

import pytest

import workloads as W
from oracle import oracle as O
import indep_model as M

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


# --------------------------------------------------------------------- a2: address map
def test_address_map_paper_example():
    """A[tidx][tidy+1] on a 100-wide array with a -1 element alignment."""
    g = GOLD["address_map_example"]
    fld = {"extent": (100, 10, 1), "pitch": (1, 100, 1000),
           "align": g["align_elems"] * g["elem"], "elem": g["elem"]}
    for tx, ty, idx in g["cases"]:
        a = O.address(fld, (tx, ty + 1, 0))
        assert a // 32 == idx, (tx, ty)


def test_address_map_pystencils_expression():
    """src_W = src + (tx + bx*BX + 1) + (ty + by*BY)*w (element units)."""
    w = 37
    fld = {"extent": (w, 20, 3), "pitch": (1, w, w * 20), "align": 0, "elem": 1}
    BX, BY = 8, 4
    for tx, bx, ty, by in [(0, 0, 0, 0), (3, 2, 1, 3), (7, 1, 3, 0)]:
        expect = (tx + bx * BX + 1) + (ty + by * BY) * w
        assert O.address(fld, (tx + bx * BX + 1, ty + by * BY, 0)) == expect


# --------------------------------------------------------------------- a3: sectors
def _one_load_kernel(n, align, fold=(1, 1, 1)):
    fld = {"extent": (n * fold[0] + 8, 2, 2), "pitch": (1, n * fold[0] + 8, 2 * (n * fold[0] + 8)),
           "align": align, "elem": 8}
    return {"name": "oneload", "fields": [fld], "accesses": [(0, 0, (0, 0, 0))],
            "dom_lo": (0, 0, 0), "dom_hi": (n * fold[0], 1, 1), "regs": 0, "flops": 0.0}


def test_sectors_32_contiguous_doubles():
    """P:474-475 + BJ north_star: 32 contiguous doubles, 256 B aligned -> 8 sectors, 2 lines;
    shifted by 8 B -> 9 sectors, 3 lines."""
    g = W.gpu_v100()
    r = O.estimate(_one_load_kernel(32, 0), g, ((32, 1, 1), (1, 1, 1), 1))
    assert (r["l1_req_ld_sectors"], r["wave_ld_sectors"], r["sm_ld_sectors"], r["sm_ld_lines"]) == (8, 8, 8, 2)
    r = O.estimate(_one_load_kernel(32, 8), g, ((32, 1, 1), (1, 1, 1), 1))
    assert (r["l1_req_ld_sectors"], r["wave_ld_sectors"], r["sm_ld_lines"]) == (9, 9, 3)


def test_sectors_strided_warp():
    """Stride-2 doubles (x fold 2): each warp instruction spans 16 sectors (P:389 pattern)."""
    g = W.gpu_v100()
    r = O.estimate(_one_load_kernel(32, 0, fold=(2, 1, 1)), g, ((32, 1, 1), (2, 1, 1), 1))
    assert r["n_instr"] == 2
    assert r["l1_req_ld_sectors"] == 2 * 16
    assert r["wave_ld_sectors"] == 16          # the union is the 64 contiguous doubles
    assert r["l1_wavefronts"] == 2 * 2 * 2     # 2 instr x 2 half-warps x 2 wavefronts


def test_unique_sectors_helper():
    assert O.unique_sectors([8 * i for i in range(32)]) == 8
    assert O.unique_sectors([8 + 8 * i for i in range(32)]) == 9
    assert O.unique_sectors([16 * i for i in range(32)]) == 16
    assert O.unique_sectors([128 * i for i in range(32)]) == 32


# --------------------------------------------------------------------- a3: wavefronts
def test_halfwarp_wavefronts_paper_examples():
    """strides 1/2/16 doubles -> 1/2/16 cycles per half warp."""
    g = W.gpu_a100()
    for stride, cyc in GOLD["halfwarp_wavefronts"]["stride_elems_to_cycles"]:
        assert O.halfwarp_wavefronts([8 * stride * i for i in range(16)], g) == cyc


def test_halfwarp_far_pairing():
    """non-conflicting addresses > 1024 B apart cannot pair: two 8-double runs
    4096 B apart -> 2 wavefronts; inside the window they pair -> 1."""
    g = W.gpu_a100()
    a = [8 * i for i in range(8)] + [4096 + 64 + 8 * i for i in range(8)]
    assert O.halfwarp_wavefronts(a, g) == 2
    b = [8 * i for i in range(8)] + [64 + 8 * i for i in range(8)]
    assert O.halfwarp_wavefronts(b, g) == 1
    # duplicates are one address (unique words, Listing 1 'unique(addresses)')
    assert O.halfwarp_wavefronts([0] * 16, g) == 1
    assert O.halfwarp_wavefronts([], g) == 0


def test_wavefronts_listing1_when_span_below_window():
    """Within a 1024 B span the rule is exactly Listing 1: max over banks of unique words."""
    import random
    g = W.gpu_a100()
    rng = random.Random(5)
    for _ in range(200):
        words = [rng.randrange(0, 128) for _ in range(16)]
        a = [8 * u for u in words]
        cnt = [0] * 16
        for u in set(words):
            cnt[u % 16] += 1
        assert O.halfwarp_wavefronts(a, g) == max(cnt)


def _k25_small(nx=64, ny=32, nz=32):
    return W.stencil_star(nx, ny, nz, 4, regs=64)


def test_l1_cycles_25pt_closed_form():
    """bx >= 16 -> one wavefront per half-warp instruction: 26 instr x 2 = 52 cycles
    per warp-wide LUP (1.625/LUP); 2z folding: 44 instr / 2 LUP -> 1.375/LUP; bx < 16 with a
    row pitch >= 1024 B: 16/bx wavefronts per half-warp instruction."""
    k = _k25_small(256, 16, 16)   # row pitch 264*8 = 2112 B >= 1024 B
    g = W.gpu_a100()
    r = O.estimate(k, g, ((32, 4, 2), (1, 1, 1), 1))
    assert r["n_instr"] == 26
    assert r["l1_cyc_per_lup"] == pytest.approx(1.625, abs=0)
    r = O.estimate(k, g, ((32, 4, 2), (1, 1, 2), 1))
    assert r["n_instr"] == 44
    assert r["l1_cyc_per_lup"] == pytest.approx(1.375, abs=0)
    for bx in (8, 4, 2, 1):
        r = O.estimate(k, g, ((bx, 16, 2), (1, 1, 1), 1))
        assert r["l1_cyc_per_lup"] == pytest.approx(26 * 2 * (16 // bx) / 32, abs=0), bx


# --------------------------------------------------------------------- a5/a6 closed forms
XS = 256  # row width of the series domain


def _series_setup(d, ry, rz):
    """domain 256x32x64, 16 SMs, k=1 -> 16-block waves of (256,1,1)
    blocks folded d-deep in z: a wave d layers deep spanning full rows."""
    k = W.stencil_star(XS, 32, 64, 4, regs=0)
    g = W.gpu_a100()
    g["n_sm"] = 16
    g["hit_abc"][1] = [ry, 0.0, 0.0]     # R_y == ry for every O
    g["hit_abc"][2] = [rz, 0.0, 0.0]     # R_z == rz
    return k, g, ((XS, 1, 1), (1, 1, d), 1)


@pytest.mark.parametrize("d,vol", GOLD["wave_depth_series"]["depth_to_BperLup"])
def test_wave_depth_series(d, vol):
    """without z-layer reuse a d-deep wave loads (d+8)/d values per LUP:
    72/40/24/16/(12)/10 B/Lup.  Exact value here: 8(d+8)/d + 8*8/XS (the x-halo of
    the XS-wide rows, 8 extra elements per row never reused; rows are whole sectors)."""
    k, g, c = _series_setup(d, 1.0, 0.0)
    r = O.estimate(k, g, c)
    assert vol == pytest.approx(8 * (d + 8) / d)
    assert r["dram_ld_Bpl"] == pytest.approx(vol + 64 / XS, rel=1e-12)
    assert r["dram_st_Bpl"] == pytest.approx(8.0, rel=1e-12)


@pytest.mark.parametrize("d", [1, 2, 4, 8, 16, 32])
def test_layer_condition_floor(d):
    """with full z-layer reuse the stencil needs one load and one store per
    point: 8 B/Lup (+ the same 64/XS B/Lup x-halo)."""
    k, g, c = _series_setup(d, 1.0, 1.0)
    r = O.estimate(k, g, c)
    assert r["dram_ld_Bpl"] == pytest.approx(GOLD["stencil_floor"]["load_BperLup"] + 64 / XS, rel=1e-12)
    assert r["dram_st_Bpl"] == pytest.approx(GOLD["stencil_floor"]["store_BperLup"], rel=1e-12)
    # no reuse at all: (d+8)/d values plus the y-halo of the 16-row wave
    k, g, c = _series_setup(d, 0.0, 0.0)
    r0 = O.estimate(k, g, c)
    assert r0["dram_ld_Bpl"] > r["dram_ld_Bpl"]


def test_lbm15_floors():
    """D3Q15 streaming moves 15 doubles in and 15 out per LUP (240 B/Lup);
    with perfect reuse the phase field adds >= 8 B/Lup load; every config loads >= 128 B/Lup
    and stores >= 128 B/Lup (15 PDFs + FD result)."""
    k = W.lbm15(24)
    g = W.gpu_a100()
    g["n_sm"] = 8
    for i in range(4):
        g["hit_abc"][i] = [1.0, 0.0, 0.0]
    for c in [((8, 2, 2), (1, 1, 1), 1), ((32, 1, 1), (1, 1, 1), 1), ((1, 8, 4), (1, 1, 1), 1)]:
        r = O.estimate(k, g, c)
        assert r["dram_ld_Bpl"] >= 128.0 - 1e-9
        assert r["dram_st_Bpl"] >= 128.0 - 1e-9
        assert r["dram_ld_Bpl"] + r["dram_st_Bpl"] >= GOLD["d3q15_streaming"]["pdf_BperLup_read_plus_write"]


# --------------------------------------------------------------------- a7 arithmetic
def test_gompertz_form():
    """R(O) = a exp(-b exp(-cO)); R(0) = a e^{-b}; SURVEY Q17 default anchors."""
    assert O.hit_rate([0.9, 2.0, -1.0], 0.0) == pytest.approx(0.9 * math.exp(-2.0), rel=1e-15)
    L1, L2y, L2z, L2st = W.HIT_ABC_DEFAULT
    assert O.hit_rate(L1, 1.0) == pytest.approx(0.90, abs=2e-3)
    assert O.hit_rate(L1, 2.0) == pytest.approx(0.20, abs=2e-3)
    assert O.hit_rate(L2z, 2.0) == pytest.approx(0.05, abs=2e-3)
    assert O.hit_rate(L2st, 1.0) == pytest.approx(0.95, abs=2e-3)
    # monotone decreasing ("With increasing oversubscription ... towards zero")
    for abc in W.HIT_ABC_DEFAULT:
        vals = [O.hit_rate(abc, o / 4) for o in range(40)]
        assert all(a >= b for a, b in zip(vals, vals[1:]))
        assert vals[-1] < 0.01


def test_model_homogeneity():
    """scaling every bandwidth and the clock by s scales predicted time by 1/s."""
    k = W.k7(16)
    g = W.gpu_v100()
    c = ((32, 2, 2), (1, 1, 1), 0)
    r1 = O.estimate(k, g, c)
    g2 = dict(g)
    s = 3.0
    g2["dram_bw"], g2["l2_bw"], g2["clock_hz"] = g["dram_bw"] * s, g["l2_bw"] * s, g["clock_hz"] * s
    r2 = O.estimate(k, g2, c)
    assert r2["t_pred"] == pytest.approx(r1["t_pred"] / s, rel=1e-12)
    assert r2["limiter"] == r1["limiter"]


def test_model_eq5_and_limiter_arithmetic():
    """Eq. 5 and the max-limiter (Q1) recomputed from the integer fields."""
    k = W.k7(24)
    g = W.gpu_v100()
    for c in W.space_k7()[:15]:
        r = O.estimate(k, g, c)
        n = r["lup_wave"]
        v_red = max(0, r["l1_req_ld_sectors"] - r["sm_ld_sectors"])
        l2l1 = r["sm_ld_sectors"] + (1 - r["R_l1"]) * v_red
        assert r["l2_ld_Bpl"] == pytest.approx(32 * l2l1 / n, rel=1e-12)
        t = max(r["t_l1"], r["t_l2"], r["t_dram"])
        assert r["t_pred"] == pytest.approx(t * 24 ** 3, rel=1e-12)
        assert [r["t_l1"], r["t_l2"], r["t_dram"]][r["limiter"]] == t


# --------------------------------------------------------------------- a1 combinatorics
def test_sweep_sizes():
    s = GOLD["sweep_constraint"]
    assert len(W.block_shapes(1024)) == s["n_shapes_1024"]
    assert len(W.block_shapes(512)) == s["n_shapes_512"]
    assert len(W.space_stencil_paper()) == s["n_shapes_1024"] * s["n_folds"]


def test_sequential_layer_condition_numbers():
    """P:762, P:996 in MiB."""
    s = GOLD["sequential_layer_condition"]
    assert 640 * 512 * 8 * 3 == s["bytes_640x512x3"] == int(s["MiB"] * 2 ** 20)
    assert int(math.sqrt(10 * 2 ** 20 / (9 * 8))) == s["xy_limit_9_layers_10MiB"]


def test_wave_size_a100():
    """108 SMs, 2048 threads/SM, 1024-thread blocks, no register limit -> 216-block wave."""
    k = W.k25(128)
    k["regs"] = 0
    r = O.estimate(k, W.gpu_a100(), ((32, 32, 1), (1, 1, 1), 0))
    assert r["k"] == 2
    assert r["wave_blocks"] == 216


def test_config_errors():
    """ABI conventions: T > max_thr_blk -> ELIMIT, fold 0 -> EINVAL."""
    k = W.k7(16)
    g = W.gpu_v100()
    assert O.estimate(k, g, ((32, 8, 8), (1, 1, 1), 0))["status"] == 2
    assert O.estimate(k, g, ((32, 1, 1), (0, 1, 1), 0))["status"] == 1
    bad = W.k7(16)
    bad["accesses"] = bad["accesses"] + [(0, 0, (2, 0, 0))]
    assert O.check_kernel(bad) == 3


# --------------------------------------------------------------------- independent brute force
SMALL_CASES = [
    (W.k7(12), W.gpu_v100(), ((32, 2, 1), (1, 1, 1), 0)),
    (W.stencil_star(20, 10, 12, 4, regs=64), dict(W.gpu_a100(), n_sm=6), ((8, 4, 2), (1, 1, 2), 1)),
    (W.stencil_star(20, 10, 12, 4, regs=64), dict(W.gpu_a100(), n_sm=5), ((4, 2, 4), (1, 2, 1), 2)),
    (W.lbm15(6), dict(W.gpu_a100(), n_sm=3), ((4, 2, 2), (1, 1, 1), 1)),
]


@pytest.mark.parametrize("case", range(len(SMALL_CASES)))
def test_oracle_vs_independent_sets(case):
    k, g, c = SMALL_CASES[case]
    r = O.estimate(k, g, c)
    m = M.set_counts(k, g, c)
    for key, v in m.items():
        assert r[key] == v, key


@pytest.mark.parametrize("seed", range(12))
def test_oracle_vs_independent_random(seed):
    k, g, c = W.random_kernel(seed, max_dom=9), W.random_gpu(seed), W.random_config(seed)
    r = O.estimate(k, g, c)
    if r["status"] != 0:
        pytest.skip("config rejected")
    m = M.set_counts(k, g, c)
    for key, v in m.items():
        assert r[key] == v, key
    l1 = M.l1_counts(k, g, c)
    for key, v in l1.items():
        assert r[key] == v, key


@pytest.mark.parametrize("case", [0, 1])
def test_oracle_vs_independent_l1(case):
    k, g, c = SMALL_CASES[case]
    r = O.estimate(k, g, c)
    l1 = M.l1_counts(k, g, c)
    for key, v in l1.items():
        assert r[key] == v, key


def test_lru_infinite_capacity_pins():
    """SURVEY 8c pins for a4-a6 via a trace-driven sectored LRU:
    cold misses of the wave = wave_ld_sectors; replaying the L_z then the wave,
    misses inside the wave = wave_ld_sectors - ov_z; with L_y: - ov_y."""
    k = W.stencil_star(16, 8, 12, 4, regs=64)
    g = dict(W.gpu_a100(), n_sm=4)
    c = ((8, 2, 2), (1, 1, 1), 1)
    r = O.estimate(k, g, c)
    geo = M.geometry(k, g, c)
    s, Wb = geo["s"], geo["W"]
    big = 1 << 40
    assert M.replay_blocks(k, g, c, range(s, s + Wb), M.SectoredLRU(big)) == r["wave_ld_sectors"]
    assert M.replay_blocks(k, g, c, range(s, s + Wb), M.SectoredLRU(big), kinds=(1,)) == r["wave_st_sectors"]
    lz0, ly0 = geo["Lz"][0], geo["Ly"][0]
    # stores of the layer set must also be cached (write-back L2, Q15): replay loads and stores
    # of the layer blocks, loads of the wave
    cache = M.SectoredLRU(big)
    M.replay_blocks(k, g, c, range(lz0, s), cache, kinds=(0, 1))
    before = cache.misses
    M.replay_blocks(k, g, c, range(s, s + Wb), cache, kinds=(0,))
    assert cache.misses - before == r["wave_ld_sectors"] - r["ov_z"]
    cache = M.SectoredLRU(big)
    M.replay_blocks(k, g, c, range(ly0, s), cache, kinds=(0, 1))
    before = cache.misses
    M.replay_blocks(k, g, c, range(s, s + Wb), cache, kinds=(0,))
    assert cache.misses - before == r["wave_ld_sectors"] - r["ov_y"]
    # per SM set with infinite capacity: misses = sm_ld_sectors
    tot = 0
    for j in range(r["n_smsets"]):
        tot += M.replay_blocks(k, g, c, list(range(s, s + Wb))[j::g["n_sm"]], M.SectoredLRU(big))
    assert tot == r["sm_ld_sectors"]


def test_lru_capacity_monotone():
    """Finite capacity: misses never decrease as capacity shrinks (S:536 invariant) and are
    bounded below by the compulsory footprint."""
    k = W.stencil_star(16, 8, 8, 4, regs=64)
    g = dict(W.gpu_a100(), n_sm=4)
    c = ((8, 2, 2), (1, 1, 1), 1)
    r = O.estimate(k, g, c)
    geo = M.geometry(k, g, c)
    blocks = range(geo["s"], geo["s"] + geo["W"])
    prev = None
    for cap in [1 << 30, 64 * 1024, 16 * 1024, 4 * 1024, 1024]:
        m = M.replay_blocks(k, g, c, blocks, M.SectoredLRU(cap))
        assert m >= r["wave_ld_sectors"]
        if prev is not None:
            assert m >= prev
        prev = m


# --------------------------------------------------------------------- invariants
@pytest.mark.parametrize("seed", range(20, 40))
def test_invariants_random(seed):
    k, g, c = W.random_kernel(seed), W.random_gpu(seed), W.random_config(seed)
    r = O.estimate(k, g, c)
    if r["status"] != 0:
        return
    assert r["sm_ld_lines"] <= r["sm_ld_sectors"] <= 4 * r["sm_ld_lines"]
    assert r["sm_ld_sectors"] <= r["l1_req_ld_sectors"]
    if not (len(c) > 3 and c[3] & 8):   # the representative block need not bound the wave
        assert r["wave_ld_sectors"] <= r["sm_ld_sectors"]
        assert r["wave_st_sectors"] <= r["l1_req_st_sectors"]
    assert r["ov_y"] <= r["ov_z"] <= r["wave_ld_sectors"]
    assert r["ly_lines"] <= r["lz_lines"]
    # shifting every field by 128 B changes nothing (sectors/lines/banks are 128 B periodic)
    k2 = dict(k, fields=[dict(f, align=f["align"] + 128) for f in k["fields"]])
    r2 = O.estimate(k2, g, c)
    for key in M.set_counts.__code__.co_varnames[:0] or ["l1_wavefronts", "l1_req_ld_sectors", "sm_ld_sectors",
                                                          "wave_ld_sectors", "wave_lines", "lz_lines", "ov_z"]:
        assert r2[key] == r[key]
    # access order permutation
    k3 = dict(k, accesses=list(reversed(k["accesses"])))
    r3 = O.estimate(k3, g, c)
    for key in ["l1_wavefronts", "l1_req_ld_sectors", "l1_req_st_sectors", "sm_ld_lines", "wave_ld_sectors",
                "wave_st_sectors", "ly_lines", "lz_lines", "ov_y", "ov_z", "t_pred"]:
        assert r3[key] == r[key]


# --------------------------------------------------------------------- NEXT-3 / NEXT-4 variants
VAR_MDIM, VAR_PREV_WAVE, VAR_L2_DUP, VAR_REP_BLOCK = 1, 2, 4, 8


def _plain_kernel(ext, accesses, align=0, elem=8, dom_lo=(0, 0, 0), dom_hi=None):
    ex, ey, ez = ext
    f = {"extent": ext, "pitch": (1, ex, ex * ey), "align": align, "elem": elem}
    nf = 1 + max(a[0] for a in accesses)
    return {"fields": [dict(f) for _ in range(nf)], "accesses": accesses, "dom_lo": dom_lo,
            "dom_hi": dom_hi or ext, "regs": 0, "flops": 0.0}


def test_mdim_paper_example():
    """P:527-532 + P:557-562: A[tidx][tidy+1] over a 256x2 thread block maps to the 2D address
    (ax = floor(tidx*8/32), ay = tidy+1): 64 x 2 = 128 distinct sectors in the multidimensional
    address space, whatever the alignment.  The linear space with the -1-element
    alignment of P:540 shares one sector between the two rows: 2 * 65 - 1 = 129."""
    k = _plain_kernel((256, 4, 1), [(0, 0, (0, 1, 0))], align=-8, dom_hi=(256, 2, 1))
    g = dict(W.gpu_a100(), n_sm=1)
    c = ((256, 2, 1), (1, 1, 1), 1)
    md = O.estimate(k, g, c + (VAR_MDIM,))
    lin = O.estimate(k, g, c)
    assert md["wave_ld_sectors"] == 128 and md["wave_lines"] == 2 * 16
    assert lin["wave_ld_sectors"] == 129
    # the warp / SM-set scopes keep linear addresses (explicit grid iteration)
    for key in ("l1_req_ld_sectors", "l1_wavefronts", "sm_ld_sectors", "sm_ld_lines"):
        assert md[key] == lin[key], key


@pytest.mark.parametrize("seed", range(4))
def test_mdim_alignment_invariance_and_line_rows(seed):
    """Multidimensional counts ignore the alignment; with line-multiple rows and a
    line-aligned base, the two address spaces count the same sets (no row shares a line)."""
    k = W.stencil_star(24, 10, 12, 1 + seed % 2, regs=0)   # rows of 26 / 28 doubles
    g = dict(W.gpu_a100(), n_sm=4)
    c = ((8, 2, 2), (1, 1 + seed % 2, 1), 1, VAR_MDIM)
    r0 = O.estimate(k, g, c)
    keys = ["wave_ld_sectors", "wave_st_sectors", "wave_lines", "ly_lines", "lz_lines", "ov_y", "ov_z"]
    for shift in (8, 24, 64 + 16 * seed):
        k2 = dict(k, fields=[dict(f, align=f["align"] + shift) for f in k["fields"]])
        r2 = O.estimate(k2, g, c)
        for key in keys:
            assert r2[key] == r0[key], (shift, key)
    # pad the rows to 32 doubles = 2 lines: linear == multidimensional
    kp = dict(k, fields=[dict(f, pitch=(1, 32, 32 * f["extent"][1])) for f in k["fields"]])
    a, b = O.estimate(kp, g, c[:3]), O.estimate(kp, g, c)
    for key in keys:
        assert a[key] == b[key], key


@pytest.mark.parametrize("d", [1, 2, 4, 8, 16])
def test_prev_wave_series(d):
    """P:583-587 (SBAC, V100): reuse only from the directly preceding wave.  A wave of 16 full
    rows, d planes deep, in the middle of a block layer: the previous wave holds exactly its
    y-neighbour rows, so with R = 1 the DRAM load is the P:993 series 8(d+8)/d B/Lup (+ the
    64/XS x-halo), independent of the z curve."""
    k = W.stencil_star(XS, 64, 64, 4, regs=0)
    g = W.gpu_a100()
    g["n_sm"] = 16
    g["hit_abc"][1] = [1.0, 0.0, 0.0]
    g["hit_abc"][2] = [0.0, 0.0, 0.0]
    r = O.estimate(k, g, ((XS, 1, 1), (1, 1, d), 1, VAR_PREV_WAVE))
    assert r["ov_y"] == r["ov_z"] and r["ly_lines"] == r["lz_lines"]
    assert r["dram_ld_Bpl"] == pytest.approx(8 * (d + 8) / d + 64 / XS, rel=1e-12)


def test_prev_wave_lru_pin():
    """Cold sectored LRU replaying the previous wave (loads + stores) then the wave's loads:
    misses inside the wave = wave_ld_sectors - ov_y (exact at infinite capacity)."""
    k = W.stencil_star(16, 8, 12, 4, regs=64)
    g = dict(W.gpu_a100(), n_sm=4)
    c = ((8, 2, 2), (1, 1, 1), 1, VAR_PREV_WAVE)
    r = O.estimate(k, g, c)
    geo = M.geometry(k, g, c)
    s, Wb = geo["s"], geo["W"]
    assert geo["Ly"] == (max(0, s - Wb), s)
    cache = M.SectoredLRU(1 << 40)
    M.replay_blocks(k, g, c, range(max(0, s - Wb), s), cache, kinds=(0, 1))
    before = cache.misses
    M.replay_blocks(k, g, c, range(s, s + Wb), cache, kinds=(0,))
    assert cache.misses - before == r["wave_ld_sectors"] - r["ov_y"] > 0


@pytest.mark.parametrize("align,pages_per_plane", [(0, 2), (8, 3)])
def test_tlb_pages_hand_count(align, pages_per_plane):
    """TLB pages accessed by the current wave.  Copy kernel B[c] = A[c] on
    1024 x 64 x 64 doubles (8 KiB rows), 64 KiB pages, a wave of 16 rows x d planes at rows
    24..39 of each plane = bytes [192 KiB, 320 KiB) of the plane: 2 pages per plane and field,
    3 when the field starts 8 B past a page boundary."""
    d = 4
    k = _plain_kernel((1024, 64, 64), [(0, 0, (0, 0, 0)), (1, 1, (0, 0, 0))], align=align)
    g = dict(W.gpu_a100(), n_sm=16, page_bytes=64 * 1024)
    r = O.estimate(k, g, ((1024, 1, 1), (1, 1, d), 1))
    assert r["wave_first_block"] % 64 == 24
    assert r["wave_pages"] == 2 * d * pages_per_plane
    assert O.estimate(k, dict(g, page_bytes=0), ((1024, 1, 1), (1, 1, d), 1))["wave_pages"] == 0


def test_l2_sections_duplication_and_link_hand_count():
    """4 SMs in 2 L2 sections (SMs 0,1 | 2,3), a wave of 4 one-row
    blocks; a 3-point y stencil loads rows y-1..y+1.  Section 0 (rows y0, y0+1) and section 1
    (rows y0+2, y0+3) both load rows y0+1, y0+2: 2 rows x 64 sectors cross the link and
    2 rows x 16 lines are held twice; the stored rows are disjoint."""
    k = _plain_kernel((256, 32, 1), [(0, 0, (0, -1, 0)), (0, 0, (0, 0, 0)), (0, 0, (0, 1, 0)),
                                      (1, 1, (0, 0, 0))], dom_lo=(0, 1, 0), dom_hi=(256, 31, 1))
    g = dict(W.gpu_a100(), n_sm=4, l2_sections=2, link_bw=1e12)
    c = ((256, 1, 1), (1, 1, 1), 1)
    r = O.estimate(k, g, c)
    assert r["l2_link_sectors"] == 128 and r["l2_dup_lines"] == 32
    n = r["lup_wave"]
    assert n == 4 * 256
    assert r["t_link"] == pytest.approx(32 * 128 / (n * 1e12), rel=1e-15)
    assert r["l2_eff_bytes"] == g["l2_bytes"] / 2                 # default: full duplication
    rd = O.estimate(k, g, c + (VAR_L2_DUP,))
    U = 6 * 16 + 4 * 16                                            # distinct lines: 6 load rows + 4 store rows
    assert rd["l2_eff_bytes"] == pytest.approx(g["l2_bytes"] * U / (U + 32), rel=1e-15)
    r1 = O.estimate(k, dict(g, l2_sections=1), c + (VAR_L2_DUP,))
    assert r1["l2_dup_lines"] == r1["l2_link_sectors"] == 0 and r1["l2_eff_bytes"] == g["l2_bytes"]
    # link-limited once the link is slow enough; limiter code 3
    rs = O.estimate(k, dict(g, link_bw=1e6), c)
    assert rs["limiter"] == 3 and rs["t_pred"] == pytest.approx(rs["t_link"] * 256 * 30, rel=1e-12)


@pytest.mark.parametrize("variant", [1, 2, 4, 7, 8, 15])
@pytest.mark.parametrize("case", range(len(SMALL_CASES)))
def test_oracle_vs_independent_variants(case, variant):
    k, g, c = SMALL_CASES[case]
    g = dict(g, page_bytes=1024, l2_sections=3 if case % 2 else 2)
    c = c + (variant,)
    r = O.estimate(k, g, c)
    m = M.set_counts(k, g, c)
    for key, v in m.items():
        assert r[key] == v, key
    if variant & VAR_REP_BLOCK:
        for key, v in M.l1_counts(k, g, c).items():
            assert r[key] == v, key


@pytest.mark.parametrize("k_res", [1, 2])
def test_rep_block_equals_exact_on_translation_invariant_grid(k_res):
    """one representative block stands for the wave.  On a grid whose blocks are all
    unclipped translates by whole lines (rows of 128 doubles = 8 lines, 16-wide blocks, aligned
    base), every block has the same warp statistics and footprint, so with one block per SM set
    the representative-block variant reproduces the exact per-SM-set counts; with two blocks per
    set it can only over-count (co-resident blocks share nothing under the variant)."""
    n = 128
    ext = (n + 2, 34, 34)
    fld = {"extent": ext, "pitch": (1, 128 * 2, 128 * 2 * 34), "align": 8 * 127, "elem": 8}
    k = {"fields": [dict(fld), dict(fld)], "accesses": [(0, 0, (0, 0, 0)), (0, 0, (1, 0, 0)), (0, 0, (-1, 0, 0)),
                                                        (0, 0, (0, 1, 0)), (0, 0, (0, -1, 0)), (0, 0, (0, 0, 1)),
                                                        (0, 0, (0, 0, -1)), (1, 1, (0, 0, 0))],
         "dom_lo": (1, 1, 1), "dom_hi": (n + 1, 33, 33), "regs": 0, "flops": 7.0}
    g = dict(W.gpu_a100(), n_sm=4)
    c = ((16, 4, 2), (1, 1, 1), k_res)
    exact, rep = O.estimate(k, g, c), O.estimate(k, g, c + (VAR_REP_BLOCK,))
    for key in ("lup_wave", "l1_wavefronts", "l1_req_ld_sectors", "l1_req_st_sectors"):
        assert rep[key] == exact[key], key
    if k_res == 1:
        assert rep["sm_ld_sectors"] == exact["sm_ld_sectors"] and rep["sm_ld_lines"] == exact["sm_ld_lines"]
    else:
        assert rep["sm_ld_sectors"] >= exact["sm_ld_sectors"] and rep["sm_ld_lines"] >= exact["sm_ld_lines"]
    for key in ("wave_ld_sectors", "wave_lines", "lz_lines", "ov_z"):   # wave scopes untouched
        assert rep[key] == exact[key], key


# --------------------------------------------------------------------- NEXT-1: simulated hit rates
SIM_CASES = [
    (W.stencil_star(24, 12, 12, 4, regs=64), dict(W.gpu_a100(), n_sm=6), ((8, 2, 2), (1, 1, 1), 1)),
    (W.stencil_star(20, 10, 12, 1, regs=0), dict(W.gpu_a100(), n_sm=4), ((4, 4, 2), (1, 1, 2), 2)),
    (W.lbm15(8), dict(W.gpu_a100(), n_sm=3), ((4, 2, 2), (1, 1, 1), 1)),
]


def test_textbook_lru_cyclic():
    """Pins the independent LRU used below: cycling over n lines misses every time with
    capacity n - 1 lines and only the n compulsory times with capacity n."""
    for n in (3, 7):
        for cap, misses in ((n - 1, 3 * n), (n, n)):
            c = M.SectoredLRU(cap * 128)
            for _ in range(3):
                for i in range(n):
                    c.access((0, 4 * i))
            assert c.misses == misses


@pytest.mark.parametrize("case", range(len(SIM_CASES)))
def test_sim_infinite_capacity(case):
    """With a cache larger than every footprint, the simulator's misses are the compulsory
    footprints the estimator counts exactly: SM-set sectors, wave store sectors, and
    every overlap sector of the layer sets is still resident (R = 1)."""
    k, g, c = SIM_CASES[case]
    r = O.estimate(k, g, c)
    s = O.simulate_batch(k, g, [c], [1 << 40])[0][0]
    assert s["status"] == 0
    assert s["l1_requests"] == r["l1_req_ld_sectors"] and s["st_requests"] == r["l1_req_st_sectors"]
    assert s["l1_misses"] == s["l1_compulsory"] == r["sm_ld_sectors"]
    assert s["st_misses"] == s["st_compulsory"] == r["wave_st_sectors"]
    assert s["ov_y"] == s["y_resident"] == r["ov_y"]
    assert s["ov_z_only"] == s["z_resident"] == r["ov_z"] - r["ov_y"]
    assert s["R_l1"] == s["R_y"] == s["R_z"] == s["R_st"] == 1.0


@pytest.mark.parametrize("case", range(len(SIM_CASES)))
def test_sim_vs_independent_lru(case):
    """Finite capacities: the oracle's counts equal an independent replay (numpy per-thread
    traces grouped into warp requests, OrderedDict LRU) of the same request streams."""
    k, g, c = SIM_CASES[case]
    caps = [2048, 8192, 32768]
    sims = O.simulate_batch(k, g, [c], caps)[0]
    geo = M.geometry(k, g, c)
    s, Wb, nsm = geo["s"], geo["W"], g["n_sm"]
    wave = list(range(s, s + Wb))
    for cap, sim in zip(caps, sims):
        l1 = 0
        for j in range(min(nsm, Wb)):
            cache = M.SectoredLRU(cap)
            for B in wave[j::nsm]:
                for key, st in M.warp_requests(k, geo, B, (0,)):
                    cache.access(key)
            l1 += cache.misses
        assert sim["l1_misses"] == l1
        cache, stm = M.SectoredLRU(cap), 0
        for B in wave:
            for key, st in M.warp_requests(k, geo, B, (0, 1)):
                before = cache.misses
                cache.access(key)
                stm += st * (cache.misses - before)
        assert sim["st_misses"] == stm
        cache = M.SectoredLRU(cap)
        for B in range(*geo["Lz"]):
            for key, st in M.warp_requests(k, geo, B, (0, 1)):
                cache.access(key)
        WLD = {key for B in wave for key, st in M.warp_requests(k, geo, B, (0,))}
        FY = {key for B in range(*geo["Ly"]) for key, st in M.warp_requests(k, geo, B, (0, 1))}
        FZ = {key for B in range(*geo["Lz"]) for key, st in M.warp_requests(k, geo, B, (0, 1))}

        def valid(key):
            line = (key[0], key[1] // 4)
            return line in cache.lines and key[1] in cache.lines[line]
        assert sim["y_resident"] == sum(valid(x) for x in WLD & FY)
        assert sim["z_resident"] == sum(valid(x) for x in (WLD & FZ) - FY)


def test_sim_monotone_in_capacity():
    """simulated hit rates never increase as the capacity shrinks."""
    k, g, c = SIM_CASES[0]
    caps = [1 << 20, 65536, 16384, 4096, 1024, 128]
    sims = O.simulate_batch(k, g, [c], caps)[0]
    for a, b in zip(sims, sims[1:]):
        assert b["l1_misses"] >= a["l1_misses"] and b["st_misses"] >= a["st_misses"]
        assert b["y_resident"] <= a["y_resident"] and b["z_resident"] <= a["z_resident"]
        assert b["O_z"] > a["O_z"]


def test_fit_recovers_known_curve():
    """SPEC S:603 round trip: exact samples of a known curve are fitted to 1e-9; with 1 %
    (deterministic) noise within 5 % per parameter.  SPEC's own example (1.0, 5.0, -2.0) is
    nearly flat at 0 on O >= 0 (R(0) = e^-5) and its parameters are not identifiable from noisy
    samples, so the noisy case uses a curve of the paper's shape ("close to one and then quickly
    drops"): (0.95, 0.02, -3.0)."""
    Os = [0.05 * i for i in range(60)]
    exact = [O.hit_rate([1.0, 5.0, -2.0], o) for o in Os]
    (a, b, c), rss = O.fit_gompertz(Os, exact)
    assert (a, b, c) == pytest.approx((1.0, 5.0, -2.0), rel=1e-9) and rss < 1e-20
    exact = [O.hit_rate([0.95, 0.02, -3.0], o) for o in Os]
    noisy = [r * (1 + 0.01 * math.sin(7.0 * i)) for i, r in enumerate(exact)]
    (a, b, c), rss = O.fit_gompertz(Os, noisy)
    assert (a, b, c) == pytest.approx((0.95, 0.02, -3.0), rel=0.05)
    # the paper's decreasing orientation is recovered from simulated z-layer samples
    k, g, cfg = SIM_CASES[0]
    sims = O.simulate_batch(k, g, [cfg], [1 << 20, 131072, 65536, 32768, 16384, 8192, 4096, 2048])[0]
    (a, b, c), rss = O.fit_gompertz([s["O_z"] for s in sims], [s["R_z"] for s in sims])
    assert c < 0 and O.hit_rate([a, b, c], 1.0) > O.hit_rate([a, b, c], 4.0)


# --------------------------------------------------------------------- NEXT-2: validation stencil definition
def test_stencil25_definition_pins():
    """The plain stencil: a constant field maps to (w0 + 6 sum w_k) * const (the weights sum to
    the discrete Laplacian's zero row sum up to w0 + 6 sum w_k); a delta at one cell spreads
    exactly to its 25 star neighbours with the weights; ghost layers stay untouched."""
    from oracle import stencil as ST
    n = (12, 10, 9)
    src = np.full((n[2] + 8, n[1] + 8, n[0] + 8), 2.0)
    dst = ST.stencil25(src, n)
    tot = ST.W[0] + 6 * sum(ST.W[1:])
    assert np.allclose(dst[4:-4, 4:-4, 4:-4], 2.0 * tot, rtol=1e-14)
    assert not dst[:4].any() and not dst[:, :, -4:].any()
    src = np.zeros_like(src)
    src[8, 9, 10] = 1.0                    # cell (x=10, y=9, z=8)
    dst = ST.stencil25(src, n)
    assert dst[8, 9, 10] == ST.W[0]
    for k in range(1, 5):
        for dz, dy, dx in ((0, 0, k), (0, k, 0), (k, 0, 0)):
            for sgn in (-1, 1):
                z, y, x = 8 + sgn * dz, 9 + sgn * dy, 10 + sgn * dx
                if 4 <= z < n[2] + 4 and 4 <= y < n[1] + 4 and 4 <= x < n[0] + 4:
                    assert dst[z, y, x] == ST.W[k]
    assert np.count_nonzero(dst) <= 25


def test_lbm15_definition_pins():
    """The plain LBM15 update: the weights sum to 1 (2/9 + 6/9 + 8/72), so a uniform state
    (f_q = w_q rho0, constant phi) is a fixed point (feq = f), the streaming pull moves a single
    population exactly by c_q, and the FD result is the 7-point Laplacian."""
    from oracle import stencil as ST
    n = (6, 5, 4)
    w = [2.0 / 9.0] + [1.0 / 9.0] * 6 + [1.0 / 72.0] * 8
    assert abs(sum(w) - 1.0) < 1e-15
    src = np.stack([np.full((n[2] + 2, n[1] + 2, n[0] + 2), wq * 1.7) for wq in w])
    phi = np.zeros((n[2] + 2, n[1] + 2, n[0] + 2))
    dst, fd = ST.lbm15(src, phi, n)
    assert np.allclose(dst[:, 1:-1, 1:-1, 1:-1], src[:, 1:-1, 1:-1, 1:-1], rtol=1e-14)
    assert not fd.any()
    src = np.zeros_like(src)
    src[8, 2, 2, 2] = 1.0                       # population q=8, c = (-1,-1,1) at cell (2,2,2)
    dst, _ = ST.lbm15(src, phi, n)
    c = ST.Q15[8]
    z, y, x = 2 + c[2], 2 + c[1], 2 + c[0]      # pulled from cell - c: lands at cell + c
    om = 1.2
    assert dst[8, z, y, x] == pytest.approx(1.0 + om * (1.0 / 72.0 * (1.0 + 3.0 * 3.0) - 1.0), rel=1e-14)
    phi[3, 3, 3] = 1.0
    _, fd = ST.lbm15(np.zeros_like(src), phi, n)
    assert fd[3, 3, 3] == -6.0 and fd[3, 3, 4] == 1.0 and fd[2, 3, 3] == 1.0


# --------------------------------------------------------------------- a6 (O), a7 closed forms (round 2)
# Each pin below is a value written out by hand from the definition of the term it checks (not
# the oracle's formula retyped): scripts/oracle_mutations.py builds deliberately broken oracles
# (a dropped factor, a swapped bandwidth, a wrong divisor, a dropped term) and records that
# these tests fail for each one (profiles/r02_oracle_mutations.md).
def _copy_kernel(X, Y, Z, loads=((0, 0, 0),), store=True, elem=8):
    """dst[c] = f(src[c + o] for o in loads): dense, 0-aligned fields, no ghost layers in y/z."""
    hx = max(max(abs(o[0]) for o in loads), 0)
    ext = (X + 2 * hx, Y, Z)
    fld = {"extent": ext, "pitch": (1, ext[0], ext[0] * ext[1]), "align": 0, "elem": elem}
    acc = [(0, 0, o) for o in loads] + ([(1, 1, (0, 0, 0))] if store else [])
    return {"name": "copy", "fields": [fld, dict(fld)] if store else [fld], "accesses": acc,
            "dom_lo": (hx, 0, 0), "dom_hi": (hx + X, Y, Z), "regs": 0, "flops": 0.0}


def _flat_gpu(n_sm=1, **kw):
    g = W.gpu_a100()
    g["n_sm"] = n_sm
    g["hit_abc"] = [[1.0, 0.0, 0.0] for _ in range(4)]
    g.update(kw)
    return g


def test_limiter_dram_floor_87_5_glups():
    """S:468 / S:649-650 (P:262-281 limiters, Table tab:av100 P:313 1400 GB/s): a stencil at the
    8 B/Lup load + 8 B/Lup store floor runs at 1400/16 = 87.5 GLup/s; load-only at 175 GLup/s.
    Streaming copy, 128-wide rows (whole lines), no reuse possible -> exactly 8 + 8 B/Lup."""
    X, Y, Z = 128, 16, 16
    g = W.gpu_a100()
    cells = X * Y * Z
    r = O.estimate(_copy_kernel(X, Y, Z), g, ((128, 1, 1), (1, 1, 1), 0))
    assert (r["dram_ld_Bpl"], r["dram_st_Bpl"]) == (8.0, 8.0)
    assert r["limiter"] == 2
    assert cells / r["t_pred"] == pytest.approx(87.5e9, rel=1e-12)
    r = O.estimate(_copy_kernel(X, Y, Z, store=False), g, ((128, 1, 1), (1, 1, 1), 0))
    assert r["dram_ld_Bpl"] == 8.0 and r["dram_st_Bpl"] == 0.0
    assert cells / r["t_pred"] == pytest.approx(175e9, rel=1e-12)


def test_limiter_l2_and_l1_absolute():
    """L2 limiter = (L2<->L1 loads + stores) / L2 bandwidth: the copy moves 8 + 8 B/Lup
    through L2 -> 5000e9 / 16 = 312.5 GLup/s (A100 L2 5000 GB/s) when DRAM is not the
    bottleneck.  L1 limiter = cycles per LUP / (n_sm * clock): a half-warp instruction over 16
    consecutive doubles is one wavefront, two instructions per LUP, 16 LUP per
    half-warp -> 1/8 cycle per LUP -> 108 * 1.41e9 * 8 = 1.21824e12 LUP/s."""
    X, Y, Z = 128, 16, 16
    cells = X * Y * Z
    g = dict(W.gpu_a100(), dram_bw=1e18)
    r = O.estimate(_copy_kernel(X, Y, Z), g, ((128, 1, 1), (1, 1, 1), 0))
    assert (r["l2_ld_Bpl"], r["l2_st_Bpl"]) == (8.0, 8.0)
    assert r["limiter"] == 1
    assert cells / r["t_pred"] == pytest.approx(312.5e9, rel=1e-12)
    g = dict(W.gpu_a100(), dram_bw=1e18, l2_bw=1e18)
    r = O.estimate(_copy_kernel(X, Y, Z), g, ((128, 1, 1), (1, 1, 1), 0))
    assert r["l1_cyc_per_lup"] == 0.125 and r["limiter"] == 0
    assert cells / r["t_pred"] == pytest.approx(108 * 1.41e9 * 8, rel=1e-12)


def test_eq5_capacity_term_hand_count():
    """Eq. 5 ("V_up=100, V_comp=60, R=.75 -> 10"): V_down = V_comp + (1-R)(V_up -
    V_comp) at the L1 level.  One 32-thread block, 1D 3-point load src[x-1], src[x], src[x+1] on
    doubles at x = 8..39 (addresses 56..327 B): the three warp instructions touch 9 + 8 + 9 = 26
    sectors (V_up), their union is sectors 1..10 = 10 (V_comp).  With R_L1 = 0.75:
    V_down = 10 + 0.25 * 16 = 14 sectors -> 14 * 32 / 32 LUP = 14 B/Lup."""
    k = _copy_kernel(32, 1, 1, loads=((-1, 0, 0), (0, 0, 0), (1, 0, 0)), store=False)
    k["fields"][0] = dict(k["fields"][0], extent=(48, 1, 1), pitch=(1, 48, 48))
    k["dom_lo"], k["dom_hi"] = (8, 0, 0), (40, 1, 1)
    g = _flat_gpu()
    g["hit_abc"][0] = [0.75, 0.0, 0.0]
    r = O.estimate(k, g, ((32, 1, 1), (1, 1, 1), 1))
    assert (r["l1_req_ld_sectors"], r["sm_ld_sectors"], r["sm_ld_lines"]) == (26, 10, 3)
    assert r["R_l1"] == 0.75
    assert r["l2_ld_Bpl"] == pytest.approx(14.0, rel=1e-15)
    g["hit_abc"][0] = [0.0, 0.0, 0.0]            # R = 0 -> V_up; R = 1 -> V_comp
    assert O.estimate(k, g, ((32, 1, 1), (1, 1, 1), 1))["l2_ld_Bpl"] == pytest.approx(26.0, rel=1e-15)
    g["hit_abc"][0] = [1.0, 0.0, 0.0]
    assert O.estimate(k, g, ((32, 1, 1), (1, 1, 1), 1))["l2_ld_Bpl"] == pytest.approx(10.0, rel=1e-15)


def test_eq4_oversubscription_l1_hand_count():
    """Eq. 4 (O = V_alloc / V_cache) at L1 with the SM set's 128 B line footprint (P:474-475,
    Q8/Q18), averaged over the SM sets.  Two 32-thread blocks of the 3-point load at x = 8..71:
    one SM with k = 2 holds both blocks: addresses 56..583 B -> lines 0..4 = 5 lines = 640 B;
    L1 = 1280 B -> O = 0.5.  Two SMs, one block each: lines 0..2 and 2..4 -> 3 lines per set on
    average = 384 B -> O = 0.3.  R_L1 = R(O) on the set's O."""
    k = _copy_kernel(64, 1, 1, loads=((-1, 0, 0), (0, 0, 0), (1, 0, 0)), store=False)
    k["fields"][0] = dict(k["fields"][0], extent=(80, 1, 1), pitch=(1, 80, 80))
    k["dom_lo"], k["dom_hi"] = (8, 0, 0), (72, 1, 1)
    abc = [1.0, 0.5, -2.0]
    g = _flat_gpu(n_sm=1, l1_bytes=1280)
    g["hit_abc"][0] = abc
    r = O.estimate(k, g, ((32, 1, 1), (1, 1, 1), 2))
    assert (r["n_smsets"], r["sm_ld_lines"]) == (1, 5)
    assert r["O_l1"] == 0.5
    assert r["R_l1"] == pytest.approx(math.exp(-0.5 * math.exp(1.0)), rel=1e-15)
    g = _flat_gpu(n_sm=2, l1_bytes=1280)
    r = O.estimate(k, g, ((32, 1, 1), (1, 1, 1), 1))
    assert (r["n_smsets"], r["sm_ld_lines"]) == (2, 6)
    assert r["O_l1"] == pytest.approx(0.3, rel=1e-15)


def test_eq4_oversubscription_layer_sets_o_z_equals_one():
    """SURVEY 8(c) "a6 (O)": O_z = 1 exactly when the z-layer set's line footprint equals the
    effective L2 (split L2 = l2_bytes / sections, Q31).  Copy kernel on a
    60 x 8 x 8 domain in rows padded to 64 doubles (512 B, line-aligned), one 64-thread block per
    row (Gx = 1, Gy = 8): a row of 60 doubles is 15 sectors but 4 lines.  L_y = the previous row
    (src + dst = 8 lines), L_z = the previous 8 rows = one z-layer (64 lines).  l2_bytes = 16 KiB
    in 2 sections -> L2_eff = 8 KiB: O_y = 1024/8192 = 0.125, O_z = 8192/8192 = 1 (the sector
    footprint would give 960/8192 and 7680/8192).  Store curve: O_st = wave lines /
    L2_eff with the 2-block wave (2 rows x 2 fields x 4 lines = 16 lines)."""
    k = _copy_kernel(60, 8, 8)
    for f in k["fields"]:
        f.update(extent=(64, 8, 8), pitch=(1, 64, 512))
    g = _flat_gpu(n_sm=2, l2_bytes=16384, l2_sections=2)
    r = O.estimate(k, g, ((64, 1, 1), (1, 1, 1), 1))
    assert r["wave_blocks"] == 2 and r["wave_first_block"] >= 8
    assert (r["ly_lines"], r["lz_lines"], r["wave_lines"]) == (8, 64, 16)
    assert r["l2_eff_bytes"] == 8192.0
    assert (r["O_y"], r["O_z"]) == (0.125, 1.0)
    assert r["O_st"] == 16 * 128 / 8192
    # the copy reads nothing twice: no overlap with either layer set
    assert (r["ov_y"], r["ov_z"]) == (0, 0)


def test_partial_store_readback_hand_count():
    """P:519-521 (Q19): redundant partial stores (several warp instructions storing parts of one
    sector) that miss in L2 are read back from DRAM: cap_st = (1 - R_st) * (req_st - wave_st).
    Copy on a 4 x 16 domain of doubles, rows of 4 = exactly one sector, blocks (2,16,1): the two
    blocks store the two halves of every row's sector -> 32 store-sector requests, 16 distinct;
    loads likewise 16 distinct sectors.  R_st = 0.5 -> DRAM loads = 16 + 0.5 * 16 = 24 sectors
    = 24 * 32 B / 64 LUP = 12 B/Lup (8 without the read-back), DRAM stores 8 B/Lup."""
    k = _copy_kernel(4, 16, 1)
    g = _flat_gpu(n_sm=2)
    g["hit_abc"][3] = [0.5, 0.0, 0.0]
    r = O.estimate(k, g, ((2, 16, 1), (1, 1, 1), 1))
    assert (r["wave_blocks"], r["lup_wave"]) == (2, 64)
    assert (r["l1_req_st_sectors"], r["wave_st_sectors"], r["wave_ld_sectors"]) == (32, 16, 16)
    assert r["R_st"] == 0.5
    assert r["dram_ld_Bpl"] == 12.0 and r["dram_st_Bpl"] == 8.0
    # L1 -> L2 stores are written through per warp instruction: 32 sectors = 16 B/Lup;
    # L2 -> L1 loads: each block's SM fetches the row sectors it reads: 2 x 16 sectors = 16 B/Lup
    assert r["l2_st_Bpl"] == 16.0 and r["l2_ld_Bpl"] == 16.0
    g["hit_abc"][3] = [1.0, 0.0, 0.0]
    assert O.estimate(k, g, ((2, 16, 1), (1, 1, 1), 1))["dram_ld_Bpl"] == 8.0


def test_alignment_must_be_element_multiple():
    """align_bytes not a multiple of elem_bytes is WS_EINVAL (an element would
    straddle two sectors); negative multiples are valid (P:540 uses -1 element)."""
    k = W.k7(8)
    k["fields"][0] = dict(k["fields"][0], align=4)
    assert O.check_kernel(k) == 1
    assert O.estimate(k, W.gpu_v100(), ((32, 1, 1), (1, 1, 1), 0))["status"] == 1
    k["fields"][0] = dict(k["fields"][0], align=-8)
    assert O.check_kernel(k) == 0


@pytest.mark.parametrize("seed", range(6))
def test_oracle_vs_independent_negative_alignment(seed):
    """Negative alignments (P:540-545 uses -1 element): floor division of negative addresses in the
    oracle vs Python's floor semantics in the independent model, every scope."""
    import random
    k, g, c = W.random_kernel(900 + seed, max_dom=8), W.random_gpu(seed), W.random_config(seed)
    rng = random.Random(seed)
    for f in k["fields"]:
        f["align"] = -f["elem"] * rng.randint(1, 300)
    r = O.estimate(k, g, c)
    if r["status"] != 0:
        pytest.skip("config rejected")
    for key, v in M.set_counts(k, g, c).items():
        assert r[key] == v, key
    for key, v in M.l1_counts(k, g, c).items():
        assert r[key] == v, key
