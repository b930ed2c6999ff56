"""Seeded, synthetic input descriptions shared by the oracle and the CUDA path.

This module holds NO arithmetic of the estimator: it only builds plain
descriptions of kernels (fields + affine accesses),
hardware parameter sets (Table tab:av100) and configuration
spaces.  Both `oracle/` and `paper_2204_14242_b200/` consume
these dictionaries; neither imports the other.

Descriptions
------------
kernel = {
  "name": str,
  "fields": [ {"extent": (ex,ey,ez), "pitch": (1,py,pz), "align": bytes, "elem": bytes}, ... ],
  "accesses": [ (field_index, is_store, (ox,oy,oz)), ... ],   # x fastest
  "dom_lo": (x,y,z), "dom_hi": (x,y,z),                       # field-index coords
  "regs": registers per thread (0 = ignore register limit),
  "flops": flops per lattice update,
}
gpu = dict with the ws_gpu fields (see include/ws.h).
config = (block (bx,by,bz), fold (fx,fy,fz), blocks_per_sm override or 0)
"""
from __future__ import annotations

import itertools
import random

MiB = 1 << 20
KiB = 1 << 10

# ---------------------------------------------------------------------------
# Hit-rate curve parameters (a, b, c) for R(O) = a*exp(-b*exp(-c*O)).
# The paper prints no values; these are SURVEY.md Q17's readings (c < 0 so
# the curve falls with oversubscription).  Order: L1, L2-over-y, L2-over-z,
# L2-store.
# ---------------------------------------------------------------------------
HIT_ABC_DEFAULT = (
    (1.0, 0.0068973, -2.72625),   # L1: R(1)=0.90, R(2)=0.20
    (1.0, 0.0376847, -1.02813),   # L2 over y: R(1)=0.90, R(4)=0.10
    (1.0, 0.0037056, -3.34756),   # L2 over z: R(1)=0.90, R(2)=0.05
    (1.0, 0.0076557, -1.90211),   # L2 store: R(1)=0.95
)


def _gpu(name, n_sm, clock_hz, l1_bytes, l2_bytes, l2_sections, dram_bw, l2_bw,
         max_thr_sm=2048, max_blk_sm=32, max_thr_blk=1024, regs_sm=65536,
         hit_abc=HIT_ABC_DEFAULT):
    return {
        "name": name, "n_sm": n_sm, "clock_hz": float(clock_hz),
        "l1_bytes": int(l1_bytes), "l2_bytes": int(l2_bytes), "l2_sections": l2_sections,
        "dram_bw": float(dram_bw), "l2_bw": float(l2_bw),
        "max_thr_sm": max_thr_sm, "max_blk_sm": max_blk_sm,
        "max_thr_blk": max_thr_blk, "regs_sm": regs_sm,
        "sector_bytes": 32, "line_bytes": 128, "n_banks": 16, "bank_bytes": 8,
        "half_warp": 16, "pair_window_bytes": 1024,
        "hit_abc": [list(t) for t in hit_abc],
    }


def gpu_v100():
    """Table tab:av100: 80 SM, 1.38 GHz, 128 kB L1, 6 MB L2, 800/2500 GB/s."""
    return _gpu("V100", 80, 1.38e9, 128 * KiB, 6 * MiB, 1, 800e9, 2500e9)


def gpu_a100():
    """Table tab:av100: 108 SM, 1.41 GHz, 192 kB L1, 2x20 MB L2 (split), 1400/5000 GB/s."""
    return _gpu("A100", 108, 1.41e9, 192 * KiB, 40 * MiB, 2, 1400e9, 5000e9)


def gpu_b200_like(hbm_gbs=6546.2):
    """B200-like parameter set (architecture exploration, BJ configs[3]).

    148 SMs, 1.965 GHz max SM clock, 256 KiB unified L1, 126 MB L2 on two dies
    (l2_sections=2 by analogy with the A100 split), DRAM bandwidth
    = the measured copy bandwidth from MEASURED_PEAKS.json.  The L2 bandwidth
    is a nominal 12 TB/s (hypothetical parameter, not measured)."""
    g = _gpu("B200-like", 148, 1.965e9, 256 * KiB, 126 * 1000 * 1000, 2,
             hbm_gbs * 1e9, 12e12)
    return g


def with_outlook(g, page_bytes=2 * MiB, link_bw=10e12):
    """A parameter set with the NEXT-4 outlook metrics on (hypothetical B200 values): 2 MiB GPU
    pages for the TLB metric; the die-to-die link between the two L2 halves at a nominal 10 TB/s."""
    return dict(g, page_bytes=page_bytes, link_bw=link_bw)


def gpu_hypothetical(l1_kib, l2_eff_mib, n_sm):
    """Hypothetical grid of BJ configs[3]: varied L1, effective L2, SM count."""
    return _gpu(f"hyp-L1{l1_kib}-L2{l2_eff_mib}-SM{n_sm}", n_sm, 1.5e9, l1_kib * KiB,
                l2_eff_mib * MiB, 1, 2000e9, 6000e9)


def hw_grid_configs3(hbm_gbs=6546.2):
    """BJ configs[3] architecture exploration: V100, A100 (Table tab:av100,
    P:307-320), the B200-like set and the hypothetical grid L1 {128, 192, 256} KiB x effective L2
    {6, 20, 40, 64} MiB x SM count {80, 108, 132, 148} (48 sets) = 51 hardware sets.  The integer
    stages read only the SM count, occupancy limits, cache geometry and L2 sections of a set: six
    groups (V100 with the 80-SM sets, A100, B200-like, the 108 / 132 / 148-SM sets)."""
    sets = [gpu_v100(), gpu_a100(), gpu_b200_like(hbm_gbs)]
    for nsm in (80, 108, 132, 148):
        for l1 in (128, 192, 256):
            for l2 in (6, 20, 40, 64):
                sets.append(gpu_hypothetical(l1, l2, nsm))
    return sets


# ---------------------------------------------------------------------------
# Kernels
# ---------------------------------------------------------------------------

def _dense_field(ext, elem=8, align=0):
    ex, ey, ez = ext
    return {"extent": (ex, ey, ez), "pitch": (1, ex, ex * ey), "align": align, "elem": elem}


def stencil_star(nx, ny, nz, radius, name=None, regs=64):
    """3D star stencil of range `radius`: 6r+1 loads from src, 1 store to dst.

    radius=4 is the paper's 3D-25pt range-4 star; radius=1 is the
    7pt stencil of BJ configs[0].  Fields are (n+2r) wide with ghost layers
    of width r; the domain is [r, n+r)."""
    r = radius
    ext = (nx + 2 * r, ny + 2 * r, nz + 2 * r)
    fields = [_dense_field(ext), _dense_field(ext)]
    acc = [(0, 0, (0, 0, 0))]
    for d in range(3):
        for k in range(1, r + 1):
            for s in (-k, k):
                o = [0, 0, 0]
                o[d] = s
                acc.append((0, 0, tuple(o)))
    acc.append((1, 1, (0, 0, 0)))
    return {
        "name": name or f"star{6 * r + 1}pt_r{r}_{nx}x{ny}x{nz}",
        "fields": fields, "accesses": acc,
        "dom_lo": (r, r, r), "dom_hi": (nx + r, ny + r, nz + r),
        "regs": regs, "flops": float(6 * r + 1),
    }


def k7(n=64):
    """BJ configs[0]: range-1 3D-7pt double stencil on n^3; thread-limited occupancy (regs=0)."""
    return stencil_star(n, n, n, 1, name=f"K7_{n}", regs=0)


def k25(n=512, ny=None, nz=None):
    """BJ configs[1]: range-4 3D-25pt double stencil; regs=64 per SURVEY Q10."""
    return stencil_star(n, ny or n, nz or n, 4, name=f"K25_{n}x{ny or n}x{nz or n}", regs=64)


def k25_paper():
    """The paper's grid 640x512x512."""
    return stencil_star(640, 512, 512, 4, name="K25p_640x512x512", regs=64)


D3Q15 = [(0, 0, 0)] + [tuple(v) for v in
                       ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1))] + \
        [(x, y, z) for x in (-1, 1) for y in (-1, 1) for z in (-1, 1)]
D3Q27 = [(x, y, z) for z in (-1, 0, 1) for y in (-1, 0, 1) for x in (-1, 0, 1)]
D3Q7 = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]


def _lbm(n, q_vel, phi_nbrs, n_extra_stores, name, regs=128):
    """Pull-scheme LBM access pattern.

    Fields (fzyx layout: one array per PDF, so PDF q's base alignment is
    (q * bytes_per_array) mod 128 within its allocation):
      src PDFs q: loaded at -c_q (pull, unaligned loads);
      dst PDFs q: stored at 0 (aligned stores);
      phase field phi: loaded at the FD neighbourhood `phi_nbrs`;
      `n_extra_stores` fields stored at 0 (FD result / velocity)."""
    ext = (n + 2, n + 2, n + 2)
    arr_bytes = ext[0] * ext[1] * ext[2] * 8
    fields, acc = [], []
    Q = len(q_vel)
    for q in range(Q):                          # src PDFs
        fields.append(_dense_field(ext, align=(q * arr_bytes) % 128))
    for q in range(Q):                          # dst PDFs
        fields.append(_dense_field(ext, align=(q * arr_bytes) % 128))
    fields.append(_dense_field(ext))            # phi
    for _ in range(n_extra_stores):
        fields.append(_dense_field(ext))
    for q, c in enumerate(q_vel):
        acc.append((q, 0, (-c[0], -c[1], -c[2])))
    for q in range(Q):
        acc.append((Q + q, 1, (0, 0, 0)))
    for o in phi_nbrs:
        acc.append((2 * Q, 0, tuple(o)))
    for e in range(n_extra_stores):
        acc.append((2 * Q + 1 + e, 1, (0, 0, 0)))
    return {"name": name, "fields": fields, "accesses": acc,
            "dom_lo": (1, 1, 1), "dom_hi": (n + 1, n + 1, n + 1),
            "regs": regs, "flops": 0.0}


def lbm15(n=256):
    """Paper's kernel: D3Q15 pull + 3D7pt phase field, 32 arrays, 22 loads / 16 stores (Q23)."""
    return _lbm(n, D3Q15, D3Q7, 1, f"LBM15_{n}")


def lbm27(n=256):
    """BJ configs[2] D3Q27 variant: 58 arrays, 54 loads / 30 stores (Q23)."""
    return _lbm(n, D3Q27, D3Q27, 3, f"LBM27_{n}")


# ---------------------------------------------------------------------------
# Configuration spaces
# ---------------------------------------------------------------------------
POW2_XY = [1 << i for i in range(11)]        # 1..1024
POW2_Z = [1 << i for i in range(7)]          # 1..64


def block_shapes(total):
    """All (X,Y,Z) with X,Y in {1..1024}, Z in {1..64} powers of two and X*Y*Z = total."""
    return [(x, y, z) for z in POW2_Z for y in POW2_XY for x in POW2_XY if x * y * z == total]


FOLDS_PAPER = [(1, 1, 1), (1, 2, 1), (1, 1, 2)]    # none, 2y, 2z


def space_stencil_paper():
    """168 = 56 shapes x {none, 2y, 2z}."""
    return [(b, f, 0) for b in block_shapes(1024) for f in FOLDS_PAPER]


def space_lbm(folds=False):
    """49 shapes of 512 threads; optionally x {none, 2y, 2z} = 147."""
    fl = FOLDS_PAPER if folds else [(1, 1, 1)]
    return [(b, f, 0) for b in block_shapes(512) for f in fl]


def space_k7():
    """BJ configs[0] / SURVEY Q24: bx=32, by,bz in {1,2,4,8}; (32,8,8) exceeds 1024 threads."""
    return [((32, y, z), (1, 1, 1), 0) for z in (1, 2, 4, 8) for y in (1, 2, 4, 8)]


def space_extended():
    """SURVEY Q34 extended throughput space: power-of-two shapes with 64..1024 threads x (fy,fz) in {1,2,4}^2."""
    shapes = [(x, y, z) for z in POW2_Z for y in POW2_XY for x in POW2_XY
              if 64 <= x * y * z <= 1024]
    folds = [(1, fy, fz) for fz in (1, 2, 4) for fy in (1, 2, 4)]
    return [(b, f, 0) for b in shapes for f in folds]


# ---------------------------------------------------------------------------
# Seeded random tiny kernels for property / parity tests
# ---------------------------------------------------------------------------

def random_kernel(seed, max_fields=3, max_acc=8, max_dom=20):
    rng = random.Random(seed)
    nf = rng.randint(1, max_fields)
    dom = [rng.randint(1, max_dom) for _ in range(3)]
    halo = 4
    ext = tuple(d + 2 * halo + rng.randint(0, 3) for d in dom)
    fields = []
    for _ in range(nf):
        elem = rng.choice([4, 8, 8, 8, 16])
        align = elem * rng.randint(0, 128 // elem - 1)
        pad_y = rng.randint(0, 2)
        px = 1
        py = ext[0] + pad_y
        pz = py * ext[1] + rng.randint(0, 3)
        fields.append({"extent": ext, "pitch": (px, py, pz), "align": align, "elem": elem})
    acc = []
    na = rng.randint(1, max_acc)
    for _ in range(na):
        f = rng.randrange(nf)
        st = 1 if rng.random() < 0.3 else 0
        o = tuple(rng.randint(-halo, halo) for _ in range(3))
        acc.append((f, st, o))
    if all(a[1] == 1 for a in acc):
        acc[0] = (acc[0][0], 0, acc[0][2])
    return {"name": f"rand{seed}", "fields": fields, "accesses": acc,
            "dom_lo": (halo, halo, halo), "dom_hi": tuple(halo + d for d in dom),
            "regs": rng.choice([0, 32, 64]), "flops": 1.0}


def random_gpu(seed):
    rng = random.Random(seed + 7919)
    g = _gpu(f"randgpu{seed}", rng.choice([2, 3, 4, 5, 8]), 1.0e9 + rng.random() * 1e9,
             rng.choice([16, 32, 64]) * KiB, rng.choice([1, 2, 4]) * MiB, rng.choice([1, 2]),
             500e9 + rng.random() * 1e12, 2000e9 + rng.random() * 2e12,
             max_thr_sm=rng.choice([512, 1024, 2048]), max_blk_sm=rng.choice([2, 4, 8, 32]))
    g["pair_window_bytes"] = rng.choice([256, 512, 1024])
    # outlook metrics (NEXT-4): TLB page size, L2 section count and link bandwidth
    g["page_bytes"] = rng.choice([0, 512, 4096, 65536])
    g["l2_sections"] = rng.choice([g["l2_sections"], g["l2_sections"], 3, 4])
    g["link_bw"] = rng.choice([0.0, 0.0, 1e11 + rng.random() * 1e12])
    return g


def random_config(seed):
    rng = random.Random(seed + 104729)
    while True:
        b = (rng.choice([1, 2, 3, 4, 8, 16, 32, 64]), rng.choice([1, 2, 3, 4, 8]), rng.choice([1, 2, 4]))
        if 1 <= b[0] * b[1] * b[2] <= 256:
            break
    f = (rng.choice([1, 1, 2]), rng.choice([1, 1, 2, 3]), rng.choice([1, 1, 2]))
    k = rng.choice([0, 0, 0, 1, 2])
    variant = rng.choice([0, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 15])   # WS_VAR_* bits (NEXT-3 / NEXT-4)
    return (b, f, k, variant)
