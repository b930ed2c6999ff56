"""Independent brute-force re-implementation used to PIN the oracle.

Written separately from oracle/ws_oracle.cpp and structured differently, so a
plausible slip in either (wrong pitch index, transposed operand, wrong block
ordering, dropped term) shows up as a mismatch:

* footprints are computed the paper's way ("numpy meshgrid ... unique"),
  over *cells* rather than (thread, instruction) pairs: the footprint of a set
  of threads is {addr(c + o) : c an active cell of those threads, o an offset
  of the field/kind} -- every active cell c = base+kappa issues instruction
  r = kappa + o, so the two definitions name the same set;
* a sectored, fully-associative LRU cache replays the trace
  (SPEC.md cachesim-oracle) for the capacity pins.

Only small grids (the whole thing is numpy over every cell of a block range).
"""
from __future__ import annotations

import itertools
from collections import OrderedDict

import numpy as np


def geometry(kernel, gpu, cfg):
    (bx, by, bz), (fx, fy, fz), kov = cfg[:3]
    variant = cfg[3] if len(cfg) > 3 else 0
    lo = np.array(kernel["dom_lo"], dtype=np.int64)
    hi = np.array(kernel["dom_hi"], dtype=np.int64)
    b = np.array([bx, by, bz], dtype=np.int64)
    f = np.array([fx, fy, fz], dtype=np.int64)
    T = int(bx * by * bz)
    G = -(-(hi - lo) // (b * f))
    N = int(np.prod(G))
    if kov:
        k = kov
    else:
        Ta = -(-T // 32) * 32
        k = min(gpu["max_thr_sm"] // Ta, gpu["max_blk_sm"])
        if kernel["regs"]:
            k = min(k, gpu["regs_sm"] // (kernel["regs"] * Ta))
    W = min(N, gpu["n_sm"] * k)
    cx, cy, cz = G[0] // 2, G[1] // 2, G[2] // 2
    centre = int(cx + G[0] * (cy + G[1] * cz))
    s = min(max(centre - W // 2, 0), N - W)
    Ly, Lz = (max(0, s - int(G[0])), s), (max(0, s - int(G[0] * G[1])), s)
    if variant & 2:   # previous wave only (SBAC)
        Ly = Lz = (max(0, s - W), s)
    return dict(lo=lo, hi=hi, b=b, f=f, T=T, G=G, N=N, k=k, W=W, s=s, Ly=Ly, Lz=Lz, variant=variant)


def block_cells(geo, blocks):
    """Active cells (n,3) of the given block ids (numpy meshgrid over the box)."""
    out = []
    G, b, f, lo, hi = geo["G"], geo["b"], geo["f"], geo["lo"], geo["hi"]
    for B in blocks:
        bc = np.array([B % G[0], (B // G[0]) % G[1], B // (G[0] * G[1])], dtype=np.int64)
        start = lo + bc * b * f
        stop = np.minimum(start + b * f, hi)
        xs, ys, zs = [np.arange(start[d], stop[d]) for d in range(3)]
        Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
        out.append(np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1))
    if not out:
        return np.zeros((0, 3), dtype=np.int64)
    return np.concatenate(out)


def addresses(field, cells):
    p = np.array(field["pitch"], dtype=np.int64)
    return field["align"] + field["elem"] * (cells @ p)


def footprint(kernel, cells, kinds, shift):
    """Set of (field, addr >> shift) over cells + offsets of the given kinds."""
    keys = set()
    for fi, fld in enumerate(kernel["fields"]):
        offs = [o for (f, st, o) in kernel["accesses"] if f == fi and st in kinds]
        if not offs or len(cells) == 0:
            continue
        allc = np.concatenate([cells + np.array(o, dtype=np.int64) for o in offs])
        a = np.unique(addresses(fld, allc) >> shift)
        keys.update((fi, int(v)) for v in a)
    return keys


def footprint_md(kernel, cells, kinds, shift):
    """Multidimensional address space: (field, z, y, (x * elem) >> shift)."""
    keys = set()
    for fi, fld in enumerate(kernel["fields"]):
        offs = [o for (f, st, o) in kernel["accesses"] if f == fi and st in kinds]
        if not offs or len(cells) == 0:
            continue
        allc = np.concatenate([cells + np.array(o, dtype=np.int64) for o in offs])
        xs = (allc[:, 0] * fld["elem"]) >> shift
        keys.update((fi, int(z), int(y), int(x)) for x, y, z in zip(xs, allc[:, 1], allc[:, 2]))
    return keys


def set_counts(kernel, gpu, cfg):
    """Union scopes a4-a6 by cell enumeration (the oracle does (thread, instr))."""
    geo = geometry(kernel, gpu, cfg)
    ls = int(np.log2(gpu["sector_bytes"]))
    ll = int(np.log2(gpu["line_bytes"]))
    s, W, nsm = geo["s"], geo["W"], gpu["n_sm"]
    wave = list(range(s, s + W))
    wcells = block_cells(geo, wave)
    rep_mode = bool(geo["variant"] & 8)   # representative block
    B_rep = s + W // 2
    md = bool(geo["variant"] & 1)
    fp = footprint_md if md else footprint
    WLD = fp(kernel, wcells, (0,), ls)
    WST = fp(kernel, wcells, (1,), ls)
    WLIN = fp(kernel, wcells, (0, 1), ll)
    sm_sec = sm_lin = 0
    if rep_mode:
        cells = block_cells(geo, [B_rep])
        sm_sec = W * len(footprint(kernel, cells, (0,), ls))
        sm_lin = W * len(footprint(kernel, cells, (0,), ll))
    else:
        for j in range(min(nsm, W)):
            cells = block_cells(geo, wave[j::nsm])
            sm_sec += len(footprint(kernel, cells, (0,), ls))
            sm_lin += len(footprint(kernel, cells, (0,), ll))
    FY = fp(kernel, block_cells(geo, range(*geo["Ly"])), (0, 1), ls)
    FZ = fp(kernel, block_cells(geo, range(*geo["Lz"])), (0, 1), ls)
    d = ll - ls
    # NEXT-4 (linear address space): TLB pages of the wave; per-L2-section footprints with SM j
    # in section j*S//n_sm and block s+i on SM i % n_sm
    pb = int(gpu.get("page_bytes", 0))
    pages = len(footprint(kernel, wcells, (0, 1), int(np.log2(pb)))) if pb else 0
    S = gpu["l2_sections"]
    sec_ld, sec_lin = [set() for _ in range(S)], [set() for _ in range(S)]
    for i, B in enumerate(wave):
        sec = (i % nsm) * S // nsm
        cells = block_cells(geo, [B])
        sec_ld[sec] |= footprint(kernel, cells, (0,), ls)
        sec_lin[sec] |= footprint(kernel, cells, (0, 1), ll)
    dup = sum(len(x) for x in sec_lin) - len(set().union(*sec_lin))
    link = sum(len(x) for x in sec_ld) - len(set().union(*sec_ld))
    if not (S > 1 and (gpu.get("link_bw", 0.0) > 0 or geo["variant"] & 4)):   # reported on request (ws.h)
        dup = link = 0
    lup = W * len(block_cells(geo, [B_rep])) if rep_mode else len(wcells)
    return dict(lup_wave=lup, sm_ld_sectors=sm_sec, sm_ld_lines=sm_lin,
                wave_ld_sectors=len(WLD), wave_st_sectors=len(WST), wave_lines=len(WLIN),
                ly_lines=len({v[:-1] + (v[-1] >> d,) for v in FY}), lz_lines=len({v[:-1] + (v[-1] >> d,) for v in FZ}),
                ov_y=len(WLD & FY), ov_z=len(WLD & FZ), k=geo["k"], wave_blocks=W,
                wave_first_block=s, grid=tuple(int(g) for g in geo["G"]),
                wave_pages=pages, l2_dup_lines=dup, l2_link_sectors=link)


# ------------------------------------------------------------- per-thread traces
def thread_trace(kernel, geo, B, t):
    """(field, kind, cell - base, addr) issued by one thread, in instruction order (deduplicated
    per thread, i.e. register reuse under folding)."""
    G, b, f, lo, hi = geo["G"], geo["b"], geo["f"], geo["lo"], geo["hi"]
    bc = np.array([B % G[0], (B // G[0]) % G[1], B // (G[0] * G[1])])
    tc = np.array([t % b[0], (t // b[0]) % b[1], t // (b[0] * b[1])])
    base = lo + (bc * b + tc) * f
    out = []
    for fi, fld in enumerate(kernel["fields"]):
        for st in (0, 1):
            offs = [o for (ff, s_, o) in kernel["accesses"] if ff == fi and s_ == st]
            seen = set()
            for kap in itertools.product(range(f[0]), range(f[1]), range(f[2])):
                c = base + np.array(kap)
                if np.any(c >= hi):
                    continue
                for o in offs:
                    cell = tuple(int(v) for v in c + np.array(o))
                    if cell in seen:
                        continue
                    seen.add(cell)
                    rel = tuple(int(v) for v in np.array(cell) - base)
                    out.append((fi, st, rel, int(addresses(fld, np.array([cell]))[0])))
    return out


def l1_counts(kernel, gpu, cfg):
    """a3 via per-warp dictionaries keyed by instruction identity (field, kind, cell - thread base)."""
    geo = geometry(kernel, gpu, cfg)
    T = geo["T"]
    SB, BB, NB, HW, PW = (gpu["sector_bytes"], gpu["bank_bytes"], gpu["n_banks"],
                          gpu["half_warp"], gpu["pair_window_bytes"])
    req = [0, 0]
    wf = 0
    rep_mode = bool(geo["variant"] & 8)
    blocks = [geo["s"] + geo["W"] // 2] if rep_mode else range(geo["s"], geo["s"] + geo["W"])
    for B in blocks:
        for w in range(-(-T // 32)):
            lanes = [t for t in range(32 * w, min(32 * w + 32, T))]
            # instruction key: (field, kind, relative cell) -> lane -> addr
            per_instr = {}
            for t in lanes:
                for (fi, st, rel, a) in thread_trace(kernel, geo, B, t):
                    per_instr.setdefault((fi, st, rel), {})[t] = a
            for (fi, st, rel), lane_addr in per_instr.items():
                req[st] += len({a // SB for a in lane_addr.values()})
                for h in range(32 // HW):
                    words = sorted({a // BB for t, a in lane_addr.items() if h * HW <= t - 32 * w < (h + 1) * HW})
                    clusters, cur = [], []
                    for u in words:
                        if cur and (u - cur[0]) * BB >= PW:
                            clusters.append(cur)
                            cur = []
                        cur.append(u)
                    if cur:
                        clusters.append(cur)
                    for c in clusters:
                        cnt = [0] * NB
                        for u in c:
                            cnt[u % NB] += 1
                        wf += max(cnt)
    m = geo["W"] if rep_mode else 1
    return dict(l1_wavefronts=m * wf, l1_req_ld_sectors=m * req[0], l1_req_st_sectors=m * req[1])


class SectoredLRU:
    """Fully-associative LRU over lines, 32 B valid bits per sector."""

    def __init__(self, capacity_bytes, line_bytes=128, sector_bytes=32):
        self.cap = max(1, capacity_bytes // line_bytes)
        self.lb, self.sb = line_bytes, sector_bytes
        self.lines = OrderedDict()
        self.misses = 0
        self.requests = 0

    def access(self, key_sector):
        field, sec = key_sector
        line = (field, sec // (self.lb // self.sb))
        self.requests += 1
        if line in self.lines:
            self.lines.move_to_end(line)
            if sec in self.lines[line]:
                return
            self.lines[line].add(sec)
            self.misses += 1
            return
        self.misses += 1
        self.lines[line] = {sec}
        if len(self.lines) > self.cap:
            self.lines.popitem(last=False)


def replay_blocks(kernel, gpu, cfg, blocks, cache, kinds=(0,), count_from=None):
    """Replay every thread of `blocks` in schedule order through `cache`.
    Returns misses incurred by blocks >= count_from (all if None)."""
    geo = geometry(kernel, gpu, cfg)
    SB = gpu["sector_bytes"]
    base_miss = None
    for B in blocks:
        if count_from is not None and B == count_from:
            base_miss = cache.misses
        for t in range(geo["T"]):
            for (fi, st, _rel, a) in thread_trace(kernel, geo, B, t):
                if st in kinds:
                    cache.access((fi, a // SB))
    return cache.misses - (base_miss or 0)


# ------------------------------------------------------------- NEXT-1 request streams
def warp_requests(kernel, geo, B, kinds):
    """Coalesced requests of block B: warps in order; per warp the instructions ordered by
    (field, kind, elem * (pitch . r)); per instruction the distinct sectors of its issuing
    lanes, ascending.  Built from the per-thread traces (thread_trace), grouped by instruction
    identity (field, kind, cell - thread base)."""
    T = geo["T"]
    out = []
    for w in range(-(-T // 32)):
        per = {}
        for t in range(32 * w, min(32 * w + 32, T)):
            for (fi, st, rel, a) in thread_trace(kernel, geo, B, t):
                if st in kinds:
                    per.setdefault((fi, st, rel), set()).add(a // 32)
        def key(item):
            (fi, st, rel), _ = item
            f = kernel["fields"][fi]
            return (fi, st, f["elem"] * sum(p * r for p, r in zip(f["pitch"], rel)))
        for (fi, st, rel), secs in sorted(per.items(), key=key):
            out += [((fi, s), st) for s in sorted(secs)]
    return out
