"""ctypes wrapper of the plain C++ CPU oracle (oracle/ws_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / `--impl reference` leg.  The product package
`paper_2204_14242_b200` never imports this module, and this module never
imports the product package (it only reads plain descriptions produced by
`workloads`).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
# WSO_LIB: load another build of the oracle (scripts/oracle_mutations.py builds deliberately
# broken copies to show that the pins in tests/test_oracle_pins.py catch each slip)
LIB = os.environ.get("WSO_LIB") or os.path.join(HERE, "libwsoracle.so")
SRC = os.path.join(HERE, "ws_oracle.cpp")

I64 = C.c_int64


class Field(C.Structure):
    _fields_ = [("extent", I64 * 3), ("pitch", I64 * 3), ("align_bytes", I64), ("elem_bytes", I64)]


class Access(C.Structure):
    _fields_ = [("field", I64), ("is_store", I64), ("off", I64 * 3)]


class Kernel(C.Structure):
    _fields_ = [("n_fields", I64), ("n_accesses", I64), ("fields", C.POINTER(Field)),
                ("accesses", C.POINTER(Access)), ("dom_lo", I64 * 3), ("dom_hi", I64 * 3),
                ("regs_per_thread", I64), ("flops_per_lup", C.c_double)]


class Gpu(C.Structure):
    _fields_ = [("n_sm", I64), ("max_thr_sm", I64), ("max_blk_sm", I64), ("max_thr_blk", I64),
                ("regs_sm", I64), ("sector_bytes", I64), ("line_bytes", I64), ("n_banks", I64),
                ("bank_bytes", I64), ("half_warp", I64), ("pair_window_bytes", I64),
                ("l2_sections", I64), ("l1_bytes", I64), ("l2_bytes", I64),
                ("clock_hz", C.c_double), ("dram_bw", C.c_double), ("l2_bw", C.c_double),
                ("hit_abc", (C.c_double * 3) * 4), ("page_bytes", I64), ("link_bw", C.c_double)]


class Config(C.Structure):
    _fields_ = [("block", I64 * 3), ("fold", I64 * 3), ("blocks_per_sm", I64), ("variant", I64)]


INT_FIELDS = ["status", "limiter", "grid", "k", "wave_blocks", "n_smsets", "wave_first_block",
              "lup_wave", "n_instr", "l1_wavefronts", "l1_req_ld_sectors", "l1_req_st_sectors",
              "sm_ld_sectors", "sm_ld_lines", "wave_ld_sectors", "wave_st_sectors", "wave_lines",
              "ly_lines", "lz_lines", "ov_y", "ov_z"]
FP_FIELDS = ["O_l1", "R_l1", "O_y", "R_y", "O_z", "R_z", "O_st", "R_st",
             "l1_cyc_per_lup", "l2_ld_Bpl", "l2_st_Bpl", "dram_ld_Bpl", "dram_st_Bpl",
             "t_l1", "t_l2", "t_dram", "t_pred"]
INT_FIELDS2 = ["wave_pages", "l2_dup_lines", "l2_link_sectors"]   # NEXT-4
FP_FIELDS2 = ["l2_eff_bytes", "t_link"]


class Result(C.Structure):
    _fields_ = ([("status", I64), ("limiter", I64), ("grid", I64 * 3)] +
                [(n, I64) for n in INT_FIELDS[3:]] +
                [(n, C.c_double) for n in FP_FIELDS] + [("addr_evals", I64)] +
                [(n, I64) for n in INT_FIELDS2] + [(n, C.c_double) for n in FP_FIELDS2])


def build(force=False, src=SRC, out=None):
    out = out or LIB
    if out != LIB or force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        tmp = f"{out}.{os.getpid()}.tmp"        # build aside, then rename: a loaded copy stays valid
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I" + HERE, "-o", tmp, src, "-lpthread"])
        os.replace(tmp, out)
    return out


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        L.wso_estimate.argtypes = [C.POINTER(Kernel), C.POINTER(Gpu), C.POINTER(Config), C.POINTER(Result)]
        L.wso_estimate.restype = I64
        L.wso_estimate_batch.argtypes = [C.POINTER(Kernel), C.POINTER(Gpu), C.POINTER(Config), I64,
                                         C.POINTER(Result), I64]
        L.wso_estimate_batch.restype = None
        L.wso_plan.argtypes = [C.POINTER(Kernel), C.POINTER(Gpu), C.POINTER(Config), C.POINTER(Result)]
        L.wso_plan.restype = I64
        L.wso_check_kernel.argtypes = [C.POINTER(Kernel)]
        L.wso_check_kernel.restype = I64
        L.wso_address.argtypes = [C.POINTER(Field), C.POINTER(I64)]
        L.wso_address.restype = I64
        L.wso_unique_sectors.argtypes = [C.POINTER(I64), I64, I64]
        L.wso_unique_sectors.restype = I64
        L.wso_halfwarp_wavefronts.argtypes = [C.POINTER(I64), I64, C.POINTER(Gpu)]
        L.wso_halfwarp_wavefronts.restype = I64
        L.wso_hit_rate.argtypes = [C.POINTER(C.c_double), C.c_double]
        L.wso_hit_rate.restype = C.c_double
        _lib = L
    return _lib


# ----------------------------------------------------------------- marshalling
def make_field(f):
    F = Field()
    F.extent[:] = list(f["extent"])
    F.pitch[:] = list(f["pitch"])
    F.align_bytes = f["align"]
    F.elem_bytes = f["elem"]
    return F


def make_kernel(k):
    fields = (Field * len(k["fields"]))(*[make_field(f) for f in k["fields"]])
    accs = (Access * len(k["accesses"]))()
    for i, (fi, st, o) in enumerate(k["accesses"]):
        accs[i].field, accs[i].is_store = fi, st
        accs[i].off[:] = list(o)
    K = Kernel()
    K.n_fields, K.n_accesses = len(k["fields"]), len(k["accesses"])
    K.fields, K.accesses = fields, accs
    K.dom_lo[:] = list(k["dom_lo"])
    K.dom_hi[:] = list(k["dom_hi"])
    K.regs_per_thread = k["regs"]
    K.flops_per_lup = k["flops"]
    K._keep = (fields, accs)
    return K


def make_gpu(g):
    G = Gpu()
    for n in ["n_sm", "max_thr_sm", "max_blk_sm", "max_thr_blk", "regs_sm", "sector_bytes",
              "line_bytes", "n_banks", "bank_bytes", "half_warp", "pair_window_bytes",
              "l2_sections", "l1_bytes", "l2_bytes"]:
        setattr(G, n, int(g[n]))
    G.clock_hz, G.dram_bw, G.l2_bw = g["clock_hz"], g["dram_bw"], g["l2_bw"]
    for i in range(4):
        for j in range(3):
            G.hit_abc[i][j] = g["hit_abc"][i][j]
    G.page_bytes = int(g.get("page_bytes", 0))
    G.link_bw = float(g.get("link_bw", 0.0))
    return G


def make_config(c):
    # (block, fold, blocks_per_sm[, variant])
    b, f, k = c[:3]
    X = Config()
    X.block[:] = list(b)
    X.fold[:] = list(f)
    X.blocks_per_sm = k
    X.variant = c[3] if len(c) > 3 else 0
    return X


def result_dict(R):
    d = {}
    for n in INT_FIELDS:
        v = getattr(R, n)
        d[n] = tuple(v) if n == "grid" else int(v)
    for n in FP_FIELDS:
        d[n] = float(getattr(R, n))
    d["addr_evals"] = int(R.addr_evals)
    for n in INT_FIELDS2:
        d[n] = int(getattr(R, n))
    for n in FP_FIELDS2:
        d[n] = float(getattr(R, n))
    return d


def estimate(kernel, gpu, config):
    """One configuration -> dict of every result field."""
    K, G, X, R = make_kernel(kernel), make_gpu(gpu), make_config(config), Result()
    lib().wso_estimate(C.byref(K), C.byref(G), C.byref(X), C.byref(R))
    return result_dict(R)


def estimate_batch(kernel, gpu, configs, n_threads=1):
    K, G = make_kernel(kernel), make_gpu(gpu)
    X = (Config * len(configs))(*[make_config(c) for c in configs])
    R = (Result * len(configs))()
    lib().wso_estimate_batch(C.byref(K), C.byref(G), X, len(configs), R, n_threads)
    return [result_dict(R[i]) for i in range(len(configs))]


def plan(kernel, gpu, config):
    """Geometry + addr_evals only (no enumeration)."""
    K, G, X, R = make_kernel(kernel), make_gpu(gpu), make_config(config), Result()
    lib().wso_plan(C.byref(K), C.byref(G), C.byref(X), C.byref(R))
    return result_dict(R)


def check_kernel(kernel):
    K = make_kernel(kernel)
    return int(lib().wso_check_kernel(C.byref(K)))


def address(field, cell):
    F = make_field(field)
    c = (I64 * 3)(*cell)
    return int(lib().wso_address(C.byref(F), c))


def unique_sectors(addrs, sector_bytes=32):
    a = (I64 * len(addrs))(*addrs)
    return int(lib().wso_unique_sectors(a, len(addrs), sector_bytes))


def halfwarp_wavefronts(addrs, gpu):
    a = (I64 * max(1, len(addrs)))(*addrs)
    G = make_gpu(gpu)
    return int(lib().wso_halfwarp_wavefronts(a, len(addrs), C.byref(G)))


def hit_rate(abc, O):
    a = (C.c_double * 3)(*abc)
    return float(lib().wso_hit_rate(a, O))


# ----------------------------------------------------------------- NEXT-1: simulated hit rates
SIM_INT = ["status", "capacity_bytes", "l1_requests", "l1_compulsory", "l1_misses", "st_requests",
           "st_compulsory", "st_misses", "ov_y", "y_resident", "ov_z_only", "z_resident"]
SIM_FP = ["O_l1", "R_l1", "O_y", "R_y", "O_z", "R_z", "O_st", "R_st"]


class SimResult(C.Structure):
    _fields_ = [(n, I64) for n in SIM_INT] + [(n, C.c_double) for n in SIM_FP]


def _sim_lib():
    L = lib()
    if not getattr(L, "_sim_ready", False):
        L.wso_simulate_batch.argtypes = [C.POINTER(Kernel), C.POINTER(Gpu), C.POINTER(Config), I64,
                                         C.POINTER(I64), I64, C.POINTER(SimResult), I64]
        L.wso_simulate_batch.restype = None
        L.wso_fit_gompertz.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), I64, C.POINTER(C.c_double)]
        L.wso_fit_gompertz.restype = C.c_double
        L._sim_ready = True
    return L


def simulate_batch(kernel, gpu, configs, capacities, n_threads=1):
    """-> [[dict per capacity] per config]"""
    K, G = make_kernel(kernel), make_gpu(gpu)
    X = (Config * len(configs))(*[make_config(c) for c in configs])
    caps = (I64 * len(capacities))(*capacities)
    R = (SimResult * (len(configs) * len(capacities)))()
    _sim_lib().wso_simulate_batch(C.byref(K), C.byref(G), X, len(configs), caps, len(capacities), R, n_threads)
    out = []
    for i in range(len(configs)):
        row = []
        for k in range(len(capacities)):
            r = R[i * len(capacities) + k]
            d = {n: int(getattr(r, n)) for n in SIM_INT}
            d.update({n: float(getattr(r, n)) for n in SIM_FP})
            row.append(d)
        out.append(row)
    return out


def fit_gompertz(O, R):
    """-> ((a, b, c), residual sum of squares)"""
    n = len(O)
    o = (C.c_double * n)(*O)
    r = (C.c_double * n)(*R)
    th = (C.c_double * 3)()
    rss = _sim_lib().wso_fit_gompertz(o, r, n, th)
    return (th[0], th[1], th[2]), float(rss)
