"""Thin ctypes binding of libwsb200.so (include/ws.h).  Argument marshalling only:
every step of the estimator runs in the library's sm_100a kernels.  There is no
CPU fallback: if the shared library or a CUDA device is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# WS_LIB selects another in-tree build of the same ABI (the bounds-check build libwsb200_check.so)
LIB_PATH = os.environ.get("WS_LIB") or os.path.join(_PKG, "libwsb200.so")

U32, I32, I64, U64, F64 = C.c_uint32, C.c_int32, C.c_int64, C.c_uint64, C.c_double

WS_OK, WS_EINVAL, WS_ELIMIT, WS_EBOUNDS, WS_ENOMEM, WS_ECUDA, WS_EUNKNOWN_ID = range(7)
STATUS_NAMES = ["WS_OK", "WS_EINVAL", "WS_ELIMIT", "WS_EBOUNDS", "WS_ENOMEM", "WS_ECUDA", "WS_EUNKNOWN_ID"]


class ws_field(C.Structure):
    _fields_ = [("extent", I64 * 3), ("pitch", I64 * 3), ("align_bytes", I64), ("elem_bytes", U32), ("pad", U32)]


class ws_access(C.Structure):
    _fields_ = [("field", U32), ("is_store", U32), ("off", I32 * 3)]


class ws_kernel(C.Structure):
    _fields_ = [("n_fields", U32), ("n_accesses", U32), ("fields", C.POINTER(ws_field)),
                ("accesses", C.POINTER(ws_access)), ("dom_lo", I64 * 3), ("dom_hi", I64 * 3),
                ("regs_per_thread", U32), ("pad", U32), ("flops_per_lup", F64)]


class ws_gpu(C.Structure):
    _fields_ = [("n_sm", U32), ("max_thr_sm", U32), ("max_blk_sm", U32), ("max_thr_blk", U32), ("regs_sm", U32),
                ("sector_bytes", U32), ("line_bytes", U32), ("n_banks", U32), ("bank_bytes", U32),
                ("half_warp", U32), ("pair_window_bytes", U32), ("l2_sections", U32),
                ("l1_bytes", U64), ("l2_bytes", U64), ("clock_hz", F64), ("dram_bw", F64), ("l2_bw", F64),
                ("hit_abc", (F64 * 3) * 4), ("page_bytes", U64), ("link_bw", F64)]


class ws_config(C.Structure):
    _fields_ = [("kernel_id", U32), ("gpu_id", U32), ("block", U32 * 3), ("fold", U32 * 3),
                ("blocks_per_sm", U32), ("variant", U32)]


RESULT_U64 = ["wave_first_block", "lup_wave", "l1_wavefronts", "l1_req_ld_sectors", "l1_req_st_sectors",
              "sm_ld_sectors", "sm_ld_lines", "wave_ld_sectors", "wave_st_sectors", "wave_lines", "ly_lines",
              "lz_lines", "ov_y", "ov_z", "addr_evals"]
RESULT_F64 = ["O_l1", "R_l1", "O_y", "R_y", "O_z", "R_z", "O_st", "R_st", "l1_cyc_per_lup", "l2_ld_Bpl",
              "l2_st_Bpl", "dram_ld_Bpl", "dram_st_Bpl", "t_l1", "t_l2", "t_dram", "t_pred"]
RESULT_U64_2 = ["wave_pages", "l2_dup_lines", "l2_link_sectors"]   # NEXT-4 outlook metrics
RESULT_F64_2 = ["l2_eff_bytes", "t_link"]
WS_VAR_MDIM, WS_VAR_PREV_WAVE, WS_VAR_L2_DUP, WS_VAR_REP_BLOCK = 1, 2, 4, 8


class ws_result(C.Structure):
    _fields_ = ([("status", I32), ("limiter", U32), ("grid", U32 * 3), ("k", U32), ("wave_blocks", U32),
                 ("n_smsets", U32), ("n_instr", U32), ("rank", U32)] +
                [(n, U64) for n in RESULT_U64] + [(n, F64) for n in RESULT_F64] +
                [(n, U64) for n in RESULT_U64_2] + [(n, F64) for n in RESULT_F64_2])


SIM_U64 = ["capacity_bytes", "l1_requests", "l1_compulsory", "l1_misses", "st_requests", "st_compulsory",
           "st_misses", "ov_y", "y_resident", "ov_z_only", "z_resident"]
SIM_F64 = ["O_l1", "R_l1", "O_y", "R_y", "O_z", "R_z", "O_st", "R_st"]


class ws_sim_result(C.Structure):
    _fields_ = [("status", I32), ("pad", U32)] + [(n, U64) for n in SIM_U64] + [(n, F64) for n in SIM_F64]


assert C.sizeof(ws_config) == 40 and C.sizeof(ws_result) == 336 and C.sizeof(ws_sim_result) == 160

CONFIG_DTYPE = np.dtype(ws_config)
RESULT_DTYPE = np.dtype(ws_result)

EXPORTS = ["ws_create", "ws_destroy", "ws_last_error", "ws_set_stream", "ws_describe_kernel", "ws_describe_gpu",
           "ws_estimate", "ws_estimate_async", "ws_rank", "ws_rank_async", "ws_last_launch_count",
           "ws_profile_enable", "ws_profile_read", "ws_kernel_name", "ws_work_read", "ws_simulate",
           "ws_sim_release", "ws_fit_gompertz", "ws_validate_stencil25", "ws_validate_lbm15",
           "ws_estimate_multi", "ws_estimate_multi_async", "ws_last_group_count", "ws_estimate_ranked_async", "ws_check_read"]

_lib = None


def load_library(path: str = LIB_PATH):
    """Load (never build) the native library; raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libwsb200.so not found at {path}: run `python -m paper_2204_14242_b200.build` "
                           "(there is no CPU fallback)")
    L = C.CDLL(path)
    P = C.c_void_p
    L.ws_create.argtypes = [C.c_int, P, C.POINTER(P)]
    L.ws_destroy.argtypes = [P]
    L.ws_destroy.restype = None
    L.ws_last_error.argtypes = [P]
    L.ws_last_error.restype = C.c_char_p
    L.ws_set_stream.argtypes = [P, P]
    L.ws_describe_kernel.argtypes = [P, C.POINTER(ws_kernel), C.POINTER(U32)]
    L.ws_describe_gpu.argtypes = [P, C.POINTER(ws_gpu), C.POINTER(U32)]
    L.ws_estimate.argtypes = [P, P, C.c_size_t, P]
    L.ws_estimate_async.argtypes = [P, P, C.c_size_t, P]
    L.ws_estimate_ranked_async.argtypes = [P, P, C.c_size_t, P, C.c_size_t, P]
    L.ws_check_read.argtypes = [P, P]
    L.ws_estimate_multi.argtypes = [P, P, C.c_size_t, P, U32, P]
    L.ws_estimate_multi_async.argtypes = [P, P, C.c_size_t, P, U32, P]
    L.ws_last_group_count.argtypes = [P]
    L.ws_last_group_count.restype = U32
    L.ws_rank.argtypes = [P, P, C.c_size_t, C.c_size_t, P]
    L.ws_rank_async.argtypes = [P, P, C.c_size_t, C.c_size_t, P]
    L.ws_last_launch_count.argtypes = [P]
    L.ws_last_launch_count.restype = U32
    L.ws_profile_enable.argtypes = [P, C.c_int]
    L.ws_profile_read.argtypes = [P, C.POINTER(F64), C.POINTER(U64), U32, C.POINTER(U32)]
    L.ws_work_read.argtypes = [P, C.POINTER(U64), U32]
    L.ws_simulate.argtypes = [P, P, C.c_size_t, P, U32, P]
    L.ws_sim_release.argtypes = [P]
    L.ws_fit_gompertz.argtypes = [P, P, P, C.c_size_t, P, P]
    L.ws_validate_stencil25.argtypes = [P, P, P, P, P, P, U32, P]
    L.ws_validate_lbm15.argtypes = [P, P, P, P, P, P, P, U32, P]
    L.ws_kernel_name.argtypes = [U32]
    L.ws_kernel_name.restype = C.c_char_p
    for n in EXPORTS:
        if n not in ("ws_destroy", "ws_last_error", "ws_last_launch_count", "ws_kernel_name", "ws_last_group_count"):
            getattr(L, n).restype = C.c_int
    _lib = L
    return L


class WSError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")
        self.status = status


# ------------------------------------------------------------------ marshalling helpers
def kernel_struct(k):
    nf, na = len(k["fields"]), len(k["accesses"])
    fields = (ws_field * nf)()
    for i, f in enumerate(k["fields"]):
        fields[i].extent[:] = list(f["extent"])
        fields[i].pitch[:] = list(f["pitch"])
        fields[i].align_bytes = f["align"]
        fields[i].elem_bytes = f["elem"]
    accs = (ws_access * na)()
    for i, (fi, st, o) in enumerate(k["accesses"]):
        accs[i].field, accs[i].is_store = fi, st
        accs[i].off[:] = list(o)
    K = ws_kernel()
    K.n_fields, K.n_accesses = nf, na
    K.fields, K.accesses = fields, accs
    K.dom_lo[:] = list(k["dom_lo"])
    K.dom_hi[:] = list(k["dom_hi"])
    K.regs_per_thread = k["regs"]
    K.flops_per_lup = k["flops"]
    K._keep = (fields, accs)
    return K


def gpu_struct(g):
    G = ws_gpu()
    for n in ["n_sm", "max_thr_sm", "max_blk_sm", "max_thr_blk", "regs_sm", "sector_bytes", "line_bytes",
              "n_banks", "bank_bytes", "half_warp", "pair_window_bytes", "l2_sections", "l1_bytes", "l2_bytes"]:
        setattr(G, n, int(g[n]))
    G.clock_hz, G.dram_bw, G.l2_bw = g["clock_hz"], g["dram_bw"], g["l2_bw"]
    for i in range(4):
        for j in range(3):
            G.hit_abc[i][j] = g["hit_abc"][i][j]
    G.page_bytes = int(g.get("page_bytes", 0))
    G.link_bw = float(g.get("link_bw", 0.0))
    return G


def config_array(kernel_id, gpu_id, configs):
    """configs: iterable of (block, fold, blocks_per_sm[, variant]) -> numpy ws_config records."""
    configs = list(configs)
    a = np.zeros(len(configs), dtype=CONFIG_DTYPE)
    for i, c in enumerate(configs):
        b, f, kov = c[:3]
        a[i]["variant"] = c[3] if len(c) > 3 else 0
        a[i]["kernel_id"], a[i]["gpu_id"] = kernel_id, gpu_id
        a[i]["block"] = b
        a[i]["fold"] = f
        a[i]["blocks_per_sm"] = kov
    return a


def result_dicts(res):
    out = []
    for r in res:
        d = {"status": int(r["status"]), "limiter": int(r["limiter"]), "grid": tuple(int(v) for v in r["grid"]),
             "k": int(r["k"]), "wave_blocks": int(r["wave_blocks"]), "n_smsets": int(r["n_smsets"]),
             "n_instr": int(r["n_instr"]), "rank": int(r["rank"])}
        for n in RESULT_U64:
            d[n] = int(r[n])
        for n in RESULT_F64 + RESULT_F64_2:
            d[n] = float(r[n])
        for n in RESULT_U64_2:
            d[n] = int(r[n])
        out.append(d)
    return out


class Context:
    """One ws_ctx on one CUDA device / stream."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self.L = load_library()
        h = C.c_void_p()
        st = self.L.ws_create(int(device), C.c_void_p(stream or 0), C.byref(h))
        if st != WS_OK:
            raise WSError(st, "ws_create failed (a CUDA device is required; there is no CPU fallback)")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.L.ws_destroy(self.h)
            self.h = None

    __del__ = close

    def _check(self, st):
        if st != WS_OK:
            raise WSError(st, self.L.ws_last_error(self.h).decode())

    def set_stream(self, stream: int):
        self._check(self.L.ws_set_stream(self.h, C.c_void_p(stream or 0)))

    def describe_kernel(self, k) -> int:
        K = kernel_struct(k)
        i = U32()
        self._check(self.L.ws_describe_kernel(self.h, C.byref(K), C.byref(i)))
        return i.value

    def describe_gpu(self, g) -> int:
        G = gpu_struct(g)
        i = U32()
        self._check(self.L.ws_describe_gpu(self.h, C.byref(G), C.byref(i)))
        return i.value

    def estimate(self, cfgs: np.ndarray) -> np.ndarray:
        """Host arrays (CONFIG_DTYPE) -> RESULT_DTYPE array; synchronous."""
        cfgs = np.ascontiguousarray(cfgs, dtype=CONFIG_DTYPE)
        out = np.zeros(len(cfgs), dtype=RESULT_DTYPE)
        self._check(self.L.ws_estimate(self.h, cfgs.ctypes.data, len(cfgs), out.ctypes.data))
        return out

    def estimate_async(self, d_cfgs: int, n: int, d_out: int):
        """Device pointers; enqueued on the context stream."""
        self._check(self.L.ws_estimate_async(self.h, C.c_void_p(d_cfgs), n, C.c_void_p(d_out)))

    def estimate_ranked_async(self, d_cfgs: int, n: int, d_out: int, k: int, d_top: int | None):
        """estimate_async + rank_async as one enqueue (model and ranking fused for n <= 1024)."""
        self._check(self.L.ws_estimate_ranked_async(self.h, C.c_void_p(d_cfgs), n, C.c_void_p(d_out), k,
                                                    C.c_void_p(d_top or 0)))

    def estimate_multi(self, cfgs: np.ndarray, gpu_ids) -> np.ndarray:
        """Every configuration against every hardware set: -> (n_gpu, n) RESULT_DTYPE array."""
        cfgs = np.ascontiguousarray(cfgs, dtype=CONFIG_DTYPE)
        ids = np.ascontiguousarray(gpu_ids, dtype=np.uint32)
        out = np.zeros(len(ids) * len(cfgs), dtype=RESULT_DTYPE)
        self._check(self.L.ws_estimate_multi(self.h, cfgs.ctypes.data, len(cfgs), ids.ctypes.data, len(ids),
                                             out.ctypes.data))
        return out.reshape(len(ids), len(cfgs))

    def estimate_multi_async(self, d_cfgs: int, n: int, gpu_ids, d_out: int):
        """Device configurations (n) and results (n * len(gpu_ids)); gpu_ids on the host."""
        ids = np.ascontiguousarray(gpu_ids, dtype=np.uint32)
        self._check(self.L.ws_estimate_multi_async(self.h, C.c_void_p(d_cfgs), n, ids.ctypes.data, len(ids),
                                                   C.c_void_p(d_out)))

    def check_read(self):
        """Bounds-check build counters: (is_check_build, violations, line, index, capacity)."""
        out = (C.c_uint64 * 5)()
        self._check(self.L.ws_check_read(self.h, out))
        return tuple(int(v) for v in out)

    def last_group_count(self) -> int:
        return int(self.L.ws_last_group_count(self.h))

    def rank(self, res: np.ndarray, k: int):
        top = np.zeros(max(1, k), dtype=np.uint32)
        self._check(self.L.ws_rank(self.h, res.ctypes.data, len(res), k, top.ctypes.data))
        return top[:min(k, len(res))]

    def rank_async(self, d_res: int, n: int, k: int, d_top: int | None):
        self._check(self.L.ws_rank_async(self.h, C.c_void_p(d_res), n, k, C.c_void_p(d_top or 0)))

    def last_launch_count(self) -> int:
        return int(self.L.ws_last_launch_count(self.h))

    def profile_enable(self, on: bool = True):
        self._check(self.L.ws_profile_enable(self.h, int(on)))

    def profile_read(self) -> dict:
        """{kernel name: (summed device ms, launches)} since the last read (synchronises)."""
        ms = (F64 * 16)()
        cnt = (U64 * 16)()
        nk = U32()
        self._check(self.L.ws_profile_read(self.h, ms, cnt, 16, C.byref(nk)))
        return {self.L.ws_kernel_name(i).decode(): (ms[i], int(cnt[i])) for i in range(nk.value)}

    def work_read(self) -> dict:
        """{kernel name: algorithmic work units of the last estimate call} (synchronises)."""
        u = (U64 * 16)()
        self._check(self.L.ws_work_read(self.h, u, 16))
        out, i = {}, 0
        while True:
            nm = self.L.ws_kernel_name(i)
            if nm is None:
                break
            out[nm.decode()] = int(u[i])
            i += 1
        return out

    # ------------------------------------------------------------ NEXT-1: simulated hit rates
    def simulate(self, cfgs: np.ndarray, capacities) -> list:
        """Host configs (CONFIG_DTYPE) x capacities (bytes) -> [[dict per capacity] per config]."""
        cfgs = np.ascontiguousarray(cfgs, dtype=CONFIG_DTYPE)
        caps = np.ascontiguousarray(np.asarray(capacities, dtype=np.uint64))
        out = (ws_sim_result * (len(cfgs) * len(caps)))()
        self._check(self.L.ws_simulate(self.h, cfgs.ctypes.data, len(cfgs), caps.ctypes.data, len(caps),
                                       C.addressof(out)))
        rows = []
        for i in range(len(cfgs)):
            row = []
            for k in range(len(caps)):
                r = out[i * len(caps) + k]
                d = {"status": int(r.status)}
                d.update({n: int(getattr(r, n)) for n in SIM_U64})
                d.update({n: float(getattr(r, n)) for n in SIM_F64})
                row.append(d)
            rows.append(row)
        return rows

    def sim_release(self):
        """Free the device buffers simulate() keeps between calls."""
        self._check(self.L.ws_sim_release(self.h))

    def fit_gompertz(self, O, R):
        """Least-squares Gompertz fit on the device -> ((a, b, c), rss)."""
        o = np.ascontiguousarray(np.asarray(O, dtype=np.float64))
        r = np.ascontiguousarray(np.asarray(R, dtype=np.float64))
        abc = np.zeros(3, dtype=np.float64)
        rss = np.zeros(1, dtype=np.float64)
        self._check(self.L.ws_fit_gompertz(self.h, o.ctypes.data, r.ctypes.data, len(o), abc.ctypes.data,
                                           rss.ctypes.data))
        return (float(abc[0]), float(abc[1]), float(abc[2])), float(rss[0])

    # ------------------------------------------------------------ NEXT-2: on-box validation kernel
    def validate_stencil25(self, d_src: int, d_dst: int, n, block, fold, reps: int = 1, stream: int = 0) -> float:
        """Run the 3D-25pt validation kernel (device pointers) `reps` times; average device ms."""
        nn = (C.c_int64 * 3)(*n)
        bb = (U32 * 3)(*block)
        ff = (U32 * 3)(*fold)
        ms = F64()
        st = self.L.ws_validate_stencil25(C.c_void_p(stream or 0), C.c_void_p(d_src), C.c_void_p(d_dst), nn, bb, ff,
                                          int(reps), C.byref(ms))
        if st != WS_OK:
            raise WSError(st, "ws_validate_stencil25 failed")
        return ms.value

    def validate_lbm15(self, d_src: int, d_dst: int, d_phi: int, d_fd: int, n, block, reps: int = 1,
                       stream: int = 0) -> float:
        """Run the LBM15 validation kernel (device pointers) `reps` times; average device ms."""
        nn = (C.c_int64 * 3)(*n)
        bb = (U32 * 3)(*block)
        ms = F64()
        st = self.L.ws_validate_lbm15(C.c_void_p(stream or 0), C.c_void_p(d_src), C.c_void_p(d_dst),
                                      C.c_void_p(d_phi), C.c_void_p(d_fd), nn, bb, int(reps), C.byref(ms))
        if st != WS_OK:
            raise WSError(st, "ws_validate_lbm15 failed")
        return ms.value
