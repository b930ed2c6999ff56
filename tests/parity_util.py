"""Helpers for GPU-vs-oracle parity (tests only)."""
from __future__ import annotations

INT_KEYS = ["status", "grid", "k", "wave_blocks", "n_smsets", "wave_first_block", "lup_wave", "n_instr",
            "l1_wavefronts", "l1_req_ld_sectors", "l1_req_st_sectors", "sm_ld_sectors", "sm_ld_lines",
            "wave_ld_sectors", "wave_st_sectors", "wave_lines", "ly_lines", "lz_lines", "ov_y", "ov_z",
            "addr_evals", "wave_pages", "l2_dup_lines", "l2_link_sectors"]
FP_KEYS = ["O_l1", "R_l1", "O_y", "R_y", "O_z", "R_z", "O_st", "R_st", "l1_cyc_per_lup", "l2_ld_Bpl",
           "l2_st_Bpl", "dram_ld_Bpl", "dram_st_Bpl", "t_l1", "t_l2", "t_dram", "t_pred", "l2_eff_bytes", "t_link"]
# north_star: predicted runtimes agree within 1e-9 relative; the FP64 model differs from the
# oracle only in exp() ulps and FMA contraction.
REL = 1e-9


def close(a, b, rel=REL):
    return a == b or abs(a - b) <= rel * max(abs(a), abs(b))


def compare(gpu, ora, where=""):
    """Element-by-element: integers exact, doubles within REL, limiter exact unless a near-tie."""
    errs = []
    for k in INT_KEYS:
        if gpu[k] != ora[k]:
            errs.append(f"{where} {k}: gpu {gpu[k]} oracle {ora[k]}")
    if ora["status"] != 0:
        return errs
    for k in FP_KEYS:
        if not close(gpu[k], ora[k]):
            errs.append(f"{where} {k}: gpu {gpu[k]!r} oracle {ora[k]!r}")
    if gpu["limiter"] != ora["limiter"]:
        ts = sorted([ora["t_l1"], ora["t_l2"], ora["t_dram"], ora["t_link"]], reverse=True)
        if not close(ts[0], ts[1]):
            errs.append(f"{where} limiter: gpu {gpu['limiter']} oracle {ora['limiter']}")
    return errs


def check_ranking(gpu_ranks, ora_results):
    """GPU ranks must order the oracle's t_pred non-decreasingly (ties / near-ties may permute)."""
    n = len(gpu_ranks)
    order = sorted(range(n), key=lambda i: gpu_ranks[i])
    assert sorted(gpu_ranks) == list(range(n))
    key = [r["t_pred"] if r["status"] == 0 else float("inf") for r in ora_results]
    for a, b in zip(order, order[1:]):
        if key[a] == float("inf"):
            assert key[b] == float("inf")
            continue
        assert key[a] <= key[b] or close(key[a], key[b]), (a, b, key[a], key[b])
