"""on-box validation of the estimator against the modelled workload.

The paper validates its per-level volume predictions and its ranking against hardware counters
of the 3D-25pt stencil.  Here the same on a B200: the library's sm_100a 25pt
kernel (ws_validate_stencil25) runs every configuration of the 168-config paper space on
512^3; ncu counts per launch

  l1tex__t_sectors_pipe_lsu_mem_global_op_ld   L1 requested load sectors   (model: l1_req_ld_sectors, V_up^L1)
  l1tex__data_pipe_lsu_wavefronts              L1 wavefronts               (model: l1_wavefronts)
  lts__t_sectors_srcunit_tex_op_read / _write  L2<-L1 loads / L1->L2 stores (model: l2_ld_Bpl / l2_st_Bpl)
  dram__bytes_read / _write                    DRAM loads / stores         (model: dram_ld_Bpl / dram_st_Bpl)

and CUDA events time each configuration (GLup/s).  The estimator (this repo's GPU path)
predicts the same quantities with B200 parameters (148 SMs, measured HBM bandwidth, 126 MB
L2 in 2 sections, the kernel's 32 registers/thread for the occupancy).

    python scripts/validate_next2.py --time OUT.json
    ncu --metrics <above>,gpu__time_duration.sum -k regex:k_st25 --csv --log-file NCU.csv \
        python scripts/validate_next2.py --ncu-pass
    python scripts/validate_next2.py --analyze OUT.json NCU.csv PREFIX   (-> PREFIX.md, PREFIX.json)
"""
import csv
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402

N = 512
REGS = 32   # registers/thread of k_st25 (cuobjdump --dump-resource-usage)
LBM = os.environ.get("WS_VALIDATE", "k25") == "lbm15"
if LBM:
    N = 256
    REGS = 128   # k_lbm15: __launch_bounds__(512, 1) -> 128 registers ("at most 512 threads")
METRICS = ["gpu__time_duration.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
           "l1tex__data_pipe_lsu_wavefronts.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
           "lts__t_sectors_srcunit_tex_op_write.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]


def fields():
    import torch
    if LBM:
        shp = (N + 2, N + 2, N + 2)
        src = torch.rand((15,) + shp, dtype=torch.float64, device="cuda")
        phi = torch.rand(shp, dtype=torch.float64, device="cuda")
        return src, torch.zeros_like(src), phi, torch.zeros_like(phi)
    src = torch.rand((N + 8, N + 8, N + 8), dtype=torch.float64, device="cuda")
    return src, torch.zeros_like(src)


def space():
    return W.space_lbm() if LBM else W.space_stencil_paper()


def kernel_desc():
    if LBM:
        k = W.lbm15(N)
        k["regs"] = REGS
        return k
    return W.stencil_star(N, N, N, 4, regs=REGS)


def launch(ctx, fl, b, f, reps):
    if LBM:
        return ctx.validate_lbm15(fl[0].data_ptr(), fl[1].data_ptr(), fl[2].data_ptr(), fl[3].data_ptr(),
                                  (N, N, N), b, reps=reps)
    return ctx.validate_stencil25(fl[0].data_ptr(), fl[1].data_ptr(), (N, N, N), b, f, reps=reps)


def run(mode, out=None):
    import torch
    from paper_2204_14242_b200 import Context
    ctx = Context(0)
    fl = fields()
    res = []
    for (b, f, _k) in space():
        if mode == "time":
            launch(ctx, fl, b, f, 1)
            ms = launch(ctx, fl, b, f, 5)
            res.append({"block": b, "fold": f, "ms": ms, "glups": N ** 3 / (ms / 1e3) / 1e9})
        else:
            launch(ctx, fl, b, f, 1)
    torch.cuda.synchronize()
    if mode == "time":
        json.dump(res, open(out, "w"), indent=0)


def parse_ncu(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    iid, iname, ival, ikern = h.index("ID"), h.index("Metric Name"), h.index("Metric Value"), h.index("Kernel Name")
    by = {}
    for r in rows[start + 1:]:
        if len(r) <= ival or ("k_st25" not in r[ikern] and "k_lbm15" not in r[ikern]):
            continue
        by.setdefault(int(r[iid]), {})[r[iname]] = float(r[ival].replace(",", ""))
    return [by[k] for k in sorted(by)]


def spearman(a, b):
    def ranks(v):
        order = sorted(range(len(v)), key=lambda i: v[i])
        r = [0.0] * len(v)
        i = 0
        while i < len(order):
            j = i
            while j + 1 < len(order) and v[order[j + 1]] == v[order[i]]:
                j += 1
            for q in range(i, j + 1):
                r[order[q]] = (i + j) / 2.0
            i = j + 1
        return r
    ra, rb = ranks(a), ranks(b)
    ma, mb = sum(ra) / len(ra), sum(rb) / len(rb)
    num = sum((x - ma) * (y - mb) for x, y in zip(ra, rb))
    den = math.sqrt(sum((x - ma) ** 2 for x in ra) * sum((y - mb) ** 2 for y in rb))
    return num / den if den else float("nan")


def b200_params():
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    return W.gpu_b200_like(pk.get("hbm_gbs", 6546.2))


def analyze(time_json, ncu_csv, prefix, hit_abc=None, title_note="Hit-rate curves: SURVEY Q17 defaults (not calibrated to B200)."):
    from paper_2204_14242_b200 import Context, config_array, result_dicts
    k = kernel_desc()
    g = b200_params()
    if hit_abc is not None:
        g["hit_abc"] = [list(t) for t in hit_abc]
    ctx = Context(0)
    sp = space()
    pred = result_dicts(ctx.estimate(config_array(ctx.describe_kernel(k), ctx.describe_gpu(g), sp)))
    tm = json.load(open(time_json))
    meas = parse_ncu(ncu_csv)
    assert len(meas) == len(sp) == len(tm), (len(meas), len(sp), len(tm))
    lup = float(N ** 3)
    rows = []
    for c, p, t, m in zip(sp, pred, tm, meas):
        rows.append({
            "block": c[0], "fold": c[1], "limiter": ["L1", "L2", "DRAM", "link"][p["limiter"]],
            "l1_sec_Bpl": (32 * m["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"] / lup,
                           32 * p["l1_req_ld_sectors"] / p["lup_wave"]),
            "l1_wf_per_lup": (m["l1tex__data_pipe_lsu_wavefronts.sum"] / lup, p["l1_cyc_per_lup"]),
            "l2_ld_Bpl": (32 * m["lts__t_sectors_srcunit_tex_op_read.sum"] / lup, p["l2_ld_Bpl"]),
            "l2_st_Bpl": (32 * m["lts__t_sectors_srcunit_tex_op_write.sum"] / lup, p["l2_st_Bpl"]),
            "dram_ld_Bpl": (m["dram__bytes_read.sum"] / lup, p["dram_ld_Bpl"]),
            "dram_st_Bpl": (m["dram__bytes_write.sum"] / lup, p["dram_st_Bpl"]),
            "glups": (t["glups"], lup / p["t_pred"] / 1e9),
        })
    keys = ["l1_sec_Bpl", "l1_wf_per_lup", "l2_ld_Bpl", "l2_st_Bpl", "dram_ld_Bpl", "dram_st_Bpl", "glups"]
    summ = {}
    for key in keys:
        errs = sorted(abs(r[key][1] - r[key][0]) / r[key][0] for r in rows if r[key][0] > 0)
        summ[key] = {"median_abs_rel_err": errs[len(errs) // 2], "p90_abs_rel_err": errs[int(0.9 * len(errs))],
                     "spearman": spearman([r[key][0] for r in rows], [r[key][1] for r in rows])}
    meas_g = [r["glups"][0] for r in rows]
    pred_g = [r["glups"][1] for r in rows]
    best_pred = max(range(len(rows)), key=lambda i: (pred_g[i], -i))
    order = sorted(range(len(rows)), key=lambda i: -meas_g[i])
    summ["ranking"] = {
        "spearman_pred_vs_measured_glups": spearman(meas_g, pred_g),
        "best_predicted": f"{rows[best_pred]['block']} fold {rows[best_pred]['fold']}",
        "best_predicted_measured_rank": order.index(best_pred) + 1,
        "best_predicted_fraction_of_best_measured": meas_g[best_pred] / max(meas_g),
        "best_measured": f"{rows[order[0]]['block']} fold {rows[order[0]]['fold']}",
        "best_measured_glups": max(meas_g),
        "top10_predicted_in_measured_top10": len(set(sorted(range(len(rows)), key=lambda i: -pred_g[i])[:10])
                                                 & set(order[:10])),
    }
    json.dump({"summary": summ, "rows": rows, "gpu": g["name"], "regs": REGS}, open(prefix + ".json", "w"), indent=0)
    with open(prefix + ".md", "w") as f:
        f.write(("# NEXT-2 on-box validation: LBM15 (D3Q15 pull + 7pt phase field) 256^3, 49 configs" if LBM else
                 "# NEXT-2 on-box validation: 3D-25pt r4 512^3, 168 configs") +
                ", B200 (measured) vs estimator (B200 parameters)\n\n")
        f.write("Per-level volumes per lattice update (ncu counters / 512^3) against the estimator's prediction; "
                "GLup/s from CUDA events (5 launches each).  " + title_note + "\n\n")
        f.write("| quantity | median abs rel err | p90 abs rel err | Spearman (measured vs predicted) |\n|---|---|---|---|\n")
        for key in keys:
            s = summ[key]
            f.write(f"| {key} | {s['median_abs_rel_err']:.3f} | {s['p90_abs_rel_err']:.3f} | {s['spearman']:.3f} |\n")
        f.write("\nRanking: " + json.dumps(summ["ranking"]) + "\n\n")
        f.write("| block | fold | limiter (pred) | " + " | ".join(f"{k} meas / pred" for k in keys) + " |\n")
        f.write("|---|---|---|" + "---|" * len(keys) + "\n")
        for r in rows:
            f.write(f"| {r['block']} | {r['fold']} | {r['limiter']} | " +
                    " | ".join(f"{r[k][0]:.2f} / {r[k][1]:.2f}" for k in keys) + " |\n")
    print(json.dumps(summ, indent=1))
    return summ


if __name__ == "__main__":
    if sys.argv[1] == "--time":
        run("time", sys.argv[2])
    elif sys.argv[1] == "--ncu-pass":
        run("ncu")
    else:
        analyze(sys.argv[2], sys.argv[3], sys.argv[4])
