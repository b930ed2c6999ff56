"""BJ configs[4] / P:976-1007 (fig:sizescan) on a B200: the layer-condition transition.

The paper scans quadratic XY planes at constant total size (z = 512 * 1024^2 / x^2) and
shows the DRAM volume of a block rising from the layer-condition floor once a block layer no
longer fits the L2 cache, earlier for deeper blocks.  Here: the library's 25pt
kernel (ws_validate_stencil25) at x = y in XS, three block shapes of increasing layer depth
(P:993 series), DRAM bytes per lattice update from ncu against the estimator's prediction with
B200 parameters (126 MB L2 in two sections -> 63 MB effective, so the transition sits at much
larger planes than the A100's ~400).  Also the estimator alone over the whole 168-config
space at every size (ranking stability), and the grid-size sweep 32^3..1024^3.

    python scripts/sizescan.py --time OUT.json
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum -k regex:k_st25 \
        --csv --log-file NCU.csv python scripts/sizescan.py --ncu-pass
    python scripts/sizescan.py --analyze OUT.json NCU.csv PREFIX
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import workloads as W  # noqa: E402
import validate_next2 as V  # noqa: E402

XS = [128, 256, 384, 512, 640, 768, 896, 1024, 1280]
BLOCKS = [((512, 2, 1), (1, 1, 1)), ((128, 1, 8), (1, 1, 1)), ((32, 1, 32), (1, 1, 1))]
TOTAL = 512 * 1024 * 1024


def dims(x):
    return (x, x, max(8, TOTAL // (x * x)))


def run(mode, out=None):
    import torch
    from paper_2204_14242_b200 import Context
    ctx = Context(0)
    res = []
    for x in XS:
        n = dims(x)
        src = torch.rand((n[2] + 8, n[1] + 8, n[0] + 8), dtype=torch.float64, device="cuda")
        dst = torch.zeros_like(src)
        for b, f in BLOCKS:
            if mode == "time":
                ctx.validate_stencil25(src.data_ptr(), dst.data_ptr(), n, b, f, reps=1)
                ms = ctx.validate_stencil25(src.data_ptr(), dst.data_ptr(), n, b, f, reps=3)
                res.append({"n": n, "block": b, "ms": ms, "glups": n[0] * n[1] * n[2] / (ms / 1e3) / 1e9})
            else:
                ctx.validate_stencil25(src.data_ptr(), dst.data_ptr(), n, b, f, reps=1)
        del src, dst
        torch.cuda.empty_cache()
    if mode == "time":
        json.dump(res, open(out, "w"), indent=0)


def analyze(time_json, ncu_csv, prefix):
    from paper_2204_14242_b200 import Context, config_array, result_dicts
    ctx = Context(0)
    g = V.b200_params()
    gid = ctx.describe_gpu(g)
    tm = json.load(open(time_json))
    meas = V.parse_ncu(ncu_csv)
    rows, i = [], 0
    for x in XS:
        n = dims(x)
        k = W.stencil_star(*n, 4, regs=V.REGS)
        kid = ctx.describe_kernel(k)
        pred = result_dicts(ctx.estimate(config_array(kid, gid, [(b, f, 0) for b, f in BLOCKS])))
        for (b, f), p in zip(BLOCKS, pred):
            m, t = meas[i], tm[i]
            i += 1
            lup = float(n[0] * n[1] * n[2])
            rows.append({"x": x, "z": n[2], "block": b, "dram_ld_meas": m["dram__bytes_read.sum"] / lup,
                         "dram_ld_pred": p["dram_ld_Bpl"], "l2_ld_meas": 32 * m["lts__t_sectors_srcunit_tex_op_read.sum"] / lup,
                         "l2_ld_pred": p["l2_ld_Bpl"], "O_z": p["O_z"], "R_z": p["R_z"],
                         "glups_meas": t["glups"], "glups_pred": lup / p["t_pred"] / 1e9})
    # estimator-only: ranking stability and throughput over the grid-size sweep (BJ configs[4])
    import numpy as np
    import torch
    sweep = []
    prev = None
    space = W.space_stencil_paper()
    for nn in (32, 48, 64, 96, 128, 192, 256, 384, 512, 768, 1024):
        kid = ctx.describe_kernel(W.k25(nn))
        cf = config_array(kid, ctx.describe_gpu(W.gpu_a100()), space)
        d_cfg = torch.from_numpy(cf.view(np.uint8).copy()).cuda()
        d_out = torch.empty(len(cf) * 336, dtype=torch.uint8, device="cuda")
        for _ in range(2):
            ctx.estimate_async(d_cfg.data_ptr(), len(cf), d_out.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            ctx.estimate_async(d_cfg.data_ptr(), len(cf), d_out.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        r = result_dicts(ctx.estimate(cf))
        t = [x["t_pred"] for x in r]
        rho = V.spearman(prev, t) if prev is not None else None
        best = min(range(len(t)), key=lambda j: (t[j], j))
        sweep.append({"n": nn, "configs_per_s": len(cf) / (ms / 1e3), "ms": ms,
                      "spearman_vs_previous_size": rho, "best": f"{space[best][0]} fold {space[best][1]}"})
        prev = t
    json.dump({"sizescan": rows, "sweep": sweep}, open(prefix + ".json", "w"), indent=0)
    with open(prefix + ".md", "w") as f:
        f.write("# BJ configs[4] / fig:sizescan on B200: layer-condition transition (P:976-1007)\n\n")
        f.write("Constant volume 512*1024^2 cells, x = y, z = 512*1024^2/x^2 (P:981); 25pt kernel on one B200, "
                "DRAM / L2->L1 bytes per LUP from ncu vs the estimator with B200 parameters (63 MB effective L2).\n\n")
        f.write("| x | z | block | DRAM ld meas | DRAM ld pred | O_z | L2 ld meas | L2 ld pred | GLup/s meas | GLup/s pred |\n")
        f.write("|---|---|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            f.write(f"| {r['x']} | {r['z']} | {r['block']} | {r['dram_ld_meas']:.2f} | {r['dram_ld_pred']:.2f} | "
                    f"{r['O_z']:.2f} | {r['l2_ld_meas']:.1f} | {r['l2_ld_pred']:.1f} | {r['glups_meas']:.1f} | "
                    f"{r['glups_pred']:.1f} |\n")
        f.write("\n## Estimator over the grid-size sweep (168 configs, A100 parameters)\n\n")
        f.write("| n^3 | configs/s | ms per batch | Spearman of t_pred vs previous size | best predicted |\n|---|---|---|---|---|\n")
        for s_ in sweep:
            rho = "" if s_["spearman_vs_previous_size"] is None else f"{s_['spearman_vs_previous_size']:.3f}"
            f.write(f"| {s_['n']} | {s_['configs_per_s']:.0f} | {s_['ms']:.3f} | {rho} | {s_['best']} |\n")
    print(open(prefix + ".md").read())


if __name__ == "__main__":
    if sys.argv[1] == "--time":
        run("time", sys.argv[2])
    elif sys.argv[1] == "--ncu-pass":
        run("ncu")
    else:
        analyze(sys.argv[2], sys.argv[3], sys.argv[4])
