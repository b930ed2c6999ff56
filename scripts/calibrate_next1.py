"""NEXT-1 + NEXT-2: calibrate the four hit-rate curves for B200 by LRU simulation and re-check
the on-box validation.

SURVEY 8(f) NEXT-1: the paper fits R(O) = a exp(-b exp(-c O)) to hit rates measured with
hardware counters; here the samples come from ws_simulate (sectored LRU
replay of each configuration's own request streams) on the 168-config 25pt space at 128^3 with
B200 parameters, at capacities from 16 KiB to 32 MiB so that O spans the curves' transition, and
ws_fit_gompertz fits each curve on the device.  The calibrated curves then replace the Q17
defaults in the 512^3 predictions and the NEXT-2 comparison (counters from
profiles/r01_next2_ncu.csv, timings from profiles/r01_next2_times.json) is redone.

    python scripts/calibrate_next1.py OUT_PREFIX
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import workloads as W  # noqa: E402
import validate_next2 as V  # noqa: E402

NCAL = int(os.environ.get("WS_CAL_N", "128"))   # grid of the simulated calibration sweep


def main(prefix):
    from paper_2204_14242_b200 import Context, config_array
    ctx = Context(0)
    g = V.b200_params()
    k = W.stencil_star(NCAL, NCAL, NCAL, 4, regs=V.REGS)
    space = W.space_stencil_paper()
    caps = [1 << e for e in range(14, 26)] if NCAL <= 128 else [1 << e for e in range(16, 28)]
    cf = config_array(ctx.describe_kernel(k), ctx.describe_gpu(g), space)
    t0 = time.time()
    rows = ctx.simulate(cf, caps)
    sim_s = time.time() - t0
    curves = {"L1": ("O_l1", "R_l1", lambda r: r["l1_requests"] > r["l1_compulsory"]),
              "L2y": ("O_y", "R_y", lambda r: r["ov_y"] > 0),
              "L2z": ("O_z", "R_z", lambda r: r["ov_z_only"] > 0),
              "L2st": ("O_st", "R_st", lambda r: r["st_requests"] > r["st_compulsory"])}
    fits, info = [], {}
    for name, (ok, rk, use) in curves.items():
        Os = [r[ok] for row in rows for r in row if r["status"] == 0 and use(r) and r[ok] <= 16.0]
        Rs = [r[rk] for row in rows for r in row if r["status"] == 0 and use(r) and r[ok] <= 16.0]
        if len(Os) >= 3:
            abc, rss = ctx.fit_gompertz(Os, Rs)
        else:
            abc, rss = tuple(W.HIT_ABC_DEFAULT[len(fits)]), None
        fits.append(abc)
        info[name] = {"abc": abc, "samples": len(Os), "rss": rss,
                      "R_at_O": {o: W_hit(abc, o) for o in (0.5, 1.0, 2.0, 4.0)}}
    out = {"workload": f"25pt 168 configs at {NCAL}^3, B200 parameters, capacities {caps[0]}..{caps[-1]} B ({len(caps)})",
           "simulate_wall_s": sim_s, "curves": info}
    res = V.analyze(os.path.join(ROOT, "profiles", "r01_next2_times.json"),
                    os.path.join(ROOT, "profiles", "r01_next2_ncu.csv"), prefix + "_validation", hit_abc=fits,
                    title_note="Hit-rate curves: fitted to LRU-simulated samples (NEXT-1, scripts/calibrate_next1.py).")
    out["validation_with_calibrated_curves"] = res
    json.dump(out, open(prefix + ".json", "w"), indent=1)
    print(json.dumps(out, indent=1))


def W_hit(abc, O):
    import math
    return abc[0] * math.exp(-abc[1] * math.exp(-abc[2] * O))


if __name__ == "__main__":
    main(sys.argv[1])
