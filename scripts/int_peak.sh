# measured integer issue peak (scripts/int_peak.cu): event-timed rates + ncu executed warp instructions
set -e
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/int_peak scripts/int_peak.cu
/tmp/int_peak > gpurun_out/int_peak_events.json
ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --csv /tmp/int_peak > gpurun_out/int_peak_ncu.csv 2>/dev/null || true
python - <<'PY'
import csv, io, json
ev = json.load(open("gpurun_out/int_peak_events.json"))
allr = list(csv.reader(io.StringIO(open("gpurun_out/int_peak_ncu.csv").read())))
h0 = next(i for i, r in enumerate(allr) if r and r[0] == "ID")
hdr, rows = allr[h0], [hdr_r for hdr_r in allr[h0:] if len(hdr_r) == len(allr[h0])]
k, m, v = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
per = {}
for r in rows[1:]:
    name = r[k].split("(")[0]
    mode = {"void k_int<0>": "alu", "void k_int<1>": "mix", "void k_int<2>": "mix_shfl"}.get(name, name)
    per.setdefault(mode, {}).setdefault(r[m], []).append(float(r[v].replace(",", "")))
out = dict(ev)
for mode, ms in zip(("alu", "mix", "mix_shfl"), ev["ms"]):
    inst = max(per[mode]["smsp__inst_executed.sum"])
    out[f"warp_inst_per_launch_{mode}"] = inst
    out[f"warp_inst_per_s_{mode}"] = inst / (ms * 1e-3)
    out[f"issue_active_pct_{mode}"] = max(per[mode]["smsp__issue_active.avg.pct_of_peak_sustained_active"])
out["issue_peak_measured_warp_inst_per_s"] = max(out[f"warp_inst_per_s_{m}"] for m in ("alu", "mix", "mix_shfl"))
out["issue_peak_nominal_warp_inst_per_s"] = ev["nominal_issue_peak"] / 32
out["how"] = ("executed warp instructions per launch (ncu smsp__inst_executed.sum) / the launch's best CUDA-event "
              "time: the measured integer issue rate the estimator kernels' executed instruction mix is compared with")
json.dump(out, open("gpurun_out/int_peak.json", "w"), indent=1)
print(json.dumps(out))
PY
