"""Summarise an `ncu --set full` report into a markdown table + per-kernel DRAM traffic JSON.

    python scripts/ncu_summary.py gpurun_out/full.ncu-rep profiles/r01_ncu_summary.md profiles/ncu_traffic.json

Reads `ncu -i <rep> --page raw --csv`; one row per profiled launch (kernels profiled more
than once are averaged).  The traffic JSON (dram__bytes_read.sum + dram__bytes_write.sum
per launch, bytes) is what bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

COLS = [
    ("duration us", "gpu__time_duration.sum", 1e-3),
    ("warp inst", "smsp__inst_executed.sum", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("grid", "launch__grid_size", 1),
    ("occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("issue active %", "sm__issue_active.avg.pct_of_peak_sustained_elapsed", 1),
    ("ALU pipe %", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    ("FMA pipe %", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    ("LSU pipe %", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    ("DRAM read MB", "dram__bytes_read.sum", 1e-6),
    ("DRAM write MB", "dram__bytes_write.sum", 1e-6),
]


def to_float(s, unit):
    s = s.replace(",", "")
    try:
        v = float(s)
    except ValueError:
        return None
    # normalise units ncu prints in the second header row
    scale = {"ns": 1.0, "us": 1e3, "ms": 1e6, "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "byte": 1.0,
             "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
    return v * scale


def main(rep, md_out, traffic_out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(head)}
    acc = defaultdict(lambda: defaultdict(list))
    order = []
    for r in data:
        name = r[idx["Kernel Name"]].split("(")[0].split("<")[0].replace("wsb::", "")
        if name not in acc:
            order.append(name)
        for label, metric, _ in COLS:
            if metric in idx:
                v = to_float(r[idx[metric]], units[idx[metric]])
                if v is not None:
                    acc[name][label].append(v)
    lines = ["| kernel | launches | " + " | ".join(c[0] for c in COLS) + " |",
             "|---|---|" + "---|" * len(COLS)]
    traffic = {}
    for name in order:
        cells = []
        n = 0
        for label, metric, scale in COLS:
            vs = acc[name][label]
            n = max(n, len(vs))
            if not vs:
                cells.append("")
                continue
            v = sum(vs) / len(vs) * scale
            cells.append(f"{v:.4g}" if abs(v) < 1e6 else f"{v:.4e}")
        rd, wr = acc[name]["DRAM read MB"], acc[name]["DRAM write MB"]
        if rd and wr:
            traffic[name] = sum(rd) / len(rd) + sum(wr) / len(wr)
        wi = acc[name]["warp inst"]
        if wi:
            traffic[name + ":warp_inst"] = sum(wi) / len(wi)
        lines.append(f"| {name} | {n} | " + " | ".join(cells) + " |")
    with open(md_out, "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(traffic_out, "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])
