"""Average per-kernel duration (us) of the third estimate in each ncu --metrics gpu__time_duration.sum CSV."""
import csv
import sys
from collections import defaultdict

for path in sys.argv[1:]:
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
    seq = [(r["Kernel Name"].split("(")[0].split("::")[-1], float(r["Metric Value"].replace(",", "")))
           for r in rows if r.get("Metric Name") == "gpu__time_duration.sum"]
    n = len(seq) // 3
    third = seq[2 * n:]
    tot = defaultdict(float)
    for k, v in third:
        tot[k] += v
    unit = rows[0].get("Metric Unit", "ns") if rows else "ns"
    scale = 1e-3 if unit == "nsecond" or unit == "ns" else (1.0 if unit.startswith("u") else 1e3)
    print(path, f"({len(third)} launches, unit {unit})")
    for k, v in tot.items():
        print(f"   {k:12s} {v * scale:9.2f} us")
