"""Top CUDA source lines of one kernel in an ncu report by warp-stall samples.

    python scripts/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [N]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
agg = {}
cur = None
for r in rows[hi + 1:]:
    if not r:
        continue
    if r[0]:  # a CUDA source line row (its sass rows follow with an empty Line No)
        if not r[0].isdigit():  # a new file / function header
            cur = None
            continue
        cur = (int(r[0]), r[1].strip()[:100])
        agg.setdefault(cur, [0, 0])
        continue
    if cur is None:
        continue
    try:
        agg[cur][0] += int(r[iss] or 0)
        agg[cur][1] += int(r[iex] or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()) or 1
print(f"total stall samples {tot}, warp instructions {sum(v[1] for v in agg.values())}")
for (ln, src), (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * s / tot:5.1f}%  {e:10d}  L{ln:5d}  {src}")
