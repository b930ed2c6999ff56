"""Mutation check of the oracle pins (VERDICT r01 "Next round" #2: "each of the four functions fails
when a plausible slip is introduced").

Builds deliberately broken copies of oracle/ws_oracle.cpp under /tmp (one plausible slip each: a
dropped factor, a swapped bandwidth, a wrong divisor, a dropped term, truncating division), points
the oracle loader at each copy (WSO_LIB) and runs tests/test_oracle_pins.py.  Every mutant must
fail at least one pin; the report lists the pins that caught it.

    python scripts/oracle_mutations.py [--out profiles/r02_oracle_mutations.md]
"""
from __future__ import annotations

import argparse
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "ws_oracle.cpp")

# (name, term it breaks, original text, mutated text)
MUTANTS = [
    ("O_l1 over W instead of the SM sets", "O_l1 (Eq. 4, P:683)",
     "/ (double)p.n_sets) / (double)g.l1_bytes", "/ (double)p.W) / (double)g.l1_bytes"),
    ("O_l1 from sectors instead of lines", "O_l1 (P:474-475)",
     "((double)sm_lin * LB", "((double)sm_sec * SB"),
    ("split L2 ignored", "O_y, O_z, O_st (P:322-326)",
     "double l2eff = (double)g.l2_bytes / (double)g.l2_sections;", "double l2eff = (double)g.l2_bytes;"),
    ("O_z from the y-layer lines", "O_z (P:612)",
     "r.O_z = (double)Fz_lines.size()", "r.O_z = (double)Fy_lines.size()"),
    ("O_y from sectors", "O_y (Eq. 4)",
     "r.O_y = (double)Fy_lines.size() * LB", "r.O_y = (double)Fy.size() * SB"),
    ("O_st from sectors", "O_st (P:519-521)",
     "r.O_st = (double)r.wave_lines * LB / l2eff;", "r.O_st = (double)r.wave_lines * SB / l2eff;"),
    ("t_dram without the sector bytes", "t_dram (P:262-281)",
     "r.t_dram = SB * (dram_ld + dram_st)", "r.t_dram = (dram_ld + dram_st)"),
    ("t_dram over the L2 bandwidth", "t_dram (P:313-315)",
     "r.t_dram = SB * (dram_ld + dram_st) / (n * g.dram_bw);", "r.t_dram = SB * (dram_ld + dram_st) / (n * g.l2_bw);"),
    ("t_l2 over the DRAM bandwidth", "t_l2 (P:313-315)",
     "r.t_l2 = SB * (l2l1_ld + l1l2_st) / (n * g.l2_bw);", "r.t_l2 = SB * (l2l1_ld + l1l2_st) / (n * g.dram_bw);"),
    ("t_l2 without the stores", "t_l2 (P:477)",
     "r.t_l2 = SB * (l2l1_ld + l1l2_st)", "r.t_l2 = SB * (l2l1_ld)"),
    ("t_l1 without the SM count", "t_l1 (P:311)",
     "(n * (double)g.n_sm * g.clock_hz)", "(n * g.clock_hz)"),
    ("Eq. 5 with R instead of 1-R", "V_cap L1 (Eq. 5, P:695-698)",
     "(1.0 - r.R_l1) * v_red_l1", "r.R_l1 * v_red_l1"),
    ("Eq. 5 capacity term dropped", "V_cap L1 (Eq. 5)",
     "double l2l1_ld = (double)sm_sec + (1.0 - r.R_l1) * v_red_l1;", "double l2l1_ld = (double)sm_sec;"),
    ("partial-store read-back dropped", "cap_st (P:519-521)",
     "double dram_ld = (double)r.wave_ld_sectors - hits + cap_st;",
     "double dram_ld = (double)r.wave_ld_sectors - hits;"),
    ("partial-store read-back with R", "cap_st (P:519-521)",
     "double cap_st = (1.0 - r.R_st) * red_st;", "double cap_st = r.R_st * red_st;"),
    ("store write-through counted once per sector", "l2_st (P:477)",
     "double l1l2_st = (double)req_st;", "double l1l2_st = (double)r.wave_st_sectors;"),
    ("truncating division of negative addresses", "floordiv (P:499)",
     "if ((a % b) != 0 && (a < 0)) q -= 1;", ""),
    ("layer hits without the z-only remainder", "hits (Q16)",
     "r.R_z * (double)(r.ov_z - r.ov_y)", "r.R_z * (double)(r.ov_z)"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_oracle_mutations.md"))
    a = ap.parse_args()
    src = open(SRC).read()
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    rows = []
    tmpdir = tempfile.mkdtemp(prefix="wso_mut_")
    for i, (name, term, old, new) in enumerate(MUTANTS):
        assert src.count(old) == 1, f"mutation anchor not unique / missing: {name}"
        msrc = os.path.join(tmpdir, f"m{i}.cpp")
        with open(msrc, "w") as f:
            f.write(src.replace(old, new))
        lib = os.path.join(tmpdir, f"libm{i}.so")
        O.build(src=msrc, out=lib)
        env = dict(os.environ, WSO_LIB=lib)
        p = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-q", "-p", "no:cacheprovider",
                            "-o", "addopts=", "--tb=no", "-rf"], cwd=ROOT, env=env, capture_output=True, text=True)
        failed = sorted({m.group(1).split("[")[0] for m in re.finditer(r"FAILED tests/test_oracle_pins.py::(\S+)",
                                                                     p.stdout)})
        if p.returncode < 0 or (p.returncode != 0 and not failed):   # the slip crashes the oracle
            failed = failed + [f"pytest exited {p.returncode} (crash): " + p.stdout.strip().splitlines()[-1][:80]
                               if p.stdout.strip() else f"pytest exited {p.returncode}"]
        caught = p.returncode != 0
        rows.append((name, term, caught, failed))
        print(f"{'CAUGHT' if caught else 'MISSED'}  {name}: {', '.join(failed[:6])}", flush=True)
    with open(a.out, "w") as f:
        f.write("# Oracle mutation check (round 2)\n\n`python scripts/oracle_mutations.py`: each row is a copy of "
                "`oracle/ws_oracle.cpp` with one plausible slip, built under /tmp and loaded via `WSO_LIB`; "
                "`tests/test_oracle_pins.py` is run against it.  A mutant is caught when at least one pin fails.\n\n"
                "| mutant | term | caught | failing pins |\n|---|---|---|---|\n")
        for name, term, caught, failed in rows:
            f.write(f"| {name} | {term} | {'yes' if caught else '**no**'} | {', '.join(failed)} |\n")
        f.write(f"\n{sum(r[2] for r in rows)} of {len(rows)} mutants caught.\n")
    print(f"{sum(r[2] for r in rows)} of {len(rows)} caught -> {a.out}")
    return 0 if all(r[2] for r in rows) else 1


if __name__ == "__main__":
    sys.exit(main())
