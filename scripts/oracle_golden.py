"""Write full-space oracle golden files under tests/golden/ (VERDICT r01 "Next round" #1).

Imports only `oracle/` (the CPU oracle, test infrastructure) and `workloads/` (plain input
descriptions, no estimator arithmetic): every stored value is the oracle's.  Nothing here
touches the CUDA path.

Sets (BASELINE.json configs, P:727-733 sweep space, P:1029-1031 best configurations):
  c1_k25_512_a100    configs[1]: 3D-25pt r4, 512^3, all 168 configurations, A100
  c2_lbm15_256_a100  configs[2]: LBM D3Q15 + phase field, 256^3, all 49 configurations
  c2_lbm27_256_a100  configs[2]: LBM D3Q27 variant, 256^3, all 49 configurations
  c3_k25_512_b200    configs[3]: the 168 configurations with the B200-like parameter set
  c3_lbm15_256_b200  configs[3]: the 49 LBM15 configurations with the B200-like parameter set
  c4_k25_{32,64,128,256}_a100   configs[4]: the grid-size sweep, all 168 configurations each
  c4_k25_1024_a100   configs[4]: deep samples at 1024^3 incl. (16,1,64)+2z and (16,2,32)+2z

Every configuration is one single-threaded oracle call (`oracle.estimate`); a thread pool runs
them largest first (cost = the oracle's own `addr_evals`), bounded by an estimated memory budget.
Per-configuration wall seconds are stored too: they are the honest full-space oracle timing
(`host` records the CPU model, threads and RAM).

Usage: python scripts/oracle_golden.py [set ...] [--threads N] [--mem-gb G] [--force]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import hashlib
import json
import os
import platform
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from oracle import oracle as O  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")

# 1024^3 samples: the deepest configurations of the space and the paper's named ones
C4_1024 = [((16, 1, 64), (1, 1, 2), 0), ((16, 2, 32), (1, 1, 2), 0), ((64, 4, 4), (1, 1, 2), 0),
           ((32, 32, 1), (1, 2, 1), 0), ((1024, 1, 1), (1, 1, 1), 0), ((256, 4, 1), (1, 1, 1), 0),
           ((8, 8, 16), (1, 1, 1), 0), ((32, 1, 32), (1, 2, 1), 0)]


def sets():
    S = W.space_stencil_paper()
    L = W.space_lbm()
    out = {
        "c1_k25_512_a100": (W.k25(512), W.gpu_a100(), S),
        "c2_lbm15_256_a100": (W.lbm15(256), W.gpu_a100(), L),
        "c2_lbm27_256_a100": (W.lbm27(256), W.gpu_a100(), L),
        "c3_k25_512_b200": (W.k25(512), W.gpu_b200_like(), S),
        "c3_lbm15_256_b200": (W.lbm15(256), W.gpu_b200_like(), L),
        "c4_k25_1024_a100": (W.k25(1024), W.gpu_a100(), C4_1024),
    }
    for n in (32, 64, 128, 256):
        out[f"c4_k25_{n}_a100"] = (W.k25(n), W.gpu_a100(), S)
    return out


def desc_hash(obj) -> str:
    """Hash of a plain description (kernel / gpu dict), to detect workload drift in the tests."""
    return hashlib.sha256(json.dumps(obj, sort_keys=True).encode()).hexdigest()[:16]


def host_info():
    model = platform.processor()
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    mem = 0
    try:
        with open("/proc/meminfo") as f:
            mem = int(f.readline().split()[1]) // (1024 * 1024)
    except OSError:
        pass
    return {"cpu": model, "nproc": os.cpu_count(), "ram_gib": mem}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--mem-gb", type=float, default=40.0)
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    all_sets = sets()
    names = a.names or list(all_sets)
    todo = []   # (cost, set name, index)
    state = {}
    for n in names:
        path = os.path.join(GOLD, f"full_{n}.json")
        if os.path.exists(path) and not a.force:
            print(f"{n}: exists, skipped", flush=True)
            continue
        k, g, cs = all_sets[n]
        costs = [O.plan(k, g, c)["addr_evals"] for c in cs]
        state[n] = {"res": [None] * len(cs), "sec": [0.0] * len(cs), "left": len(cs), "path": path}
        todo += [(costs[i], n, i) for i in range(len(cs))]
    todo.sort(key=lambda t: -t[0])
    budget = int(a.mem_gb * 1e9)
    cv = threading.Condition()
    used = [0]
    lock = threading.Lock()
    t_start = time.time()

    def mem_of(cost):        # measured: ~2.6 B of RSS per address evaluation (std::set nodes)
        return min(budget, int(cost * 3.0) + (64 << 20))

    def write(n):
        k, g, cs = all_sets[n]
        st = state[n]
        doc = {
            "what": f"oracle results for golden set {n} (scripts/oracle_golden.py; only oracle/ computed them)",
            "kernel": k["name"], "kernel_sha": desc_hash(k), "gpu": g["name"], "gpu_sha": desc_hash(g),
            "host": host_info(), "oracle_threads_each": 1,
            "configs": [[list(c[0]), list(c[1]), c[2]] for c in cs],
            "oracle_seconds": st["sec"], "results": st["res"],
        }
        tmp = st["path"] + ".tmp"
        with open(tmp, "w") as f:
            json.dump(doc, f, separators=(",", ":"))
        os.replace(tmp, st["path"])
        print(f"{n}: written ({len(cs)} configs, {sum(st['sec']):.0f} thread-s)", flush=True)

    def run(item):
        cost, n, i = item
        need = mem_of(cost)
        with cv:
            while used[0] + need > budget and used[0] > 0:
                cv.wait()
            used[0] += need
        try:
            k, g, cs = all_sets[n]
            t0 = time.time()
            r = O.estimate(k, g, cs[i])
            dt = time.time() - t0
        finally:
            with cv:
                used[0] -= need
                cv.notify_all()
        with lock:
            st = state[n]
            st["res"][i], st["sec"][i] = r, dt
            st["left"] -= 1
            done = st["left"] == 0
        if done:
            write(n)
        return cost, dt

    total = sum(t[0] for t in todo)
    done_cost = 0
    with cf.ThreadPoolExecutor(a.threads) as ex:
        for cost, dt in ex.map(run, todo):
            done_cost += cost
            el = time.time() - t_start
            print(f"[{el:7.0f}s] {done_cost / total * 100:5.1f}% of {total:.3g} evals  (last {dt:.1f}s)",
                  flush=True)


if __name__ == "__main__":
    main()
