"""Per-kernel device times of the 168-config 25pt space at n^3 (A100 parameters), WS_SERIAL optional.

    python scripts/probe_n.py 64"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from probe import run  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
run(f"K25 {n}^3 A100 168", W.k25(n), W.gpu_a100(), W.space_stencil_paper())
