"""SURVEY 4 test layer 5 without compute-sanitizer (closed on this GPU pool): the bounds-check
build (-DWS_CHECK, libwsb200_check.so) runs the estimate chain on the paper's workloads at full
size, on the extended space, the variants / outlook metrics, the fused model + rank path, the
multi-hardware fan-out and the simulator, and every dynamically computed scratch index is checked
against its capacity on the device (ws_check_read must report zero violations)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bounds_check_build_clean():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2204_14242_b200 import build as B
    lib = B.CHECK_LIB
    assert os.path.exists(lib), "libwsb200_check.so missing: __graft_entry__.build() builds it"
    env = dict(os.environ, WS_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "check_target.py")], capture_output=True,
                       text=True, env=env, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "bounds check target ok" in out, out[-2000:]
