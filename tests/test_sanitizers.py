"""SURVEY 4 test layer 5: compute-sanitizer (memcheck, racecheck, synccheck) over a tiny
workload that launches every kernel of the library once (scripts/sanitize_target.py)."""
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    env = dict(os.environ, WS_GRAPH="0")
    r = subprocess.run([SAN, "--tool", tool, "--error-exitcode", "3", "python",
                        os.path.join(ROOT, "scripts", "sanitize_target.py")],
                       capture_output=True, text=True, env=env, timeout=1200)
    out = r.stdout + r.stderr
    if r.returncode == 86 and "closed on this pool" in out:
        # the GPU pool's compute-sanitizer wrapper refuses every run (exit 86); the in-library
        # bounds checks (WS_CHECK build, tests/test_gpu_round2.py) stand in for memcheck there
        pytest.skip("compute-sanitizer closed on this GPU pool: " + out.strip().splitlines()[-1][:200])
    assert r.returncode == 0, out[-4000:]
    assert "sanitize target ok" in out
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-2000:]
