"""The estimator's alternate launch paths against the oracle, each in a fresh process (the
switches are read once per process): fold by CTA / by warp (WS_FOLD_MODE), every chain on the
context stream (WS_SERIAL), eager launches instead of CUDA-graph replay (WS_GRAPH=0), batches split into scratch-bounded chunks
(WS_SCRATCH_MB)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("env", [{"WS_FOLD_MODE": "1"}, {"WS_FOLD_MODE": "2"}, {"WS_SERIAL": "1"},
                                 {"WS_GRAPH": "0"}, {"WS_SCRATCH_MB": "8"}],
                         ids=["fold-cta", "fold-warp", "serial", "eager", "chunked"])
def test_launch_modes(env):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    r = subprocess.run([sys.executable, os.path.join(HERE, "mode_target.py")], capture_output=True, text=True,
                       env=dict(os.environ, **env), timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "mode target ok" in out
