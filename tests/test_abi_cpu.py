"""CPU-side checks of the C-ABI library: it builds, loads, exports every symbol
include/ws.h declares, the Python mirrors match the header layout, and it
refuses to run without a GPU (no CPU fallback)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "ws.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ws_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_exports_header_symbols():
    from paper_2204_14242_b200 import build, ws
    build.build()
    L = ws.load_library()
    names = _header_functions()
    assert "ws_estimate" in names and "ws_describe_kernel" in names and "ws_rank" in names
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(ws.EXPORTS)


def test_struct_layouts():
    import ctypes as C
    from paper_2204_14242_b200 import ws
    assert C.sizeof(ws.ws_config) == 40
    assert C.sizeof(ws.ws_result) == 336
    assert C.sizeof(ws.ws_field) == 64
    assert C.sizeof(ws.ws_access) == 20
    src = open(os.path.join(ROOT, "include", "ws.h")).read()
    assert "/* 336 bytes */" in src and "/* 40 bytes */" in src and "/* 160 bytes */" in src
    assert C.sizeof(ws.ws_sim_result) == 160


def test_sm100a_cubin_present():
    """The shared library carries sm_100a SASS (not PTX-only / not another arch)."""
    import subprocess
    from paper_2204_14242_b200 import ws
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", ws.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2204_14242_b200 import ws
    with pytest.raises(ws.WSError):
        ws.Context(0)


def test_product_does_not_import_oracle():
    for dp, _, fs in os.walk(os.path.join(ROOT, "paper_2204_14242_b200")):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                s = open(os.path.join(dp, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|libwsoracle|#include\s+[<\"].*oracle)", s), f
