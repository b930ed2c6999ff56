"""Full-space, full-size parity: the CUDA path through the C ABI against oracle golden files.

`tests/golden/full_*.json` are written by `scripts/oracle_golden.py`, which calls only `oracle/`
(one single-threaded oracle run per configuration, every (thread, instruction) address into
std::set).  Each GPU test runs a whole golden set in ONE `ws_estimate` launch — the launch
configuration `bench.py` times — and compares every record element by element: integers
bit-exact, doubles within 1e-9 relative (BASELINE.json north_star; `parity_util.compare`).

Sets (BASELINE.json configs; sweep space P:727-733; best configurations P:1029-1031):
configs[1] 25pt 512^3 A100 (168), configs[2] LBM15 / LBM27 256^3 A100 (49 each), configs[3]
25pt 512^3 and LBM15 256^3 with the B200-like parameter set, configs[4] the grid-size sweep
32^3-256^3 (168 each) and deep 1024^3 samples incl. (16,1,64)+2z and (16,2,32)+2z.

The `-m "not gpu"` tests check that every golden file matches the current workload
descriptions (hash of the plain description) and re-run the oracle on the cheapest entry of
each file (the stored values are the current oracle's).
"""
import glob
import json
import os

import pytest

import workloads as W
from parity_util import compare

HERE = os.path.dirname(os.path.abspath(__file__))
FILES = sorted(glob.glob(os.path.join(HERE, "golden", "full_*.json")))
NAMES = [os.path.basename(f)[5:-5] for f in FILES]


def _sets():
    import importlib.util
    spec = importlib.util.spec_from_file_location("oracle_golden", os.path.join(HERE, "..", "scripts",
                                                                                 "oracle_golden.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def load(name):
    with open(os.path.join(HERE, "golden", f"full_{name}.json")) as f:
        doc = json.load(f)
    cfgs = [(tuple(b), tuple(fo), k) for b, fo, k in doc["configs"]]
    return doc, cfgs


@pytest.fixture(scope="module")
def gsets():
    return _sets()


@pytest.mark.parametrize("name", NAMES)
def test_golden_matches_workloads(name, gsets):
    """Golden file describes today's workload (kernel / GPU descriptions and configuration list)."""
    doc, cfgs = load(name)
    k, g, cs = gsets.sets()[name]
    assert doc["kernel_sha"] == gsets.desc_hash(k), f"{name}: kernel description changed; regenerate"
    assert doc["gpu_sha"] == gsets.desc_hash(g), f"{name}: GPU description changed; regenerate"
    assert cfgs == [(tuple(c[0]), tuple(c[1]), c[2]) for c in cs]
    assert len(doc["results"]) == len(cfgs) and all(r is not None for r in doc["results"])


@pytest.mark.parametrize("name", NAMES)
def test_golden_is_current_oracle(name, gsets):
    """The cheapest stored record is reproduced by the current oracle, field by field."""
    from oracle import oracle as O
    doc, cfgs = load(name)
    k, g, _ = gsets.sets()[name]
    i = min(range(len(cfgs)), key=lambda j: doc["results"][j]["addr_evals"])
    r = O.estimate(k, g, cfgs[i])
    r["grid"] = list(r["grid"])
    errs = compare(r, doc["results"][i], f"{name}[{i}]")
    assert not errs, "\n".join(errs)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_full_space_vs_golden(name, gsets):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2204_14242_b200 import Context, config_array, result_dicts
    doc, cfgs = load(name)
    k, g, _ = gsets.sets()[name]
    ctx = Context(0)
    kid, gid = ctx.describe_kernel(k), ctx.describe_gpu(g)
    res = result_dicts(ctx.estimate(config_array(kid, gid, cfgs)))
    errs = []
    for i, (a, b) in enumerate(zip(res, doc["results"])):
        a = dict(a, grid=list(a["grid"]))
        errs += compare(a, b, f"{name}[{i}] {cfgs[i]}")
    ctx.close()
    assert not errs, f"{len(errs)} mismatches\n" + "\n".join(errs[:40])
    # the space is fully evaluated (no failed configuration hides a skipped comparison)
    assert sum(r["status"] == 0 for r in res) == sum(r["status"] == 0 for r in doc["results"]) > 0
