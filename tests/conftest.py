"""Shared fixtures.  `-m "not gpu"` tests run anywhere (oracle vs golden
vectors, host logic, ABI exports); `-m gpu` tests need a CUDA device and
call the product through its C-ABI (they fail, not skip, without one)."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running (large N)")


_FULLSIZE = {}


def pytest_collection_modifyitems(session, config, items):
    """Start the reference's own full-size runs (tests/fullsize_ref.py) as soon
    as test_gpu_fullsize.py is part of the selected session, so the CPU work
    overlaps the GPU tests that run before it."""
    sel = [it.nodeid for it in items if "test_gpu_fullsize" in it.nodeid]
    if not sel:
        return
    from oracle import pyoracle
    if not pyoracle.available("reference"):
        return  # the fixture reports it
    import tempfile

    import fullsize_ref
    d = tempfile.mkdtemp(prefix="nufft_fullsize_ref_")
    need = fullsize_ref.runs_for(sel)
    _FULLSIZE["runner"] = fullsize_ref.Runner(d, runs=need)


def pytest_sessionfinish(session, exitstatus):
    r = _FULLSIZE.pop("runner", None)
    if r is not None:
        r.close()


@pytest.fixture(scope="session")
def fullsize_ref_runs():
    r = _FULLSIZE.get("runner")
    if r is None:
        pytest.fail("oracle/_ref/libnufft_ref.so missing: the reference's own output is the full-size oracle")
    return r


@pytest.fixture(scope="session")
def port():
    from oracle import pyoracle
    if not pyoracle.available("port"):
        pyoracle.build()
    return pyoracle.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import pyoracle
    if not pyoracle.available("reference"):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return pyoracle.Oracle("reference")


@pytest.fixture(scope="session")
def nb():
    """The product library on a real GPU."""
    import paper_1701_04492_b200 as pkg
    if pkg.device_count() < 1:
        pytest.fail("no CUDA device visible — GPU tests must run on the B200 box")
    return pkg


def golden(name: str) -> dict:
    d = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return {k: d[k] for k in d.files}


def rel_l2(got, want, scale=None) -> float:
    got, want = np.asarray(got), np.asarray(want)
    s = np.linalg.norm(want if scale is None else scale)
    return float(np.linalg.norm(got - want) / s) if s > 0 else float(np.linalg.norm(got - want))


def rel_inf(got, want) -> float:
    got, want = np.asarray(got), np.asarray(want)
    m = np.max(np.abs(want))
    return float(np.max(np.abs(got - want)) / m) if m > 0 else float(np.max(np.abs(got - want)))
