"""compute-sanitizer over the hand-written sm_100a kernels: memcheck,
racecheck (shared-memory hazards) and synccheck (barrier misuse) on one small
invocation of each fused kernel family (tests/sanitize_case.py).  These kernels
hand state between warp groups through named barriers, mbarriers, TMA bulk
copies and tensor memory, so a missing barrier shows up here first."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = "/usr/local/cuda/bin/compute-sanitizer"
KERNELS = "regex:k2_pass|k1_pass|k2d_|k_unpermute"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("case", ["type2", "type2_2048", "type1", "type2d"])
def test_sanitizer_clean(nb, tool, case):
    if not os.path.exists(SAN):
        pytest.fail("compute-sanitizer missing from the CUDA toolkit")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "17", "--kernel-name", KERNELS,
           "--print-limit", "20"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "hazard"]
    cmd += [sys.executable, os.path.join(ROOT, "tests", "sanitize_case.py"), case]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "OK " + case in out, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-4000:]
