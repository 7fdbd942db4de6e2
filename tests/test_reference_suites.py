"""The reference's own test suites, compiled unmodified (oracle/Makefile):

* CPU: unit_<suite> = reference headers + FFTW-API shim + minigtest.  All
  pass, and the acceptance binary reproduces proj/test_output.txt (10/12 with
  the same two red cells) — the oracle build is pinned by the reference's own
  known answers and tolerances.
* GPU: conf_<suite> = the same sources against the drop-in headers in
  include/nufft linked to libnufft_b200.so — the conformance suite; conf_cli
  runs the reference's CLI tests against the B200 CLI binary.
"""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
SUITES = ["fft", "special", "lowrank", "oracle", "transforms", "transform2d", "inverse"]


def _bin(name):
    path = os.path.join(REF, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (oracle/Makefile needs /root/reference at build time)")
    return path


@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_suite_on_oracle_build(suite):
    r = subprocess.run([_bin(f"unit_{suite}")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " 0 failed" in r.stdout


def test_reference_acceptance_reproduces_recorded_output():
    """proj/test_output.txt: 10/12 criteria, red cells [1] (N=16) and [3] (10.3 eps).

    Criterion [11] is a wall-clock measurement (cost slope and exec/FFT ratio); on a
    loaded host it can miss its window, so it is retried once and is the only line
    allowed to differ from the recorded output."""
    for attempt in range(2):
        r = subprocess.run([_bin("acceptance")], capture_output=True, text=True, timeout=600)
        out = r.stdout + r.stderr
        if "10/12 criteria passed" in out:
            break
    timing_only = "9/12 criteria passed" in out and "[11] FAIL" in out
    assert "10/12 criteria passed" in out or timing_only, out[-2000:]
    assert "[ 1] FAIL" in out and "[ 3] FAIL" in out
    assert "max residual 2.260e-15 = 10.3*eps" in out
    assert "medians 1 -> 11 -> 21 -> 115" in out
    for k in (2, 4, 5, 6, 7, 8, 9, 10, 12):
        assert f"[{k:2d}] PASS" in out


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES + ["cli"])
def test_reference_unit_suite_on_b200_dropin(nb, suite):
    """conf_cli is the reference CLI's own test (proj/tests/cli_test.cpp: CSV round
    trips, exit codes 0/1/2/3, transform/verify/bench/cgstudy end to end) against
    the drop-in csv/oracle/random headers and the B200 CLI (tools/nufft_cli.cpp)."""
    r = subprocess.run([_bin(f"conf_{suite}")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]


@pytest.mark.gpu
def test_cpp_dropin_example(nb):
    exe = os.path.join(ROOT, "paper_1701_04492_b200", "_build", "example_dropin")
    assert os.path.exists(exe), "build() compiles tests/cpp/example_dropin.cpp"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    # (NCCL may print its version banner first when NCCL_DEBUG is set)
    last = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else ""
    assert r.returncode == 0 and last.startswith("OK"), r.stdout + r.stderr
