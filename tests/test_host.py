"""Host-side logic of the product library, no GPU needed:

* the C-ABI library loads and exports every symbol include/nufft_b200.h declares;
* the plan-time scalar math (rank rule, Bessel-product coefficients, Lambert-W,
  Bessel J) is bit-identical to the oracle (hence to the reference);
* the truncated Bessel series the kernels evaluate meets its error budget;
* without a CUDA device, compute calls fail loudly (no CPU fallback).
"""
from __future__ import annotations

import math
import os
import re
import subprocess

import numpy as np
import pytest
import scipy.special as sp

import paper_1701_04492_b200 as nb
from paper_1701_04492_b200._lib import LIB_PATH

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "nufft_b200.h")).read()
    return sorted(set(re.findall(r"\b(nufft_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    nm = subprocess.run(["nm", "-D", "--defined-only", LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (nufft_[a-z0-9_]+)$", nm, re.M))
    declared = set(header_symbols())
    assert declared, "no declarations parsed"
    assert declared <= exported, declared - exported
    # and the Python binding binds all of them
    assert declared <= set(nb.exported_symbols()), declared - set(nb.exported_symbols())


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_scalars_bit_identical_to_oracle(port):
    for gamma in (0.0, 1 / 40, 1 / 32, 0.05, 0.1, 0.25, 0.3, 0.4, 0.4999, 0.5):
        for eps in (2.2e-16, 3.3e-16, 1e-14, 1e-12, 1e-9, 1.2e-7, 1e-5, 9.8e-4, 1e-2, 0.3):
            assert nb.select_rank(gamma, eps) == port.select_rank(gamma, eps), (gamma, eps)
    for gamma in (1 / 32, 0.3, 0.5):
        for K in (1, 6, 24):
            a = nb.cheb_coefficients(gamma, K)
            b = port.cheb_coefficients(gamma, K)
            assert a.tobytes() == b.tobytes()
    for x in (0.0, 1e-3, 0.5, 3.0, 1e3, 1e8):
        assert nb.lambert_w(x) == port.lambert_w(x)
    for order in (0, 1, 5, 20):
        for z in (-2.0, -0.7, 0.0, 0.3, 1.9):
            assert nb.bessel_j_int(order, z) == port.bessel_j_int(order, z)
    assert nb.bessel_j_signed(-3, 0.4) == -nb.bessel_j_int(3, 0.4)


def test_host_errors_have_reference_types():
    with pytest.raises(nb.DomainError):
        nb.select_rank(0.1, 0.0)
    with pytest.raises(nb.DomainError):
        nb.select_rank(0.7, 1e-12)
    with pytest.raises(nb.DomainError):
        nb.lambert_w(-1.0)
    with pytest.raises(nb.DomainError):
        nb.bessel_j_int(2, 3.0)
    with pytest.raises(nb.InvalidArgument):
        nb.cheb_coefficients(0.6, 4)


def test_bessel_series_truncation_budget():
    """The Horner degree chosen per r (bessel_series_degrees) keeps the
    truncated tail of 2 |h|^r g_r below 2^-62 — checked here in extended
    precision against scipy's J_r over |delta| <= gamma."""
    coef = np.zeros((64, 16))
    for r in range(64):
        for m in range(16):
            coef[r, m] = (-1) ** m / (math.factorial(m) * math.factorial(m + r))
    for gamma in (0.5, 0.3, 1 / 32):
        K = nb.select_rank(gamma, 1e-14)
        d = np.linspace(-gamma, gamma, 101)
        h = -np.pi * d / 2
        for r in range(K):
            full = 2 * h ** r * np.polyval(coef[r, ::-1], h * h)
            exact = 2 * sp.jv(r, -np.pi * d)
            assert np.max(np.abs(full - exact)) <= 1e-15  # a few ulp of |2 J_r| <= 2


def test_compute_fails_loudly_without_gpu():
    if nb.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(nb.NufftError):
        nb.plan_nufft2([0.1, 0.2], 1e-12)
    with pytest.raises(nb.NufftError):
        nb.fft_forward([1, 2, 3])


def test_sampler_bit_identical_to_reference_sampler(port):
    """nufft_sampler_* / include/nufft/random.hpp draw the reference's
    GaussianSampler streams (random.hpp:14-60) bit for bit — bench.py's two
    arms and the full-size parity tests rely on it.  Host-only, no GPU."""
    from oracle import pyoracle
    o = pyoracle.Oracle("reference") if pyoracle.available("reference") else port
    for seed in (0, 1, 20240, 2 ** 63 + 5):
        a, b = nb.GaussianSampler(seed), o.sampler(seed)
        assert np.array_equal(a.uniform_vector(1001, -0.5, 0.5), b.uniform_vector(1001, -0.5, 0.5))
        assert np.array_equal(a.complex_vector(777), b.complex_vector(777))  # odd count: spare carried
        assert a() == b.normal()
        assert np.array_equal(a.uniform_vector(5, 0.0, 4096.0), b.uniform_vector(5, 0.0, 4096.0))


def test_bench_fp64_roofline_block_from_committed_profile():
    """bench.py's roofline.fp64 reads profiles/fp64.json (the committed ncu capture)."""
    import json
    import sys
    sys.path.insert(0, ROOT)
    import bench
    fp = json.load(open(os.path.join(ROOT, "profiles", "fp64.json")))
    out = bench.fp64_roofline(fp, fp["n"], fp["K"], {"k2_pass1": 1.65, "k2_pass2": 2.19})
    assert out and set(out["per_kernel"]) == {"k2_pass1", "k2_pass2"}
    for v in out["per_kernel"].values():
        assert 0.1 < v["frac_of_fp64_peak"] < 1.0
    assert bench.fp64_roofline(fp, 1 << 22, fp["K"], {"k2_pass1": 1.0}) is None
    assert bench.fp64_roofline(None, 1, 1, {}) is None
