"""GPU parity of the inverse NUFFT (inverse.hpp) against
the CPU oracle (whose inverse equals the reference bit for bit,
tests/test_oracle.py::test_inverse_port_bit_identical_to_reference).

Tolerances: the Toeplitz first column / spectrum / matvec are single
transforms (max(eps, 4e-15) relative, as test_gpu_parity.check); CG amplifies
rounding differences by the condition number, so solutions are compared to
1e-10 relative and iteration counts to within one step, with the reference's
own round-trip contracts (inverse_test.cpp:234-248, 292-303) on top.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _x(port, n, gamma):
    return port.worst_grid(n, gamma)


@pytest.mark.parametrize("n,gamma", [(16, 0.3), (100, 0.2), (256, 0.125), (1024, 0.25), (4096, 0.4)])
def test_toeplitz_normal_vs_oracle(nb, port, n, gamma):
    x = _x(port, n, gamma)
    pg, po = nb.plan_nufft2(x, 2.2e-16), port.plan2(x, 2.2e-16)
    tg, to = nb.toeplitz_from_normal(pg), port.toeplitz_from_normal(po)
    assert rel_l2(tg.firstColumn, to.firstColumn) <= 4e-15
    sg, so = tg.spectrum, to.spectrum
    assert np.all(sg.imag == 0.0)
    assert np.max(np.abs(sg - so)) <= 1e-13 * np.max(np.abs(so))
    v = port.sampler(3 + n).complex_vector(n)
    assert rel_l2(nb.toeplitz_matvec(tg, v), to.matvec(v)) <= 1e-13


@pytest.mark.parametrize("n,gamma", [(64, 0.125), (256, 0.125), (1000, 0.2), (4096, 0.3)])
def test_inufft2_vs_oracle(nb, port, n, gamma):
    x = _x(port, n, gamma)
    pg, po = nb.plan_nufft2(x, 2.2e-16), port.plan2(x, 2.2e-16)
    c_true = port.sampler(10 + n).complex_vector(n)
    f = po.execute(c_true)
    rg, ro = nb.inufft2(pg, f, 1e-12), port.inufft2(po, f, 1e-12)
    assert rg["converged"] and ro["converged"]
    assert abs(rg["iterations"] - ro["iterations"]) <= 1
    assert len(rg["residualHistory"]) == rg["iterations"]
    assert rel_l2(rg["solution"], ro["solution"]) <= 1e-10
    assert rel_l2(rg["solution"], c_true) <= 1e-10                     # inverse_test.cpp:244
    assert rel_l2(nb.exec_nufft2(pg, rg["solution"]), f) <= 1e-11     # :247


@pytest.mark.parametrize("n,shift", [(32, 0.0), (128, 0.1), (1024, 0.25), (4096, 0.3)])
def test_inufft1_vs_oracle(nb, port, n, shift):
    rng = port.sampler(20 + n)
    w = np.clip(np.arange(n) + (rng.uniform_vector(n, -shift, shift) if shift else 0.0), 0.0, float(n))
    pg, po = nb.plan_nufft1(w, 2.2e-16), port.plan1(w, 2.2e-16)
    c_true = rng.complex_vector(n)
    assert rel_l2(nb.exec_nufft1_adjoint(pg, c_true), po.adjoint(c_true)) <= 4e-15
    f = po.execute(c_true)
    rg, ro = nb.inufft1(pg, f, 1e-12), port.inufft1(po, f, 1e-12)
    assert rg["converged"] and abs(rg["iterations"] - ro["iterations"]) <= 1
    assert rel_l2(rg["solution"], ro["solution"]) <= 1e-9
    assert rel_l2(rg["solution"], c_true) <= 1e-9                      # inverse_test.cpp:302
    if shift == 0.0:
        assert rg["iterations"] == 1                                    # :278-290


def test_inverse_edge_cases(nb, port):
    p = nb.plan_nufft2(port.worst_grid(32, 0.1), 2.2e-16)
    r = nb.inufft2(p, np.zeros(32, np.complex128), 1e-12)               # :264-270
    assert r["converged"] and r["iterations"] == 0 and not np.any(r["solution"])
    with pytest.raises(nb.DomainError):                                 # :272-276
        nb.inufft2(nb.plan_nufft2(port.worst_grid(16, 0.5), 2.2e-16), np.ones(16, np.complex128), 1e-12)
    with pytest.raises(nb.InvalidArgument):
        nb.inufft2(p, np.ones(31, np.complex128), 1e-12)
    op = nb.toeplitz_from_first_column(np.ones(4, np.complex128))
    with pytest.raises(nb.InvalidArgument):                             # :167-170
        nb.toeplitz_matvec(op, np.ones(3, np.complex128))
    with pytest.raises(nb.DomainError):
        nb.cg_solve_toeplitz(op, np.ones(4, np.complex128), 0.0, 10)
    col = np.array([2.0, 1.0, 0.5], np.complex128)                      # :138-147
    got = nb.toeplitz_matvec(nb.toeplitz_from_first_column(col), np.array([1.0, 0.0, -1.0], np.complex128))
    assert np.max(np.abs(got - np.array([1.5, 0.0, -1.5]))) <= 1e-13


def test_cg_residual_history_matches_oracle(nb, port):
    """cg_solve with the Toeplitz operator: same stopping behaviour, non-increasing
    residuals (inverse_test.cpp:218-232)."""
    n = 256
    x = port.worst_grid(n, 1.0 / 8)
    tg = nb.toeplitz_from_normal(nb.plan_nufft2(x, 2.2e-16))
    to = port.toeplitz_from_normal(port.plan2(x, 2.2e-16))
    rhs = port.sampler(9).complex_vector(n)
    rg, ro = nb.cg_solve_toeplitz(tg, rhs, 1e-13, 400), port.cg_toeplitz(to, rhs, 1e-13, 400)
    assert rg["converged"] and abs(rg["iterations"] - ro["iterations"]) <= 1
    h = rg["residualHistory"]
    assert np.all(h[1:] <= h[:-1] + 1e-14)
    k = min(len(h), len(ro["residualHistory"])) - 1
    assert np.allclose(h[:k], ro["residualHistory"][:k], rtol=1e-6, atol=0)


@pytest.mark.slow
def test_inufft2_large_round_trip(nb):
    """N = 2^20 (fused transforms, 2N = 2^21 Toeplitz FFTs): the solve recovers c."""
    n = 1 << 20
    rng = np.random.default_rng(21)
    x = (np.arange(n) + rng.uniform(-0.25, 0.25, n)) / n % 1.0
    p = nb.plan_nufft2(x, 1e-14)
    c = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    f = nb.exec_nufft2(p, c)
    r = nb.inufft2(p, f, 1e-11)
    assert r["converged"] and r["iterations"] < nb.default_cg_max_iter(n)
    assert rel_l2(r["solution"], c) <= 1e-9
