"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs, against the golden fixtures, and against the direct
O(N^2) sums.

Tolerances (written per the north star, tied to epsilon):
  rel_l2 = ||f_gpu - f_ref||_2 / ||f_ref||_2           <= eps
  rel_inf = max|f_gpu - f_ref| / max|f_ref|            <= 10 eps
and the reference's own contracts against the direct sums:
  type II  ||f - f_direct|| <= N eps ||c||   (transforms_test.cpp:151-181)
  type III ||f - f_direct|| <= 4 N eps ||c|| (transforms_test.cpp:385-398)
  2D       ||f - f_direct|| <= 4 m n eps ||C||_F (transform2d_test.cpp:143-163)
Both sides compute the same rank-K sum, so observed differences are at the
rounding level (~1e-15), far inside these bounds.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, rel_inf, rel_l2

pytestmark = pytest.mark.gpu


def check(got, want, eps):
    """eps-tied tolerance; floored at 4e-15 because two correct fp64
    implementations of the same rank-K sum differ by rounding (~1e-15) even
    when eps itself is at machine precision (2.2e-16)."""
    tol = max(eps, 4e-15)
    assert rel_l2(got, want) <= tol, rel_l2(got, want)
    assert rel_inf(got, want) <= 10 * tol, rel_inf(got, want)


# ------------------------------------------------------------------ golden fixtures
def test_cfg1_golden(nb):
    g = golden("cfg1_type2")
    p = nb.plan_nufft2(g["x"], float(g["eps"]))
    assert p.rank() == int(g["rank"]) == 18 and p.gamma() == float(g["gamma"])
    f = nb.exec_nufft2(p, g["c"])
    check(f, g["f"], 1e-12)
    n = len(g["x"])
    assert rel_l2(f, g["f_direct"], g["c"]) <= n * 1e-12


def test_type2_golden_iid_and_worst(nb):
    g = golden("type2_iid_4096")
    p = nb.plan_nufft2(g["x"], 1e-14)
    assert p.rank() == 20 and p.fused
    check(nb.exec_nufft2(p, g["c"]), g["f"], 1e-14)
    _, s, t = p.samples()
    assert np.array_equal(s, g["s"]) and np.array_equal(t.astype(np.int64), g["t"])
    check(nb.exec_nufft2_adjoint(p, g["c"]), g["adj"], 1e-14)
    g = golden("type2_worst_64")
    p = nb.plan_nufft2(g["x"], 2.2e-16)
    assert p.rank() == 16
    f = nb.exec_nufft2(p, g["c"])
    check(f, g["f"], 1e-14)
    assert rel_l2(f, g["f_direct"], g["c"]) <= 64 * 2.2e-16
    u, v = p.factors()
    assert np.max(np.abs(u - g["u"])) <= 1e-14 and np.max(np.abs(v - g["v"])) <= 1e-14


def test_type1_golden(nb):
    g = golden("type1_jitter")
    p = nb.plan_nufft1(g["omega"], 1e-12)
    assert p.rank() == int(g["rank"])
    check(nb.exec_nufft1(p, g["c"]), g["f"], 1e-12)


@pytest.mark.parametrize("name", ["type3_a", "type3_b", "type3_c"])
def test_type3_golden(nb, name):
    g = golden(name)
    p = nb.plan_nufft3(g["x"], g["omega"], 1e-9)
    assert p.bTrivial == bool(g["btrivial"])
    assert p.effective_rank() == int(g["effective"]) and p.rank_a == int(g["rank_a"])
    f = nb.exec_nufft3(p, g["c"])
    check(f, g["f"], 1e-9)
    assert rel_l2(f, g["f_direct"], g["c"]) <= 4 * len(g["x"]) * 1e-9


def test_type2d_golden(nb):
    g = golden("type2d")
    p = nb.plan_nufft2d2(g["x"], g["y"], int(g["m"]), int(g["n"]), 1e-9)
    assert (p.rank_x(), p.rank_y()) == (int(g["rank_x"]), int(g["rank_y"]))
    assert np.array_equal(p.grid()["flatIndex"].astype(np.int64), g["flat"])
    f = nb.exec_nufft2d2(p, g["C"])
    check(f, g["f"], 1e-9)
    m, n = int(g["m"]), int(g["n"])
    assert np.linalg.norm(f - g["f_direct"]) <= 4 * m * n * 1e-9 * np.linalg.norm(g["C"])


# ------------------------------------------------------------------ live oracle, seeded
@pytest.mark.parametrize("n,eps", [
    (1, 1e-12), (7, 1e-12), (16, 2.2e-16), (37, 1e-14), (100, 1e-9), (255, 1e-12),
    (256, 1e-14), (1000, 1e-12), (1024, 1e-12), (4096, 1e-14), (8192, 1e-14),
    (1 << 14, 1e-12), (1 << 16, 1e-14), (3 * 4096, 1e-12),
])
def test_type2_vs_oracle(nb, port, n, eps):
    rng = port.sampler(1000 + n)
    x = rng.uniform_vector(n, 0.0, 1.0)
    c = rng.complex_vector(n)
    po, pg = port.plan2(x, eps), nb.plan_nufft2(x, eps)
    assert pg.rank() == po.rank and pg.gamma() == po.gamma
    check(nb.exec_nufft2(pg, c), po.execute(c), eps)


@pytest.mark.parametrize("n", [256, 4096, 1 << 16])
def test_type2_jittered_cfg1_shape(nb, port, n):
    rng = port.sampler(7 + n)
    d = rng.uniform_vector(n, -0.5, 0.5)
    x = ((np.arange(n) + d) / n) % 1.0
    c = rng.complex_vector(n)
    po, pg = port.plan2(x, 1e-12), nb.plan_nufft2(x, 1e-12)
    assert pg.rank() == po.rank == 18
    check(nb.exec_nufft2(pg, c), po.execute(c), 1e-12)


def test_type2_uniform_is_fft(nb, port):
    for n in (64, 96, 4096, 1 << 15):
        x = np.arange(n) / n
        c = port.sampler(n).complex_vector(n)
        p = nb.plan_nufft2(x, 2.2e-16)
        assert p.rank() == 1
        want = np.fft.fft(c)
        assert rel_l2(nb.exec_nufft2(p, c), want) <= 1e-14


def test_type2_clustered_rows_overflow(nb, port):
    """All samples in a few grid bins: rows far above the per-CTA capacity."""
    n = 1 << 14
    rng = port.sampler(99)
    x = (rng.uniform_vector(n, 0.0, 1.0) * 4 / n + 0.5) % 1.0   # ~4 bins
    c = rng.complex_vector(n)
    po, pg = port.plan2(x, 1e-12), nb.plan_nufft2(x, 1e-12)
    check(nb.exec_nufft2(pg, c), po.execute(c), 1e-12)


@pytest.mark.parametrize("n,eps", [(16, 2.2e-16), (33, 1e-12), (1024, 1e-12), (4096, 1e-12), (1 << 14, 1e-12)])
def test_type1_vs_oracle(nb, port, n, eps):
    rng = port.sampler(300 + n)
    d = rng.uniform_vector(n, -0.5, 0.5)
    w = np.clip(np.arange(n) + d, 0.0, float(n))
    c = rng.complex_vector(n)
    po, pg = port.plan1(w, eps), nb.plan_nufft1(w, eps)
    assert pg.rank() == po.rank
    check(nb.exec_nufft1(pg, c), po.execute(c), eps)
    # iid frequencies (collisions in bins)
    w = rng.uniform_vector(n, 0.0, float(n))
    po, pg = port.plan1(w, eps), nb.plan_nufft1(w, eps)
    check(nb.exec_nufft1(pg, c), po.execute(c), eps)


def test_type1_clustered_rows_overflow(nb, port):
    """Frequencies packed into a few bins: fused pass-A rows far above the
    per-CTA sample capacity (chunked accumulation) and long duplicate-bin runs."""
    n = 1 << 14
    rng = port.sampler(77)
    w = 100.0 + rng.uniform_vector(n, 0.0, 6.0)
    c = rng.complex_vector(n)
    po, pg = port.plan1(w, 1e-12), nb.plan_nufft1(w, 1e-12)
    check(nb.exec_nufft1(pg, c), po.execute(c), 1e-12)


@pytest.mark.parametrize("n", [1 << 16, 1 << 17])
def test_type1_fused_sizes_vs_oracle(nb, port, n):
    """N1 < N2 and N1 == N2 splits of the fused transpose core."""
    rng = port.sampler(400 + n)
    w = rng.uniform_vector(n, 0.0, float(n))
    c = rng.complex_vector(n)
    po, pg = port.plan1(w, 1e-14), nb.plan_nufft1(w, 1e-14)
    assert pg.fused
    check(nb.exec_nufft1(pg, c), po.execute(c), 1e-14)


@pytest.mark.parametrize("n", [16, 48, 256, 1024])
def test_type3_vs_oracle(nb, port, n):
    for seed in range(3):
        rng = port.sampler(50 + 7 * seed + n)
        x = rng.uniform_vector(n, 0.0, 1.0)
        w = rng.uniform_vector(n, 0.0, float(n))
        c = rng.complex_vector(n)
        po, pg = port.plan3(x, w, 1e-9), nb.plan_nufft3(x, w, 1e-9)
        bt, ka, ke, _ = po.info3()
        assert (pg.bTrivial, pg.rank_a, pg.effective_rank()) == (bt, ka, ke)
        check(nb.exec_nufft3(pg, c), po.execute(c), 1e-9)


@pytest.mark.parametrize("m,n,cnt", [(4, 3, 10), (8, 8, 64), (7, 6, 48), (64, 64, 4096), (32, 128, 3000)])
def test_type2d_vs_oracle(nb, port, m, n, cnt):
    rng = port.sampler(60 + m * n)
    x = rng.uniform_vector(cnt, 0.0, 1.0)
    y = rng.uniform_vector(cnt, 0.0, 1.0)
    C2 = rng.complex_vector(m * n).reshape(m, n)
    po, pg = port.plan2d2(x, y, m, n, 1e-9), nb.plan_nufft2d2(x, y, m, n, 1e-9)
    assert (pg.rank_x(), pg.rank_y()) == po.info2d()[:2]
    check(nb.exec_nufft2d2(pg, C2), po.execute(C2), 1e-9)


@pytest.mark.parametrize("m,n,cnt", [(16, 16, 300), (256, 128, 20000), (128, 512, 40000), (4096, 16, 30000)])
def test_type2d_fused_vs_oracle(nb, port, m, n, cnt):
    """Power-of-two grids take the fused row/column kernels (m = 4096: the column
    kernel's two-level FFT with X gathered from its in-place slots)."""
    rng = port.sampler(900 + m + n)
    x = rng.uniform_vector(cnt, 0.0, 1.0)
    y = rng.uniform_vector(cnt, 0.0, 1.0)
    C2 = rng.complex_vector(m * n).reshape(m, n)
    po, pg = port.plan2d2(x, y, m, n, 1e-12), nb.plan_nufft2d2(x, y, m, n, 1e-12)
    assert pg.fused
    check(nb.exec_nufft2d2(pg, C2), po.execute(C2), 1e-12)
    check(nb.exec_nufft2d2_impl(pg, C2, False), po.execute(C2), 1e-12)


def test_type2d_fused_clustered_and_uniform_axes(nb, port):
    """Columns far above the per-CTA capacity (chunked), and on-grid axes
    (u = v = 1 on that axis)."""
    m, n = 64, 32
    rng = port.sampler(4242)
    cnt = 1500
    x = (0.25 + rng.uniform_vector(cnt, 0.0, 1.0) * 2.0 / n) % 1.0     # ~2 columns
    y = rng.uniform_vector(cnt, 0.0, 1.0)
    C2 = rng.complex_vector(m * n).reshape(m, n)
    for xx, yy in ((x, y), (np.arange(cnt) % n / n, y), (x, np.arange(cnt) % m / m)):
        po, pg = port.plan2d2(xx, yy, m, n, 1e-12), nb.plan_nufft2d2(xx, yy, m, n, 1e-12)
        assert (pg.rank_x(), pg.rank_y()) == po.info2d()[:2]
        check(nb.exec_nufft2d2(pg, C2), po.execute(C2), 1e-12)


def test_adjoint_vs_oracle(nb, port):
    for n in (8, 16, 32, 128, 1000, 4096, 1 << 15):
        rng = port.sampler(30 + n)
        x = rng.uniform_vector(n, 0.0, 1.0)
        f = rng.complex_vector(n)
        check(nb.exec_nufft2_adjoint(nb.plan_nufft2(x, 2.2e-16), f),
              port.plan2(x, 2.2e-16).adjoint(f), 1e-13)


def test_factor_mirrors_vs_oracle(nb, port):
    rng = port.sampler(42)
    x = rng.uniform_vector(300, 0.0, 1.0)
    uo, vo = port.plan2(x, 1e-12).factors()
    ug, vg = nb.plan_nufft2(x, 1e-12).factors()
    assert np.max(np.abs(ug - uo)) <= 1e-14 and np.max(np.abs(vg - vo)) <= 1e-14
    d = rng.uniform_vector(50, -0.25, 0.25)
    ko, uo, vo = port.build_factors(d, 0.25, np.arange(20) / 20, 1e-9)
    kg, ug, vg = nb.build_factors(d, 0.25, np.arange(20) / 20, 1e-9)
    assert ko == kg and np.max(np.abs(ug - uo)) <= 1e-14 and np.max(np.abs(vg - vo)) <= 1e-14


# ------------------------------------------------------------------ GPU direct sums (oracle.hpp:70-107)
def test_gpu_nudft_direct_vs_oracle(nb, port):
    """The device direct sum (exact phase split, Neumaier, ascending k) against
    the oracle's long-double-phase direct sum."""
    for n in (1, 17, 1024, 3000):
        rng = port.sampler(700 + n)
        x = rng.uniform_vector(n, 0.0, 1.0)
        w = rng.uniform_vector(n, 0.0, float(n))
        c = rng.complex_vector(n)
        assert rel_l2(nb.nudft_direct(x, w, c), port.nudft_direct(x, w, c)) <= 1e-15
    m, nn, cnt = 24, 40, 300
    rng = port.sampler(800)
    x, y = rng.uniform_vector(cnt, 0.0, 1.0), rng.uniform_vector(cnt, 0.0, 1.0)
    C2 = rng.complex_vector(m * nn).reshape(m, nn)
    assert rel_l2(nb.nudft2d_direct(x, y, C2), port.nudft2d_direct(x, y, C2)) <= 1e-15


def test_type2_large_vs_gpu_direct_sum(nb):
    """Exact-error sweep at N = 2^18 the CPU oracle cannot reach in seconds:
    every output of the fused type-II transform against the GPU direct sum,
    within the reference's contract ||f - f_direct|| <= N eps ||c|| (with eps-level
    actual agreement)."""
    n = 1 << 18
    rng = np.random.default_rng(18)
    x = rng.random(n)
    c = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    for eps in (1e-14, 1e-9):
        f = nb.exec_nufft2(nb.plan_nufft2(x, eps), c)
        want = nb.nudft_direct(x, np.arange(n, dtype=np.float64), c)
        err = np.linalg.norm(f - want)
        assert err <= n * eps * np.linalg.norm(c)
        assert err / np.linalg.norm(want) <= 10 * eps


# ------------------------------------------------------------------ every fused shape
@pytest.mark.parametrize("log_n", list(range(4, 23)))
def test_pow2_sweep_type2_type1_adjoint_vs_gpu_direct(nb, log_n):
    """Every power-of-two size selects a different kernel shape (N1 x N2 split,
    single-pass N1 = 1, small/warp-specialized/two-group pass 2, one- or
    two-worker pass 1 and transpose passes).  Each is checked against exact
    direct sums on up to 512 outputs; eps = 1e-12 (K = 18) and ragged
    (duplicate-bin, clustered-row) samples."""
    n = 1 << log_n
    rng = np.random.default_rng(1000 + log_n)
    x = rng.random(n)
    x[: n // 8] = (0.3 + rng.random(n // 8) * 4.0 / n) % 1.0   # crowded rows / duplicate bins
    c = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    idx = np.sort(rng.choice(n, min(n, 512), replace=False))
    k = np.arange(n, dtype=np.float64)
    p = nb.plan_nufft2(x, 1e-12)
    assert p.fused
    f = nb.exec_nufft2(p, c)
    want = nb.nudft_direct(x[idx], k, c)
    assert rel_l2(f[idx], want) <= 1e-12
    # adjoint: (A^H g)_k = sum_j g_j exp(+2 pi i x_j k)
    g = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    a = nb.exec_nufft2_adjoint(p, g)
    want_a = np.conj(nb.nudft_direct(idx.astype(np.float64), x, np.conj(g)))
    assert rel_l2(a[idx], want_a) <= 1e-12
    # type I on jittered frequencies: f_j = sum_k c_k exp(-2 pi i (j/N) w_k)
    w = np.clip(k + rng.uniform(-0.5, 0.5, n), 0.0, float(n))
    f1 = nb.exec_nufft1(nb.plan_nufft1(w, 1e-12), c)
    want1 = nb.nudft_direct(idx / n, w, c)
    assert rel_l2(f1[idx], want1) <= 1e-12


@pytest.mark.parametrize("m,n", [(16, 4096), (4096, 16), (64, 1024), (1024, 64), (512, 512), (2048, 256)])
def test_2d_fused_shapes_vs_gpu_direct(nb, m, n):
    rng = np.random.default_rng(m * 7 + n)
    cnt = m * n
    x, y = rng.random(cnt), rng.random(cnt)
    C2 = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
    p = nb.plan_nufft2d2(x, y, m, n, 1e-12)
    assert p.fused
    f = nb.exec_nufft2d2(p, C2)
    idx = np.sort(rng.choice(cnt, 256, replace=False))
    want = nb.nudft2d_direct(x[idx], y[idx], C2)
    assert rel_l2(f[idx], want) <= 1e-12
