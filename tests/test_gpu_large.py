"""Full-size (BASELINE.json) checks through size-independent properties:
exact direct sums at sampled outputs (no O(N^2) oracle needed), linearity,
bit-identical determinism, batch == repeated single executions, and r-term
partial sums adding up to the full transform (the multi-GPU sharding unit).

cfg2: NUFFT-II N = 2^24, eps = 1e-14, x iid U[0,1)  (K = 20)
cfg3: NUFFT-I  N = 2^24, eps = 1e-12, omega_k = clamp(k + d_k, 0, N)  (K = 18)
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N24 = 1 << 24


def _split(v, bits):
    """v = hi + lo with hi carrying `bits` fractional bits (exact)."""
    hi = np.round(v * 2.0 ** bits) / 2.0 ** bits
    return hi, v - hi


def direct_type2_at(x_j: float, c: np.ndarray) -> complex:
    """sum_k c_k exp(-2 pi i x_j k), k < N <= 2^24, phases reduced exactly."""
    n = len(c)
    k = np.arange(n, dtype=np.int64)
    m = int(round(x_j * 2 ** 29))
    lo = x_j - m / 2 ** 29
    frac_hi = ((m * k) & ((1 << 29) - 1)).astype(np.float64) / 2 ** 29
    phase = frac_hi + lo * k.astype(np.float64)
    return complex(np.sum(c * np.exp(-2j * np.pi * phase)))


def direct_type1_at(j: int, omega: np.ndarray, c: np.ndarray) -> complex:
    """sum_k c_k exp(-2 pi i (j/N) omega_k), phases reduced exactly."""
    n = len(c)
    kint = np.floor(omega).astype(np.int64)
    d = omega - kint
    dh, dl = _split(d, 26)
    t1 = ((j * kint) % n).astype(np.float64) / n
    t2 = np.modf(j * dh / n)[0]
    phase = t1 + t2 + j * dl / n
    return complex(np.sum(c * np.exp(-2j * np.pi * phase)))


@pytest.fixture(scope="module")
def cfg2():
    rng = np.random.default_rng(20240)
    x = rng.random(N24)
    c = rng.standard_normal(N24) + 1j * rng.standard_normal(N24)
    return x, c


def test_cfg2_direct_sum_spot_check(nb, cfg2):
    x, c = cfg2
    p = nb.plan_nufft2(x, 1e-14)
    assert p.rank() == 20 and p.fused
    f = nb.exec_nufft2(p, c)
    rms = np.sqrt(np.mean(np.abs(f) ** 2))
    idx = np.random.default_rng(3).choice(N24, 8, replace=False)
    for j in idx:
        err = abs(f[j] - direct_type2_at(float(x[j]), c))
        assert err <= 1e-14 * rms, (j, err, rms)


def test_cfg2_properties(nb, cfg2):
    import torch
    x, c = cfg2
    p = nb.plan_nufft2(x, 1e-14)
    dev = torch.device("cuda", p.device)
    c_d = torch.from_numpy(c).to(dev)
    f1, f2 = torch.empty_like(c_d), torch.empty_like(c_d)
    p.execute_device(c_d.data_ptr(), f1.data_ptr())
    p.execute_device(c_d.data_ptr(), f2.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(torch.view_as_real(f1), torch.view_as_real(f2))  # bit-identical
    # linearity: T(a c + b c') = a T(c) + b T(c')
    c2 = torch.roll(c_d, 12345)
    a, b = 0.75 - 0.5j, -1.25 + 2.0j
    mix = a * c_d + b * c2
    g, g2 = torch.empty_like(c_d), torch.empty_like(c_d)
    p.execute_device(mix.data_ptr(), g.data_ptr())
    p.execute_device(c2.data_ptr(), g2.data_ptr())
    torch.cuda.synchronize()
    lin = a * f1 + b * g2
    assert (torch.linalg.norm(g - lin) / torch.linalg.norm(lin)).item() <= 1e-14
    # r-term shards sum to the full transform
    K = p.rank()
    acc = torch.zeros_like(c_d)
    for r0 in range(0, K, 6):
        part = torch.empty_like(c_d)
        p.execute_terms_device(c_d.data_ptr(), part.data_ptr(), r0, min(K, r0 + 6))
        acc += part
    torch.cuda.synchronize()
    assert (torch.linalg.norm(acc - f1) / torch.linalg.norm(f1)).item() <= 1e-14


def test_cfg2_batch8_equals_singles(nb):
    import torch
    rng = np.random.default_rng(8)
    n = 1 << 22
    x = rng.random(n)
    p = nb.plan_nufft2(x, 1e-14)
    dev = torch.device("cuda", p.device)
    cs = torch.randn(8, n, dtype=torch.complex128, device=dev)
    fb = torch.empty_like(cs)
    p.execute_device(cs.data_ptr(), fb.data_ptr(), batch=8)
    for b in (0, 5, 7):
        fs = torch.empty_like(cs[b])
        p.execute_device(cs[b].data_ptr(), fs.data_ptr())
        torch.cuda.synchronize()
        assert torch.equal(torch.view_as_real(fs), torch.view_as_real(fb[b]))


def test_cfg3_direct_sum_spot_check(nb):
    rng = np.random.default_rng(33)
    d = rng.uniform(-0.5, 0.5, N24)
    w = np.clip(np.arange(N24) + d, 0.0, float(N24))
    c = rng.standard_normal(N24) + 1j * rng.standard_normal(N24)
    p = nb.plan_nufft1(w, 1e-12)
    assert p.rank() == 18
    f = nb.exec_nufft1(p, c)
    rms = np.sqrt(np.mean(np.abs(f) ** 2))
    for j in np.random.default_rng(4).choice(N24, 6, replace=False):
        err = abs(f[j] - direct_type1_at(int(j), w, c))
        assert err <= 1e-12 * rms, (j, err, rms)


def test_cfg2_adjoint_identity(nb, cfg2):
    """<A c, g> == <c, A^H g> at full size (the fused transpose core against the
    fused type-II passes), and the adjoint is bit-reproducible."""
    x, c = cfg2
    p = nb.plan_nufft2(x, 1e-14)
    g = np.random.default_rng(5).standard_normal(N24) + 1j * np.random.default_rng(6).standard_normal(N24)
    f = nb.exec_nufft2(p, c)
    a1 = nb.exec_nufft2_adjoint(p, g)
    a2 = nb.exec_nufft2_adjoint(p, g)
    assert np.array_equal(a1.view(np.float64), a2.view(np.float64))
    lhs = np.vdot(g, f)          # <A c, g> = g^H A c
    rhs = np.vdot(a1, c)         # <c, A^H g> = (A^H g)^H c
    scale = np.linalg.norm(g) * np.linalg.norm(f)
    assert abs(lhs - rhs) <= 1e-13 * scale, (lhs, rhs)


def _exact_frac_phase(x: float, k: np.ndarray) -> np.ndarray:
    """frac(x * k) for integer k < 2^24 with the product reduced exactly."""
    m = int(round(x * 2 ** 29))
    lo = x - m / 2 ** 29
    return ((m * k) & ((1 << 29) - 1)).astype(np.float64) / 2 ** 29 + lo * k.astype(np.float64)


def test_cfg5_direct_sum_spot_check(nb):
    """2D 4096 x 4096 -> 2^24 samples, eps 1e-14 (cfg5) against exact direct sums."""
    m = n = 4096
    cnt = 1 << 24
    rng = np.random.default_rng(55)
    x, y = rng.random(cnt), rng.random(cnt)
    C2 = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
    p = nb.plan_nufft2d2(x, y, m, n, 1e-14)
    assert p.fused
    f = nb.exec_nufft2d2(p, C2)
    rms = np.sqrt(np.mean(np.abs(f) ** 2))
    kx = np.arange(n, dtype=np.int64)
    ky = np.arange(m, dtype=np.int64)
    for j in np.random.default_rng(9).choice(cnt, 4, replace=False):
        ex = np.exp(-2j * np.pi * _exact_frac_phase(float(x[j]), kx))
        ey = np.exp(-2j * np.pi * _exact_frac_phase(float(y[j]), ky))
        want = complex(ey @ (C2 @ ex))
        assert abs(f[j] - want) <= 1e-13 * rms, (j, abs(f[j] - want), rms)


def test_cfg2_error_sweep_vs_gpu_direct(nb, cfg2):
    """4096 outputs of the N = 2^24 transform against the GPU direct sum
    (oracle.hpp:70-86 on the device): the eps = 1e-14 contract holds at scale."""
    x, c = cfg2
    p = nb.plan_nufft2(x, 1e-14)
    f = nb.exec_nufft2(p, c)
    idx = np.sort(np.random.default_rng(12).choice(N24, 4096, replace=False))
    want = nb.nudft_direct(x[idx], np.arange(N24, dtype=np.float64), c)
    rel = np.linalg.norm(f[idx] - want) / np.linalg.norm(want)
    assert rel <= 1e-14, rel


def test_cfg3_error_sweep_vs_gpu_direct(nb):
    """Type I at 2^24: f_j = sum_k c_k exp(-2 pi i (j/N) w_k) for 2048 outputs."""
    rng = np.random.default_rng(33)
    d = rng.uniform(-0.5, 0.5, N24)
    w = np.clip(np.arange(N24) + d, 0.0, float(N24))
    c = rng.standard_normal(N24) + 1j * rng.standard_normal(N24)
    f = nb.exec_nufft1(nb.plan_nufft1(w, 1e-14), c)
    idx = np.sort(np.random.default_rng(13).choice(N24, 2048, replace=False))
    want = nb.nudft_direct(idx / N24, w, c)
    rel = np.linalg.norm(f[idx] - want) / np.linalg.norm(want)
    assert rel <= 1e-14, rel


def test_cfg3_type1_adjoint_identity(nb):
    """Type-I adjoint at full size runs the fused-sample pass 2 on the type-I plan
    (delta and key from the frequencies, k2_pass2_fs<., DSRC>): check it against
    the transpose core through <A1 c, g> == <c, A1^H g>, and bit-reproducibility."""
    rng = np.random.default_rng(31)
    w = np.clip(np.arange(N24) + rng.uniform(-0.5, 0.5, N24), 0, N24)
    c = rng.standard_normal(N24) + 1j * rng.standard_normal(N24)
    g = rng.standard_normal(N24) + 1j * rng.standard_normal(N24)
    p = nb.plan_nufft1(w, 1e-12)
    f = nb.exec_nufft1(p, c)
    a1 = nb.exec_nufft1_adjoint(p, g)
    a2 = nb.exec_nufft1_adjoint(p, g)
    assert np.array_equal(a1.view(np.float64), a2.view(np.float64))
    lhs = np.vdot(g, f)
    rhs = np.vdot(a1, c)
    scale = np.linalg.norm(g) * np.linalg.norm(f)
    assert abs(lhs - rhs) <= 1e-13 * scale, (lhs, rhs)
