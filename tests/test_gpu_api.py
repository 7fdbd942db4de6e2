"""GPU semantics of the drop-in API: FFT conventions and known answers
(fft_test.cpp), error types, the FFT-count test hook,
bit-identical determinism, concurrent executions of one plan, batching and
r-term partial sums (the multi-GPU sharding unit)."""
from __future__ import annotations

import threading

import numpy as np
import pytest

from conftest import golden, rel_l2

pytestmark = pytest.mark.gpu


def test_fft_known_answers(nb):
    f = nb.fft_forward([1, 0, 0, 0])
    assert np.max(np.abs(f - 1)) <= 1e-15
    f = nb.fft_forward(np.ones(4))
    assert abs(f[0] - 4) <= 1e-14 and np.max(np.abs(f[1:])) <= 1e-14
    g = nb.fft_inverse([4, 0, 0, 0])
    assert np.max(np.abs(g - 1)) <= 1e-15


def test_fft_golden_and_numpy(nb, port):
    g = golden("fft_sizes")
    for n in (1, 5, 7, 12, 33, 100, 256):
        assert rel_l2(nb.fft_forward(g[f"in_{n}"]), g[f"fwd_{n}"]) <= 1e-14
        assert rel_l2(nb.fft_inverse(g[f"in_{n}"]), g[f"inv_{n}"]) <= 1e-14
    for n in (2, 8, 16, 64, 1000, 2048, 3000, 4096, 5000, 8192, 12288, 1 << 16, 1 << 20, 3 * 5 * 7 * 11 * 13):
        v = port.sampler(n).complex_vector(n)
        want = np.fft.fft(v)
        assert rel_l2(nb.fft_forward(v), want) <= 1e-13, n
        assert rel_l2(nb.fft_inverse(v), np.fft.ifft(v)) <= 1e-13, n


def test_fft_2d_and_columns(nb, port):
    for m, n in ((4, 6), (32, 64), (3, 5), (128, 4096)):
        a = port.sampler(m * n).complex_vector(m * n).reshape(m, n)
        assert rel_l2(nb.fft_2d_forward(a), np.fft.fft2(a)) <= 1e-13
        assert rel_l2(nb.fft_cols_forward(a), np.fft.fft(a, axis=0)) <= 1e-13
        assert rel_l2(nb.fft_rows_forward(a), np.fft.fft(a, axis=1)) <= 1e-13


def test_errors_match_reference_types(nb):
    with pytest.raises(nb.InvalidArgument):
        nb.plan_nufft2([], 1e-12)
    with pytest.raises(nb.DomainError):
        nb.plan_nufft2([0.5], 0.0)
    with pytest.raises(nb.DomainError):
        nb.plan_nufft2([0.5], 1.0)
    with pytest.raises(nb.InvalidArgument):
        nb.plan_nufft2([0.5, np.nan], 1e-12)
    with pytest.raises(nb.InvalidArgument):
        nb.normalize_samples([np.inf])
    p = nb.plan_nufft2(np.arange(8) / 8, 2.2e-16)
    with pytest.raises(nb.InvalidArgument):
        nb.exec_nufft2(p, np.zeros(7, complex))
    with pytest.raises(nb.InvalidArgument):
        nb.plan_nufft1([-0.5], 2.2e-16)
    nb.plan_nufft1([0.5], 2.2e-16)
    with pytest.raises(nb.InvalidArgument):
        nb.plan_nufft3([0.1, 0.2], [0.0], 2.2e-16)
    with pytest.raises(nb.InvalidArgument):
        nb.plan_nufft3([0.1], [1.0], 2.2e-16)
    with pytest.raises(nb.InvalidArgument):
        nb.plan_nufft3([0.1], [-0.2], 2.2e-16)
    with pytest.raises(nb.InvalidArgument):
        nb.fft_forward([])
    with pytest.raises(nb.InvalidArgument):
        nb.fft_inverse([])
    with pytest.raises(nb.DomainError):
        nb.select_rank(0.7, 2.2e-16)
    with pytest.raises(nb.InvalidArgument):
        nb.cheb_coefficients(0.0, 4)
    with pytest.raises(nb.DomainError):
        nb.cheb_eval_matrix([1.0 + 1e-11], 3)
    nb.cheb_eval_matrix([1.0 + 5e-13], 3)
    pd = nb.plan_nufft2d2([0.1, 0.4], [0.2, 0.8], 3, 4, 2.2e-16)
    with pytest.raises(nb.InvalidArgument):
        nb.exec_nufft2d2(pd, np.zeros((4, 3), complex))
    with pytest.raises(nb.InvalidArgument):
        nb.plan_nufft2d2([0.1], [0.2], 0, 4, 2.2e-16)


def test_grid_and_normalize_known_answers(nb):
    s, t, _ = nb.grid_assign([0.029, 0.044, 0.055, 0.425, 0.575, 0.638, 0.788, 0.944], 8)
    assert list(s) == [0, 0, 0, 3, 5, 5, 6, 8] and list(t) == [0, 0, 0, 3, 5, 5, 6, 0]
    s, t, g = nb.grid_assign([0.99], 8)
    assert s[0] == 8 and t[0] == 0
    s, t, g = nb.grid_assign(np.arange(16) / 16, 16)
    assert list(s) == list(range(16)) and g == 0.0
    v = nb.normalize_samples([0.25, 0.75, 1.25, -0.25, -3.1, -1e-20])
    assert list(v[:4]) == [0.25, 0.75, 0.25, 0.75]
    assert abs(v[4] - 0.9) <= 1e-15 and 0.0 <= v[5] < 1.0
    g2 = nb.plan_nufft2d2([2 / 5, 0.99], [3 / 5, 0.5], 5, 5, 2.2e-16).grid()
    assert list(g2["sx"]) == [2, 5] and list(g2["tx"]) == [2, 0] and list(g2["sy"]) == [3, 3]


def test_rank_rules(nb):
    assert nb.plan_nufft2(np.arange(32) / 32, 2.2e-16).rank() == 1
    wg = (np.array([(j + 0.5) if j <= 16 else (j - 0.5) for j in range(32)]) / 32) % 1.0
    assert nb.plan_nufft2(wg, 2.2e-16).rank() == 16
    assert nb.plan_nufft1(np.arange(16.0), 2.2e-16).rank() == 1
    p = nb.plan_nufft1(np.arange(16.0) + 0.3, 2.2e-16)
    assert abs(p.gamma() - 0.3) <= 1e-12 and p.rank() == 16
    f = nb.exec_nufft2(nb.plan_nufft2([0.37], 2.2e-16), [2 - 1j])
    assert abs(f[0] - (2 - 1j)) <= 1e-13


def test_fft_exec_counts(nb):
    n = 96
    p = nb.plan_nufft2(np.arange(n) / n, 2.2e-16)
    nb.fft_reset_exec_counts()
    nb.exec_nufft2(p, np.ones(n, complex))
    assert nb.fft_exec_count(n) == 1
    x = np.random.default_rng(1).random(64)
    p = nb.plan_nufft2(x, 1e-12)
    nb.fft_reset_exec_counts()
    nb.exec_nufft2(p, np.ones(64, complex))
    assert nb.fft_exec_count(64) == p.rank()
    # 2D cost model (transform2d_test.cpp:230-244)
    rng = np.random.default_rng(14)
    pd = nb.plan_nufft2d2(rng.random(32), rng.random(32), 4, 8, 2.2e-16)
    nb.fft_reset_exec_counts()
    nb.exec_nufft2d2(pd, np.ones((4, 8), complex))
    assert nb.fft_exec_count(8) == pd.rank_x() * 4
    assert nb.fft_exec_count(4) == pd.rank_x() * pd.rank_y() * 8


def test_determinism_and_concurrency(nb, port):
    n = 1 << 12
    rng = port.sampler(71)
    x = rng.uniform_vector(n, 0.0, 1.0)
    c1, c2 = rng.complex_vector(n), rng.complex_vector(n)
    p = nb.plan_nufft2(x, 1e-14)
    w1, w2 = nb.exec_nufft2(p, c1), nb.exec_nufft2(p, c2)
    assert nb.exec_nufft2(p, c1).tobytes() == w1.tobytes()
    assert nb.exec_nufft2(p, c1, 3).tobytes() == w1.tobytes()
    got = {}

    def run(k, c):
        for _ in range(5):
            got.setdefault(k, []).append(nb.exec_nufft2(p, c))

    ts = [threading.Thread(target=run, args=(1, c1)), threading.Thread(target=run, args=(2, c2))]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert all(g.tobytes() == w1.tobytes() for g in got[1])
    assert all(g.tobytes() == w2.tobytes() for g in got[2])
    # 2D row-stage reuse is bit-identical (transform2d_test.cpp:215-227)
    rng2 = np.random.default_rng(12)
    pd = nb.plan_nufft2d2(rng2.random(40), rng2.random(40), 6, 5, 2.2e-16)
    C2 = rng2.standard_normal((6, 5)) + 1j * rng2.standard_normal((6, 5))
    assert nb.exec_nufft2d2_impl(pd, C2, True).tobytes() == nb.exec_nufft2d2_impl(pd, C2, False).tobytes()


def test_batch_and_term_ranges(nb, port):
    import torch
    n = 1 << 14
    rng = port.sampler(5)
    x = rng.uniform_vector(n, 0.0, 1.0)
    cs = np.stack([rng.complex_vector(n) for _ in range(3)])
    p = nb.plan_nufft2(x, 1e-14)
    single = np.stack([nb.exec_nufft2(p, c) for c in cs])
    assert nb.exec_nufft2(p, cs).tobytes() == single.tobytes()
    dev = torch.device("cuda", p.device)
    c_d = torch.from_numpy(cs[0]).to(dev)
    full = torch.empty_like(c_d)
    p.execute_device(c_d.data_ptr(), full.data_ptr())
    parts = []
    K = p.rank()
    for r0, r1 in ((0, 7), (7, 13), (13, K)):
        out = torch.empty_like(c_d)
        p.execute_terms_device(c_d.data_ptr(), out.data_ptr(), r0, r1)
        parts.append(out)
    torch.cuda.synchronize()
    total = (parts[0] + parts[1] + parts[2]).cpu().numpy()
    assert rel_l2(total, full.cpu().numpy()) <= 1e-14
    assert rel_l2(full.cpu().numpy(), single[0]) == 0.0


def test_batched_exec_equals_singles_all_types(nb):
    """batch > 1 through the device entry points of type I, adjoint-free type III
    and 2D: bit-identical to single executions (fused and generic shapes)."""
    import torch
    rng = np.random.default_rng(77)
    dev = torch.device("cuda", 0)
    for n in (1 << 12, 1000):
        w = np.clip(np.arange(n) + rng.uniform(-0.4, 0.4, n), 0, n)
        p1 = nb.plan_nufft1(w, 1e-12)
        x = rng.random(n)
        p3 = nb.plan_nufft3(x, rng.uniform(0, n, n), 1e-9)
        for p in (p1, p3):
            cs = torch.randn(3, n, dtype=torch.complex128, device=dev)
            fb = torch.empty_like(cs)
            p.execute_device(cs.data_ptr(), fb.data_ptr(), 3)
            for b in range(3):
                fs = torch.empty_like(cs[b])
                p.execute_device(cs[b].data_ptr(), fs.data_ptr(), 1)
                torch.cuda.synchronize()
                assert torch.equal(torch.view_as_real(fs), torch.view_as_real(fb[b]))
    m, nn, cnt = 64, 128, 5000
    pd = nb.plan_nufft2d2(rng.random(cnt), rng.random(cnt), m, nn, 1e-12)
    Cs = torch.randn(2, m, nn, dtype=torch.complex128, device=dev)
    fb = torch.empty(2, cnt, dtype=torch.complex128, device=dev)
    pd.execute_device(Cs.data_ptr(), fb.data_ptr(), 2)
    for b in range(2):
        fs = torch.empty(cnt, dtype=torch.complex128, device=dev)
        pd.execute_device(Cs[b].data_ptr(), fs.data_ptr(), 1)
        torch.cuda.synchronize()
        assert torch.equal(torch.view_as_real(fs), torch.view_as_real(fb[b]))


def test_stacked_passA_equals_singles(nb):
    """N = 2^21 (row FFT 2048, 1024 rows): batch > 1 runs pass A of the transpose core as
    ONE stacked launch per four vectors (transpose_fused.cu, the path type III uses for its
    inner transforms); a batch of 5 (groups of 4 + 1) must be bit-identical to five single
    executions, which take the unstacked launches."""
    import torch
    n = 1 << 21
    rng = np.random.default_rng(2121)
    w = np.clip(np.arange(n) + rng.uniform(-0.45, 0.45, n), 0, n)
    p1 = nb.plan_nufft1(w, 1e-9)
    dev = torch.device("cuda", 0)
    cs = torch.randn(5, n, dtype=torch.complex128, device=dev)
    fb = torch.empty_like(cs)
    p1.execute_device(cs.data_ptr(), fb.data_ptr(), 5)
    for b in range(5):
        fs = torch.empty_like(cs[b])
        p1.execute_device(cs[b].data_ptr(), fs.data_ptr(), 1)
        torch.cuda.synchronize()
        assert torch.equal(torch.view_as_real(fs), torch.view_as_real(fb[b])), b

@pytest.mark.parametrize("logn", [14, 24])
def test_type2_host_batch_pipelined_equals_singles(nb, logn):
    """exec_host with batch > 1 streams the vectors through two device slots on three
    streams (H2D / transform / D2H overlapped): results must be bit-identical to
    one host call per vector, including the slot reuse from the third vector on."""
    n = 1 << logn
    rng = np.random.default_rng(41 + logn)
    p = nb.plan_nufft2(rng.random(n), 1e-14)
    batch = 5 if logn < 20 else 3
    c = (rng.standard_normal((batch, n)) + 1j * rng.standard_normal((batch, n))).astype(np.complex128)
    f = np.empty_like(c)
    p.execute_host_ptr(c.ctypes.data, f.ctypes.data, batch)
    for b in range(batch):
        fb = np.empty(n, dtype=np.complex128)
        p.execute_host_ptr(c[b].ctypes.data, fb.ctypes.data, 1)
        assert np.array_equal(f[b].view(np.float64), fb.view(np.float64)), b
