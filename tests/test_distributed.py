"""Multi-GPU path (the in-library r-split of
csrc/nufft2_multi.cu and paper_1701_04492_b200/parallel.py).

CPU (gloo, world size 2, no GPU): the term partition (nufft_multi_term_range,
host-only C-ABI) and the collective protocol of exec_multi — bucket-order
partials summed chunk by chunk, then one un-permute — with per-rank partials
computed from the ORACLE's factors (f_r = u_r .* gather_t(FFT(v_r .* c)),
transforms.hpp:152-161) and the plan's bucket order restated on the host.

GPU: a one-rank NCCL communicator through nufft_plan2_exec_multi (bit-identical
to the single-GPU exec), the bucket-order pieces against exec_terms, and two
gloo ranks that both run the product's partials on the one GPU and reduce
over CPU tensors (parallel.exec_rsplit_torch), compared with the full
transform.  (More than one NCCL rank needs more than one GPU; the driver's
8-GPU step runs bench.py --mode rsplit through the same library call.)"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_1701_04492_b200.parallel import batch_range, term_range


def test_term_ranges_cover_each_term_once():
    for K in (1, 16, 18, 20, 64):
        for world in (1, 2, 3, 4, 8, 24):
            seen = []
            for r in range(world):
                a, b = term_range(K, world, r)
                seen.extend(range(a, b))
            assert seen == list(range(K))
    # the reference's worker split of r-ranges (transforms.hpp:181-192) for K = 20 on 8
    assert [term_range(20, 8, r) for r in range(8)] == [(0, 2), (2, 5), (5, 7), (7, 10), (10, 12),
                                                         (12, 15), (15, 17), (17, 20)]
    for B in (1, 8, 9):
        got = []
        for r in range(4):
            a, b = batch_range(B, 4, r)
            got.extend(range(a, b))
        assert got == list(range(B))
    from paper_1701_04492_b200.api import InvalidArgument
    with pytest.raises(InvalidArgument):
        term_range(20, 2, 2)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bucket_order(t: np.ndarray, n: int):
    """The plan's bucket order (plan_kernels.cu build_buckets): key (t mod N1, t div N1),
    stable in j; N = N1 N2, N2 = 2^ceil(l/2).  Returns perm (sorted -> sample) and the
    row offsets."""
    l = n.bit_length() - 1
    log_n2 = (l + 1) // 2
    n1 = 1 << (l - log_n2)
    key = (t % n1) * (1 << log_n2) + (t // n1)
    perm = np.argsort(key, kind="stable")
    rows = np.searchsorted(key[perm] >> log_n2, np.arange(n1 + 1), side="left")
    return perm, rows, n1


def _cpu_worker(rank, world, port, n, eps, nchunks, q):
    import torch
    import torch.distributed as dist

    from oracle.pyoracle import Oracle
    from paper_1701_04492_b200.parallel import reduce_chunks_torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle("port")
    rng = o.sampler(77)
    x = rng.uniform_vector(n, 0.0, 1.0)
    c = rng.complex_vector(n)
    plan = o.plan2(x, eps)
    u, v = plan.factors()
    _, _, t = plan.samples()
    t = t.astype(np.int64)
    r0, r1 = term_range(plan.rank, world, rank)
    part = np.zeros(n, np.complex128)
    for r in range(r0, r1):
        part += u[r] * np.fft.fft(v[r] * c)[t]
    perm, rows, n1 = _bucket_order(t, n)
    fs = torch.from_numpy(part[perm].copy())             # bucket order
    off = [int(rows[n1 * qq // nchunks]) for qq in range(nchunks + 1)]
    reduce_chunks_torch(fs, off, dst=0)
    if rank == 0:
        f = np.empty(n, np.complex128)
        f[perm] = fs.numpy()                               # un-permute
        want = plan.execute(c)
        q.put(float(np.linalg.norm(f - want) / np.linalg.norm(want)))
    dist.barrier()
    dist.destroy_process_group()


def test_rsplit_chunked_reduce_protocol_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cpu_worker, args=(r, 2, port, 512, 1e-12, 4, q)) for r in range(2)]
    [p.start() for p in procs]
    [p.join(120) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    err = q.get(timeout=5)
    assert err <= 1e-13, err


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("n", [1 << 12, 1 << 16, 3000])
def test_exec_multi_single_rank_nccl_equals_exec(nb, n):
    import torch
    from paper_1701_04492_b200.parallel import NcclComm, unique_id
    rng = nb.GaussianSampler(n)
    x = rng.uniform_vector(n, 0.0, 1.0)
    p = nb.plan_nufft2(x, 1e-14, device=0)
    comm = NcclComm(unique_id(), 1, 0, 0)
    dev = torch.device("cuda", 0)
    c = torch.from_numpy(np.stack([rng.complex_vector(n) for _ in range(3)])).to(dev)
    want = torch.empty_like(c)
    p.execute_device(c.data_ptr(), want.data_ptr(), 3)
    for allreduce in (False, True):
        got = torch.full_like(c, float("nan"))
        p.execute_multi_device(c.data_ptr(), got.data_ptr(), comm, batch=3, allreduce=allreduce)
        torch.cuda.synchronize()
        assert torch.equal(torch.view_as_real(got), torch.view_as_real(want)), allreduce
    comm.close()


@pytest.mark.gpu
def test_sorted_partials_and_unpermute_match_exec_terms(nb):
    import torch
    n = 1 << 16
    rng = nb.GaussianSampler(5)
    p = nb.plan_nufft2(rng.uniform_vector(n, 0.0, 1.0), 1e-14, device=0)
    c = torch.from_numpy(rng.complex_vector(n)).cuda()
    K = p.rank()
    off = p.reduce_chunks(4)
    assert off[0] == 0 and off[-1] == n and np.all(np.diff(off) >= 0)
    for r0, r1 in [(0, K), (0, 7), (7, K), (3, 3)]:
        fs, f, want = torch.empty_like(c), torch.empty_like(c), torch.empty_like(c)
        p.execute_terms_sorted_device(c.data_ptr(), fs.data_ptr(), r0, r1)
        p.unpermute_device(fs.data_ptr(), f.data_ptr())
        p.execute_terms_device(c.data_ptr(), want.data_ptr(), r0, r1)
        torch.cuda.synchronize()
        assert torch.equal(torch.view_as_real(f), torch.view_as_real(want)), (r0, r1)


def _gpu_worker(rank, world, port, n, q):
    import torch
    import torch.distributed as dist

    import paper_1701_04492_b200 as nb
    from paper_1701_04492_b200.parallel import exec_rsplit_torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = nb.GaussianSampler(123)
    x = rng.uniform_vector(n, 0.0, 1.0)
    c = torch.from_numpy(rng.complex_vector(n)).cuda(0)
    p = nb.plan_nufft2(x, 1e-14, device=0)
    f = torch.zeros_like(c)
    exec_rsplit_torch(p, c, f, nchunks=4, dst=None)   # all-reduce: both ranks hold f
    want = torch.empty_like(c)
    p.execute_device(c.data_ptr(), want.data_ptr())
    torch.cuda.synchronize()
    q.put((rank, float((torch.linalg.norm(f - want) / torch.linalg.norm(want)).item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_rsplit_two_gloo_ranks_product_partials(nb):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, 1 << 18, q)) for r in range(2)]
    [p.start() for p in procs]
    [p.join(300) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    errs = dict(q.get(timeout=5) for _ in range(2))
    assert max(errs.values()) <= 1e-14, errs


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1 << 16, 1 << 22, 3000])
def test_type1_term_shards_and_single_rank_multi(nb, n):
    """Type-I r-split: term-range partials (transpose core, both passes) sum to the full
    transform, and exec_multi over a one-rank NCCL communicator equals exec."""
    import torch
    from paper_1701_04492_b200.parallel import NcclComm, unique_id
    rng = nb.GaussianSampler(n + 1)
    w = np.clip(np.arange(n) + rng.uniform_vector(n, -0.5, 0.5), 0.0, float(n))
    p = nb.plan_nufft1(w, 1e-12, device=0)
    c = torch.from_numpy(rng.complex_vector(n)).cuda()
    full = torch.empty_like(c)
    p.execute_device(c.data_ptr(), full.data_ptr())
    K = p.rank()
    acc = torch.zeros_like(c)
    for g in range(3):
        r0, r1 = term_range(K, 3, g)
        part = torch.empty_like(c)
        p.execute_terms_device(c.data_ptr(), part.data_ptr(), r0, r1)
        acc += part
    torch.cuda.synchronize()
    assert (torch.linalg.norm(acc - full) / torch.linalg.norm(full)).item() <= 1e-14
    comm = NcclComm(unique_id(), 1, 0, 0)
    got = torch.full_like(c, float("nan"))
    p.execute_multi_device(c.data_ptr(), got.data_ptr(), comm)
    torch.cuda.synchronize()
    assert torch.equal(torch.view_as_real(got), torch.view_as_real(full))
    comm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [4041, 4040])  # bTrivial; B made non-trivial below
def test_type3_term_shards_and_single_rank_multi(nb, seed):
    """Type-III outer-term split: partials over term ranges (inner transforms, beta dot
    products, the epilogue's partial Horner sum times (ih)^r0) add up to the full
    transform; exec_multi on a one-rank communicator equals exec."""
    import torch
    from paper_1701_04492_b200.parallel import NcclComm, unique_id
    n = 1 << 16
    rng = nb.GaussianSampler(seed)
    x = rng.uniform_vector(n, 0.0, 1.0)
    if seed == 4040:
        x[7] = 1.0 - 0.25 / n  # a sample on the node at 1: B non-trivial
    w = rng.uniform_vector(n, 0.0, float(n))
    p = nb.plan_nufft3(x, w, 1e-9, device=0)
    assert p.bTrivial == (seed == 4041)
    c = torch.from_numpy(rng.complex_vector(n)).cuda()
    full = torch.empty_like(c)
    p.execute_device(c.data_ptr(), full.data_ptr())
    K = p.rank_a
    acc = torch.zeros_like(c)
    for g in range(3):
        r0, r1 = term_range(K, 3, g)
        part = torch.empty_like(c)
        p.execute_terms_device(c.data_ptr(), part.data_ptr(), r0, r1)
        acc += part
    torch.cuda.synchronize()
    assert (torch.linalg.norm(acc - full) / torch.linalg.norm(full)).item() <= 1e-14
    comm = NcclComm(unique_id(), 1, 0, 0)
    got = torch.full_like(c, float("nan"))
    p.execute_multi_device(c.data_ptr(), got.data_ptr(), comm)
    torch.cuda.synchronize()
    assert torch.equal(torch.view_as_real(got), torch.view_as_real(full))
    comm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("m,n", [(4096, 64), (256, 512), (64, 16)])
def test_2d_r1_shards_and_single_rank_multi(nb, m, n):
    """2D r1 split (row-stage terms): partials over r1 ranges add up to the full transform
    (both column kernels: m = 4096 two-group, others single-group), exec_multi on a one-rank
    communicator equals exec."""
    import torch
    from paper_1701_04492_b200.parallel import NcclComm, unique_id
    cnt = 3 * m * n // 4 + 5
    rng = nb.GaussianSampler(m + n)
    p = nb.plan_nufft2d2(rng.uniform_vector(cnt, 0.0, 1.0), rng.uniform_vector(cnt, 0.0, 1.0), m, n, 1e-9, device=0)
    assert p.fused
    C = torch.from_numpy(rng.complex_vector(m * n)).cuda()
    full = torch.empty(cnt, dtype=torch.complex128, device="cuda")
    p.execute_device(C.data_ptr(), full.data_ptr())
    K = p.rank_x()
    acc = torch.zeros_like(full)
    for g in range(3):
        r0, r1 = term_range(K, 3, g)
        part = torch.empty_like(full)
        p.execute_terms_device(C.data_ptr(), part.data_ptr(), r0, r1)
        acc += part
    torch.cuda.synchronize()
    assert (torch.linalg.norm(acc - full) / torch.linalg.norm(full)).item() <= 1e-14
    comm = NcclComm(unique_id(), 1, 0, 0)
    got = torch.full_like(full, float("nan"))
    p.execute_multi_device(C.data_ptr(), got.data_ptr(), comm)
    torch.cuda.synchronize()
    assert torch.equal(torch.view_as_real(got), torch.view_as_real(full))
    comm.close()
