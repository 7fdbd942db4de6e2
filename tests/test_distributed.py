"""Multi-process (world_size 2, gloo, CPU) coverage of the multi-GPU host path:
term/batch partitioning and the partial-f reduce of r-term sharding.  The
per-rank partial sums are computed here from the ORACLE's factors
(f_r = u_r .* gather_t(FFT(v_r .* c)), transforms.hpp:152-161) so the
plumbing is checked end to end on CPU; on the B200 box the same
`parallel.exec_rsplit` is driven by nufft_plan2_exec_terms over NCCL
(bench.py --mode rsplit)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_1701_04492_b200.parallel import batch_range, term_range


def test_term_ranges_cover_each_term_once():
    for K in (1, 16, 18, 20, 64):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                a, b = term_range(K, world, r)
                seen.extend(range(a, b))
            assert seen == list(range(K))
    assert [term_range(20, 8, r) for r in range(8)] == [(0, 2), (2, 5), (5, 7), (7, 10), (10, 12),
                                                         (12, 15), (15, 17), (17, 20)]
    for B in (1, 8, 9):
        got = []
        for r in range(4):
            a, b = batch_range(B, 4, r)
            got.extend(range(a, b))
        assert got == list(range(B))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, eps, q):
    import torch
    import torch.distributed as dist

    from oracle.pyoracle import Oracle
    from paper_1701_04492_b200.parallel import exec_rsplit

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

    def partial(r0, r1):
        f = np.zeros(n, np.complex128)
        for r in range(r0, r1):
            f += u[r] * np.fft.fft(v[r] * c)[t]
        return torch.from_numpy(f)

    out = exec_rsplit(partial, plan.rank)
    if rank == 0:
        want = plan.execute(c)
        q.put(float(np.linalg.norm(out.numpy() - want) / np.linalg.norm(want)))
    dist.barrier()
    dist.destroy_process_group()


def test_rsplit_reduce_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 512, 1e-12, q)) for r in range(2)]
    [p.start() for p in procs]
    [p.join(120) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    err = q.get(timeout=5)
    assert err <= 1e-13, err
