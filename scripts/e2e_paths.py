#!/usr/bin/env python3
"""Where the host-API time goes for one 2^24 vector (bench.py's inputs): the C-ABI
call with pinned vs pageable (pre-touched) host buffers, and the cost of a fresh
256 MiB output allocation touched for the first time (what a std::vector result
costs the caller).  Median of 5 calls each."""
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_04492_b200 as nb  # noqa: E402

n = 1 << 24
smp = nb.GaussianSampler(20240)
p = nb.plan_nufft2(smp.uniform_vector(n, 0.0, 1.0), 1e-14, device=0)
c = smp.complex_vector(n)


def med(fn, k=5):
    fn()
    t = []
    for _ in range(k):
        t0 = time.perf_counter()
        fn()
        t.append(time.perf_counter() - t0)
    return statistics.median(t) * 1e3


f = np.ones(n, np.complex128)
pageable = med(lambda: p.execute_host_ptr(c.ctypes.data, f.ctypes.data, 1))
cp = torch.from_numpy(c).pin_memory()
fp = torch.empty_like(cp).pin_memory()
pinned = med(lambda: p.execute_host_ptr(cp.data_ptr(), fp.data_ptr(), 1))
alloc = med(lambda: np.zeros(n, np.complex128).fill(0))
print(f"exec_host batch 1: pageable {pageable:.1f} ms, pinned {pinned:.1f} ms; "
      f"fresh 256 MiB output zero-filled {alloc:.1f} ms")

# PCIe: one 256 MiB pinned copy each way, alone and both at once (two streams)
d = torch.empty(n, dtype=torch.complex128, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty_like(d)


def h2d():
    with torch.cuda.stream(s1):
        d.copy_(cp, non_blocking=True)
    s1.synchronize()


def d2h():
    with torch.cuda.stream(s2):
        fp.copy_(d2, non_blocking=True)
    s2.synchronize()


def both():
    with torch.cuda.stream(s1):
        d.copy_(cp, non_blocking=True)
    with torch.cuda.stream(s2):
        fp.copy_(d2, non_blocking=True)
    s1.synchronize()
    s2.synchronize()


gb = 16 * n / 1e9
th, td, tb = med(h2d), med(d2h), med(both)
print(f"PCIe pinned 256 MiB: H2D {th:.2f} ms ({gb / th * 1e3:.1f} GB/s), D2H {td:.2f} ms ({gb / td * 1e3:.1f} GB/s), "
      f"both concurrently {tb:.2f} ms ({2 * gb / tb * 1e3:.1f} GB/s aggregate)")
