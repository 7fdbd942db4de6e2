#!/usr/bin/env python3
"""One exec each of cfg3 (type I 2^24, 1e-12), the type-II adjoint (2^24, 1e-14) and cfg5 (2D
4096^2, 1e-9), after one warm-up each — for an ncu launch list (per-kernel device times)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_04492_b200 as nb  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 24
smp = nb.GaussianSampler(7)
c = torch.from_numpy(smp.complex_vector(n)).to(dev)
f = torch.empty_like(c)
w = np.clip(np.arange(n) + smp.uniform_vector(n, -0.5, 0.5), 0, n)
p1 = nb.plan_nufft1(w, 1e-12, device=0)
for _ in range(2):
    p1.execute_device(c.data_ptr(), f.data_ptr())
p2 = nb.plan_nufft2(smp.uniform_vector(n, 0.0, 1.0), 1e-14, device=0)
for _ in range(2):
    nb.api._check(nb.lib().nufft_plan2_adjoint(p2._h, c.data_ptr(), f.data_ptr(), None))
pd = nb.plan_nufft2d2(smp.uniform_vector(n, 0.0, 1.0), smp.uniform_vector(n, 0.0, 1.0), 4096, 4096, 1e-9, device=0)
for _ in range(2):
    pd.execute_device(c.data_ptr(), f.data_ptr())
torch.cuda.synchronize()
print("done")
