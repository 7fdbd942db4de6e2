#!/usr/bin/env python3
"""Short type-II run for ncu (bench.py's workload: N = 2^24, eps 1e-14, the
GaussianSampler inputs): `warm` execs then `reps` execs on one stream.  Kernel
launches per exec: k2_pass1_tma, k2_pass2_fs.

  python scripts/profile_type2.py [warm] [reps] [type]    type: 2 (default) | 1 | 3 | 2d
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_04492_b200 as nb  # noqa: E402

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
kind = sys.argv[3] if len(sys.argv) > 3 else "2"
smp = nb.GaussianSampler(20240)
dev = torch.device("cuda", 0)
if kind == "2":
    n = 1 << 24
    p = nb.plan_nufft2(smp.uniform_vector(n, 0.0, 1.0), 1e-14, device=0)
elif kind == "1":
    import numpy as np
    n = 1 << 24
    p = nb.plan_nufft1(np.clip(np.arange(n) + smp.uniform_vector(n, -0.5, 0.5), 0, n), 1e-12, device=0)
elif kind == "3":
    n = 1 << 22
    p = nb.plan_nufft3(smp.uniform_vector(n, 0.0, 1.0), smp.uniform_vector(n, 0.0, float(n)), 1e-9, device=0)
else:
    n = 1 << 24
    p = nb.plan_nufft2d2(smp.uniform_vector(n, 0.0, 1.0), smp.uniform_vector(n, 0.0, 1.0), 4096, 4096, 1e-9, device=0)
c = torch.from_numpy(smp.complex_vector(n)).to(dev)
f = torch.empty(n, dtype=torch.complex128, device=dev)
for _ in range(warm + reps):
    p.execute_device(c.data_ptr(), f.data_ptr())
torch.cuda.synchronize()
print("done", kind, float(torch.linalg.norm(f).item()))
