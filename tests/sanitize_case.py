"""TEST HELPER: one small invocation of a fused kernel family, to be run under
compute-sanitizer by tests/test_gpu_sanitizer.py.  Sizes are the smallest at
which the sm_100a kernels in question are selected (the 4096-point two-level
FFT / TMA kernels need N1 or N2 = 4096); term ranges are cut to two terms so
the instrumented run stays short while every barrier/mbarrier/TMA hand-off
(group handoffs, unit boundaries, staging) still executes.

    python tests/sanitize_case.py type2|type2_2048|type1|type2d
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_04492_b200 as nb  # noqa: E402

case = sys.argv[1]
rng = nb.GaussianSampler(99)
dev = torch.device("cuda", 0)
if case in ("type2", "type2_2048"):
    n = 1 << (24 if case == "type2" else 22)
    p = nb.plan_nufft2(rng.uniform_vector(n, 0.0, 1.0), 1e-14, device=0)
    c = torch.from_numpy(rng.complex_vector(n)).to(dev)
    f = torch.empty_like(c)
    K = p.rank()
    p.execute_terms_device(c.data_ptr(), f.data_ptr(), K - 2, K)   # k2_pass1_tma + k2_pass2_fs (r0 > 0)
elif case == "type1":
    n = 1 << 24
    w = np.clip(np.arange(n) + rng.uniform_vector(n, -0.5, 0.5), 0.0, float(n))
    p = nb.plan_nufft1(w, 1e-2, device=0)                            # few terms: k1_passA_tm / k1_passB_tm
    c = torch.from_numpy(rng.complex_vector(n)).to(dev)
    f = torch.empty_like(c)
    p.execute_device(c.data_ptr(), f.data_ptr())
elif case == "type2d":
    m = 4096
    cnt = 1 << 20
    p = nb.plan_nufft2d2(rng.uniform_vector(cnt, 0.0, 1.0), rng.uniform_vector(cnt, 0.0, 1.0), m, m, 1e-1,
                         device=0)                                    # k2d_rows / k2d_cols at m = 4096
    C = torch.from_numpy(rng.complex_vector(m * m)).to(dev)
    f = torch.empty(cnt, dtype=torch.complex128, device=dev)
    p.execute_device(C.data_ptr(), f.data_ptr())
else:
    raise SystemExit(f"unknown case {case}")
torch.cuda.synchronize()
print("OK", case, float(torch.linalg.norm(f).item()))
