#!/usr/bin/env python3
"""A/B: type-II exec with pass 2 scattering f[perm] (current) vs pass 2 writing the
bucket-order partial + a gather un-permute kernel (f[j] = fs[invperm[j]]).
Same stream, CUDA events, N = 2^24, eps = 1e-14; prints ms per exec of each and of
the un-permute alone, and checks the two results are bit-identical."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_04492_b200 as nb  # noqa: E402

n = 1 << 24
smp = nb.GaussianSampler(20240)
p = nb.plan_nufft2(smp.uniform_vector(n, 0.0, 1.0), 1e-14, device=0)
c = torch.from_numpy(smp.complex_vector(n)).cuda()
f1, f2, fs = torch.empty_like(c), torch.empty_like(c), torch.empty_like(c)
st = torch.cuda.Stream()
sh = st.cuda_stream
K = p.rank()


def timeit(fn, reps=20, warm=3):
    with torch.cuda.stream(st):
        for _ in range(warm):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


a = timeit(lambda: p.execute_device(c.data_ptr(), f1.data_ptr(), 1, sh))
b = timeit(lambda: (p.execute_terms_sorted_device(c.data_ptr(), fs.data_ptr(), 0, K, sh),
                    p.unpermute_device(fs.data_ptr(), f2.data_ptr(), 1, sh)))
u = timeit(lambda: p.unpermute_device(fs.data_ptr(), f2.data_ptr(), 1, sh))
same = torch.equal(torch.view_as_real(f1), torch.view_as_real(f2))
print(f"scatter f[perm] in pass 2: {a:.3f} ms | bucket-order pass 2 + gather: {b:.3f} ms "
      f"(gather alone {u:.3f} ms) | bit-identical: {same}")
