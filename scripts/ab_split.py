#!/usr/bin/env python3
"""A/B of two library builds (NUFFT_B200_LIB) on N = 2^22 transforms: prints ms per exec
of type II (eps 1e-14), type I (1e-12), type III (cfg4, 1e-9) and saves the outputs so a
second run can compare them.  Usage: ab_split.py TAG OUTDIR"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_04492_b200 as nb  # noqa: E402

tag, outdir = sys.argv[1], sys.argv[2]
n = 1 << 22
dev = torch.device("cuda", 0)
st = torch.cuda.Stream()


def timeit(fn, reps=10, warm=2):
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


smp = nb.GaussianSampler(4040)
x = smp.uniform_vector(n, 0.0, 1.0)
w = smp.uniform_vector(n, 0.0, float(n))
c = torch.from_numpy(smp.complex_vector(n)).to(dev)
f = torch.empty_like(c)
res = {}
p2 = nb.plan_nufft2(x, 1e-14, device=0)
res["II"] = timeit(lambda: p2.execute_device(c.data_ptr(), f.data_ptr(), 1, st.cuda_stream))
np.save(os.path.join(outdir, f"{tag}_II.npy"), f.cpu().numpy())
wj = np.clip(np.arange(n) + smp.uniform_vector(n, -0.5, 0.5), 0, n)
p1 = nb.plan_nufft1(wj, 1e-12, device=0)
res["I"] = timeit(lambda: p1.execute_device(c.data_ptr(), f.data_ptr(), 1, st.cuda_stream))
np.save(os.path.join(outdir, f"{tag}_I.npy"), f.cpu().numpy())
p3 = nb.plan_nufft3(x, w, 1e-9, device=0)
res["III"] = timeit(lambda: p3.execute_device(c.data_ptr(), f.data_ptr(), 1, st.cuda_stream), reps=3, warm=1)
np.save(os.path.join(outdir, f"{tag}_III.npy"), f.cpu().numpy())
print(tag, " ".join(f"{k}: {v:.3f} ms" for k, v in res.items()), "lib", nb.LIB_PATH)
if tag == "B":
    for k in ("II", "I", "III"):
        a, b = np.load(os.path.join(outdir, f"A_{k}.npy")), np.load(os.path.join(outdir, f"B_{k}.npy"))
        print(k, "rel diff A vs B", np.linalg.norm(a - b) / np.linalg.norm(a))
