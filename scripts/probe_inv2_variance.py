"""inverse NUFFT-II (N = 2^22) solve time, repeated in one process: alone, and after the big
type-I / type-III plans of the config sweep have come and gone (pool trimmed in between)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_04492_b200 as nb

torch.cuda.set_device(0)
stream = torch.cuda.Stream(); sh = stream.cuda_stream
rng = np.random.default_rng(76)
n = 1 << 22
x = ((np.arange(n) + rng.uniform(-0.25, 0.25, n)) / n) % 1.0
p = nb.plan_nufft2(x, 1e-14)
op = nb.toeplitz_from_normal(p)
c = rng.standard_normal(n) + 1j * rng.standard_normal(n)
f = nb.exec_nufft2(p, c)
fd = torch.from_numpy(f).to("cuda"); sd = torch.empty_like(fd)

def solves(tag, k=5):
    ts = []
    for _ in range(k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = nb.inufft2_device(p, fd.data_ptr(), 1e-10, sd.data_ptr(), op, sh)
        e1.record(stream); torch.cuda.synchronize()
        ts.append(round(e0.elapsed_time(e1), 2))
    print(tag, ts, r["iterations"], flush=True)

solves("alone")
big = 1 << 24
w = np.clip(np.arange(big) + rng.uniform(-0.5, 0.5, big), 0, big)
p1 = nb.plan_nufft1(w, 1e-12)
cc = torch.randn(big, dtype=torch.complex128, device="cuda"); ff = torch.empty_like(cc)
for _ in range(3): p1.execute_device(cc.data_ptr(), ff.data_ptr(), 1, sh)
torch.cuda.synchronize()
solves("with a 2^24 type-I plan alive")
del p1, cc, ff; torch.cuda.empty_cache()
solves("after destroying it (pool trimmed)")
solves("again")
