"""Design probe: where the inverse NUFFT's time goes (matvec, CG, host API)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1701_04492_b200 as nb
n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
rng = np.random.default_rng(76)
x = ((np.arange(n) + rng.uniform(-0.25, 0.25, n)) / n) % 1.0
p = nb.plan_nufft2(x, 1e-14)
op = nb.toeplitz_from_normal(p)
v = torch.randn(n, dtype=torch.complex128, device="cuda"); o = torch.empty_like(v)
for _ in range(3): op.matvec_device(v.data_ptr(), o.data_ptr())
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10): op.matvec_device(v.data_ptr(), o.data_ptr())
torch.cuda.synchronize(); print("matvec ms", (time.perf_counter() - t0) / 10 * 1e3)
c = rng.standard_normal(n) + 1j * rng.standard_normal(n)
f = nb.exec_nufft2(p, c)
for tol in (1e-3, 1e-10):
    t0 = time.perf_counter(); r = nb.inufft2(p, f, tol, op); dt = time.perf_counter() - t0
    print("inufft2 tol", tol, "iters", r["iterations"], "ms", dt * 1e3, "ms/iter", dt * 1e3 / max(1, r["iterations"]))
rhs = nb.exec_nufft2_adjoint(p, f)
t0 = time.perf_counter(); r = nb.cg_solve_toeplitz(op, rhs, 1e-10, 400); dt = time.perf_counter() - t0
print("cg only iters", r["iterations"], "ms", dt * 1e3)
t0 = time.perf_counter(); a = nb.exec_nufft2_adjoint(p, f); print("adjoint host ms", (time.perf_counter() - t0) * 1e3)
