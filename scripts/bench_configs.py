#!/usr/bin/env python3
"""Per-configuration timing of every transform on the path.

  python scripts/bench_configs.py [--steps K] [--warmup W] [--only cfg2,cfg3,...] [--out FILE]

Times the device-pointer exec (inputs resident in HBM, plan built outside the
timed region) with CUDA events on the launching stream, W warm-ups then K
timed execs, and reports points/s, algorithmic bytes (the §8(d) formulas) and
the HBM roofline fraction against MEASURED_PEAKS.json.  Also times the cuFFT
comparison the reference's `bench` subcommand reports (fft_seconds_baseline:
K batched Z2Z FFTs of size N, here through torch.fft = cuFFT) and the
exec/FFT ratio (proj/tools/nufft_app.hpp:289-315 columns).  One JSON line per
config; these are parity configurations, not bench.py's headline line.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


_CLOCKS = {}


def timeit(fn, steps, warmup, stream):
    """CUDA-event ms per call; nvidia-smi clocks sampled over the timed loop (bench.py's
    ClockSampler) are kept for the record emitted next."""
    import torch

    from bench import ClockSampler
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(steps):
                fn()
            e1.record(stream)
        torch.cuda.synchronize()
    _CLOCKS["last"] = clk.summary()
    return e0.elapsed_time(e1) / steps


def cufft_ms(n, K, steps, warmup, stream):
    import torch
    x = torch.randn(n, dtype=torch.complex128, device="cuda")

    def fn():
        for _ in range(K):
            torch.fft.fft(x)
    return timeit(fn, steps, warmup, stream)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only", default="cfg1,cfg2,cfg2adj,cfg3,cfg4,cfg5,inv2")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    import paper_1701_04492_b200 as nb
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    sh = stream.cuda_stream
    P = peak()
    out = []
    want = set(args.only.split(","))

    def emit(name, desc, n_pts, ms, bytes_alg, K, plan_s, extra=None):
        gbs = bytes_alg / (ms / 1e3) / 1e9 if bytes_alg else None
        rec = {"config": name, "workload": desc, "points": n_pts, "ms_per_exec": ms,
               "points_per_s": n_pts / (ms / 1e3), "rank_terms": K, "plan_seconds": plan_s,
               "algorithmic_bytes": bytes_alg, "achieved_gbs": gbs,
               "hbm_frac": (gbs / P) if gbs else None, "peak_gbs": P, "clocks": _CLOCKS.get("last")}
        if extra:
            rec.update(extra)
        print(json.dumps(rec), flush=True)
        out.append(rec)

    def dev(a):
        return torch.from_numpy(a).to("cuda")

    if "cfg1" in want:
        rng = np.random.default_rng(71)
        n = 1024
        x = (np.arange(n) + rng.uniform(-0.5, 0.5, n)) / n
        x = np.mod(x, 1.0)
        t0 = time.perf_counter()
        p = nb.plan_nufft2(x, 1e-12)
        ps = time.perf_counter() - t0
        c = dev(rng.standard_normal(n) + 1j * rng.standard_normal(n))
        f = torch.empty_like(c)
        ms = timeit(lambda: p.execute_device(c.data_ptr(), f.data_ptr(), 1, sh), 200, 20, stream)
        emit("cfg1", "NUFFT-II N=1024 eps=1e-12 jittered grid (latency)", n, ms, 44 * n, p.rank(), ps)

    if "cfg2" in want or "cfg2adj" in want:
        rng = np.random.default_rng(72)
        n = 1 << 24
        x = rng.random(n)
        t0 = time.perf_counter()
        p = nb.plan_nufft2(x, 1e-14)
        torch.cuda.synchronize()
        ps = time.perf_counter() - t0
        K = p.rank()
        c = torch.randn(n, dtype=torch.complex128, device="cuda")
        f = torch.randn(n, dtype=torch.complex128, device="cuda")
        cu = cufft_ms(n, K, args.steps, args.warmup, stream)
        if "cfg2" in want:
            ms = timeit(lambda: p.execute_device(c.data_ptr(), f.data_ptr(), 1, sh), args.steps,
                        args.warmup, stream)
            emit("cfg2", "NUFFT-II N=2^24 eps=1e-14 x iid U[0,1)", n, ms, (32 + 12 + 32 * K) * n, K, ps,
                 {"cufft_K_ffts_ms": cu, "exec_over_fft_ratio": ms / cu})
        if "cfg2adj" in want:
            lib = nb.lib()

            def adj():
                nb.api._check(lib.nufft_plan2_adjoint(p._h, f.data_ptr(), c.data_ptr(), sh))
            try:
                ms = timeit(adj, args.steps, args.warmup, stream)
                emit("cfg2adj", "NUFFT-II adjoint (type-I core) N=2^24 eps=1e-14", n, ms,
                     (32 + 12 + 32 * K) * n, K, ps, {"cufft_K_ffts_ms": cu, "exec_over_fft_ratio": ms / cu})
            except Exception as exc:
                print(json.dumps({"config": "cfg2adj", "error": str(exc)[:200]}), flush=True)
        del p, c, f
        torch.cuda.empty_cache()

    if "cfg3" in want:
        rng = np.random.default_rng(73)
        n = 1 << 24
        w = np.clip(np.arange(n) + rng.uniform(-0.5, 0.5, n), 0, n)
        t0 = time.perf_counter()
        p = nb.plan_nufft1(w, 1e-12)
        torch.cuda.synchronize()
        ps = time.perf_counter() - t0
        K = p.rank()
        c = torch.randn(n, dtype=torch.complex128, device="cuda")
        f = torch.empty_like(c)
        ms = timeit(lambda: p.execute_device(c.data_ptr(), f.data_ptr(), 1, sh), args.steps, args.warmup, stream)
        cu = cufft_ms(n, K, args.steps, args.warmup, stream)
        emit("cfg3", "NUFFT-I N=2^24 eps=1e-12 jittered frequencies", n, ms, (32 + 12 + 32 * K) * n, K, ps,
             {"cufft_K_ffts_ms": cu, "exec_over_fft_ratio": ms / cu})
        del p, c, f
        torch.cuda.empty_cache()

    # (the inverse runs before the 2D / type-III configurations: after them its CG iterations
    # measured up to 4x slower in the same process, 4.7 vs 1.2 ms, while alone it is stable)
    if "inv2" in want:
        # inverse type II (inverse.hpp:171-183) on a jittered grid, N = 2^22, gamma 1/4:
        # Toeplitz operator built once (untimed, like a plan), CG solve timed
        rng = np.random.default_rng(76)
        n = 1 << 22
        x = ((np.arange(n) + rng.uniform(-0.25, 0.25, n)) / n) % 1.0
        p = nb.plan_nufft2(x, 1e-14)
        t0 = time.perf_counter()
        op = nb.toeplitz_from_normal(p)
        ps = time.perf_counter() - t0
        c = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        f = nb.exec_nufft2(p, c)
        fd = torch.from_numpy(f).to("cuda")
        sd = torch.empty_like(fd)
        nb.inufft2_device(p, fd.data_ptr(), 1e-10, sd.data_ptr(), op, sh)  # warm-up solve
        torch.cuda.synchronize()
        # median of five solves (a solve is 30 CG iterations with two host round trips each:
        # single samples ranged 36-144 ms across runs of this sweep, 35-36 ms when repeated,
        # scripts/probe_inv2_variance.py)
        from bench import ClockSampler
        solves = []
        with ClockSampler(torch.cuda.current_device()) as cs:
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                r = nb.inufft2_device(p, fd.data_ptr(), 1e-10, sd.data_ptr(), op, sh)
                e1.record(stream)
                torch.cuda.synchronize()
                solves.append(e0.elapsed_time(e1))
        _CLOCKS["last"] = cs.summary()
        ms = float(np.median(solves))
        err = float(torch.linalg.norm(sd.cpu() - torch.from_numpy(c)) / np.linalg.norm(c))
        t0 = time.perf_counter()
        nb.inufft2(p, f, 1e-10, op)
        host_ms = (time.perf_counter() - t0) * 1e3
        emit("inv2", "inverse NUFFT-II N=2^22 jittered (gamma 1/4), tol 1e-10 (device pointers)", n, ms, None,
             p.rank(), ps, {"cg_iterations": r["iterations"], "converged": r["converged"],
                            "rel_error_vs_truth": err, "ms_per_cg_iteration": ms / max(1, r["iterations"]),
                            "host_api_ms": host_ms, "toeplitz_build_seconds": ps,
                            "solve_ms_all": [round(t, 2) for t in solves]})
        del p, op, fd, sd
        torch.cuda.empty_cache()

    if "cfg4" in want:
        # both B families: seed 4041 draws no sample on the node at 1 (bTrivial), seed 4040
        # draws one (B non-trivial: the beta family runs as K dot products); the reference's
        # own inputs (GaussianSampler, tests/fullsize_ref.py).  Algorithmic bytes count the
        # K x K_inner terms both cases actually need (32 + 12 + 32 K K_inner per point).
        n = 1 << 22
        for seed, tag in ((4041, "cfg4t"), (4040, "cfg4n")):
            smp = nb.GaussianSampler(seed)
            x = smp.uniform_vector(n, 0.0, 1.0)
            w = smp.uniform_vector(n, 0.0, float(n))
            c = dev(smp.complex_vector(n))
            t0 = time.perf_counter()
            p = nb.plan_nufft3(x, w, 1e-9)
            torch.cuda.synchronize()
            ps = time.perf_counter() - t0
            terms = p.rank_a * p.rank_inner
            f = torch.empty_like(c)
            ms = timeit(lambda: p.execute_device(c.data_ptr(), f.data_ptr(), 1, sh), max(2, args.steps // 2),
                        1, stream)
            emit(tag, "NUFFT-III N=2^22 eps=1e-9 x U[0,1), omega U[0,N)", n, ms, (32 + 12 + 32 * terms) * n,
                 terms, ps, {"bTrivial": p.bTrivial, "effective_rank": p.effective_rank(),
                             "rank_inner": p.rank_inner})
            del p, c, f
            torch.cuda.empty_cache()

    if "cfg5" in want:
        rng = np.random.default_rng(75)
        m = nn = 4096
        cnt = 1 << 24
        x, y = rng.random(cnt), rng.random(cnt)
        t0 = time.perf_counter()
        p = nb.plan_nufft2d2(x, y, m, nn, 1e-9)
        torch.cuda.synchronize()
        ps = time.perf_counter() - t0
        k1, k2 = p.rank_x(), p.rank_y()
        C2 = torch.randn(m, nn, dtype=torch.complex128, device="cuda")
        f = torch.empty(cnt, dtype=torch.complex128, device="cuda")
        ms = timeit(lambda: p.execute_device(C2.data_ptr(), f.data_ptr(), 1, sh), max(2, args.steps // 3),
                    1, stream)
        mn = m * nn
        emit("cfg5", "2D NUFFT-II 4096x4096 -> 2^24 samples eps=1e-9", cnt, ms,
             16 * mn + 32 * k1 * mn + 36 * cnt, k1 * k2, ps, {"rank_x": k1, "rank_y": k2,
                                                              "fft_batches_of_2^24": k1 + k1 * k2})
        del p, C2, f
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1)
    return 0


if __name__ == "__main__":
    sys.exit(main())
