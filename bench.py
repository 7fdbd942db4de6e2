#!/usr/bin/env python3
"""Benchmark: NUFFT-II N=2^24, fp64, eps=1e-14 (BASELINE.json cfg2) — points/s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--mode batch|rsplit] [--batch B] [--n N] [--eps E]

One process per GPU (torchrun for N > 1; NCCL process group).  A step is one
type-II execution of the fused two-pass kernels over one batch of
device-resident coefficients (plan built once, outside the timed region, as
in the reference's plan/online split, transforms.hpp:133 vs :168).

  --mode batch  (default, weak scaling): every rank transforms its own c
                 with the shared x — no data-path collective.
  --mode rsplit (strong scaling): the K rank terms are split across ranks,
                 each computes a partial f (nufft_plan2_exec_terms) and the
                 partials are summed with an NCCL reduce to rank 0.

Timing: W untimed warm-up steps, then exactly K steps bracketed by barrier +
synchronize, CUDA events on the launching stream, max over ranks.  Inputs are
larger than L2 (c 256 MiB, spectra 5 GiB per transform).  Extra keys:
roofline (per-pass CUDA events inside the timed region, algorithmic bytes
from SURVEY.md §8(d)), cpu_baseline (the reference compiled here, or the C
port, on this host's cores), e2e (the host-pointer C-ABI call with pinned
buffers on --e2e-batch vectors per call, copies inside the timed region), clocks (nvidia-smi sampled during
the timed region), gpu_launches (library kernel-launch counter).
`--impl reference` times the reference's own CPU exec_nufft2 instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NUFFT-II N=2^24 fp64 ε=1e-14: points/s and % HBM roofline at 1/2/4/8 B200"
UNIT = "points/s"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", choices=["batch", "rsplit"], default="batch")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--eps", type=float, default=1e-14)
    ap.add_argument("--seed", type=int, default=20240)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-batch", type=int, default=8,
                    help="vectors per host call in the e2e measurement (cfg2's batch of 8 c vectors "
                         "sharing x; the host API pipelines their PCIe copies with the transforms)")
    ap.add_argument("--cpu-sample-n", type=int, default=1 << 22)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.lines:
            return None
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "samples": len(sm),
                "reasons": sorted(reasons)}


def algorithmic_bytes(n: int, K: int, batch: int):
    """bytes_II = B*16N (c) + B*16N (f) + 12N (x + index) + B*32*K*N."""
    pass1 = batch * (16 * n + 16 * K * n)            # c read once, K spectra written
    pass2 = batch * (16 * K * n + 16 * n) + 12 * n   # K spectra read, f written, xs + perm
    return pass1, pass2, pass1 + pass2


def cpu_baseline_run(n: int, eps: float, seed: int, steps: int, warmup: int):
    """The reference's own exec_nufft2 (oracle/_ref) or the C port, all host threads."""
    from oracle import pyoracle
    kind = "reference" if pyoracle.available("reference") else "port"
    if not pyoracle.available(kind):
        pyoracle.build()
    o = pyoracle.Oracle(kind)
    rng = np.random.default_rng(seed)
    x = rng.random(n)
    c = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    t0 = time.perf_counter()
    plan = o.plan2(x, eps)
    plan_s = time.perf_counter() - t0
    cores = os.cpu_count() or 1
    threads = min(cores, plan.rank)
    for _ in range(warmup):
        plan.execute(c, threads)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        plan.execute(c, threads)
        times.append(time.perf_counter() - t0)
    t = statistics.mean(times)
    return {
        "value": n / t, "unit": UNIT, "cores": threads, "host_cores": cores, "kind": kind,
        "sample": (f"exec_nufft2 at N=2^{n.bit_length() - 1} (x iid U[0,1), eps={eps:g}, K={plan.rank}), "
                   f"threads={threads} (reference uses min(threads, K) workers), "
                   f"{steps} timed execs after {warmup} warm-up; plan {plan_s:.1f}s untimed; "
                   "FFT backend: oracle/fft_shim.c radix-2 (FFTW3 absent)"),
        "seconds_per_exec": t,
    }


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    steps, warmup = args.steps, args.warmup
    cb = cpu_baseline_run(args.cpu_sample_n, args.eps, args.seed, steps, warmup)
    line = {
        "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": warmup, "ms_per_step": cb["seconds_per_exec"] * 1e3,
        "higher_is_better": True, "scaling": "weak" if args.mode == "batch" else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded x iid U[0,1), c ~ N(0,1)+iN(0,1))",
        "config": {"workload": "NUFFT-II N=2^24 eps=1e-14 x iid U[0,1) (cfg2)",
                   "sample_n": args.cpu_sample_n, "eps": args.eps, "batch": 1},
        "impl": "reference",
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1701_04492_b200 as nb

    world, rank, local = dist_env()
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n, eps, batch = args.n, args.eps, args.batch

    rng = np.random.default_rng(args.seed)
    x = rng.random(n)                     # shared samples (the plan), same on every rank
    t0 = time.perf_counter()
    plan = nb.plan_nufft2(x, eps, device=local)
    torch.cuda.synchronize(dev)
    plan_s = time.perf_counter() - t0
    K = plan.rank()
    gen = torch.Generator(device=dev).manual_seed(args.seed + 1 + rank)
    c = torch.randn(batch, n, dtype=torch.complex128, device=dev, generator=gen)
    f = torch.empty_like(c)
    stream = torch.cuda.Stream(device=dev)
    sh = stream.cuda_stream

    if args.mode == "rsplit" and world > 1:
        r0, r1 = K * rank // world, K * (rank + 1) // world

        def step():
            plan.execute_terms_device(c.data_ptr(), f.data_ptr(), r0, r1, batch, sh)
            dist.reduce(f, dst=0)
        scaling = "strong"
        points_per_step = n * batch
    else:
        def step():
            plan.execute_device(c.data_ptr(), f.data_ptr(), batch, sh)
        scaling = "weak"
        points_per_step = n * batch * world

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize(dev)
    barrier()

    lib = nb.lib()
    launches0 = lib.nufft_kernel_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize(dev)
        barrier()
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(args.steps):
                step()
            ev1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
    launches = lib.nufft_kernel_launch_count() - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = points_per_step / (ms_max / 1e3)

    # ---- roofline: per-pass device time inside a timed loop of the same exec
    p1_bytes, p2_bytes, total_bytes = algorithmic_bytes(n, K, 1)
    nslots = min(args.steps, 50)
    with torch.cuda.stream(stream):
        for i in range(nslots):
            plan.execute_timed_device(c[0].data_ptr(), f[0].data_ptr(), sh, i)
    torch.cuda.synchronize(dev)
    ms1, ms2 = plan.timing_read(nslots)
    ms1, ms2 = ms1 / nslots, ms2 / nslots
    peak, peak_src = measured_peak()
    dom = ("k2_pass2", p2_bytes, ms2) if ms2 >= ms1 else ("k2_pass1", p1_bytes, ms1)
    achieved = dom[1] / (dom[2] / 1e3) / 1e9
    traffic, traffic_kernel = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:  # ncu dram read+write of the same kernel (its template instance name starts with dom[0])
            for name, val in json.load(open(tpath)).items():
                if name.startswith(dom[0]):
                    traffic, traffic_kernel = val, name
                    break
        except Exception:
            traffic = None
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "traffic": traffic, "kernel": traffic_kernel or dom[0],
        "peak_source": peak_src,
        "algorithmic_bytes_per_launch": dom[1],
        "per_pass_ms": {"k2_pass1": ms1, "k2_pass2": ms2},
        "transform": {"bytes": total_bytes, "ms": ms1 + ms2,
                      "achieved_gbs": total_bytes / ((ms1 + ms2) / 1e3) / 1e9,
                      "frac": total_bytes / ((ms1 + ms2) / 1e3) / 1e9 / peak},
    }

    # ---- e2e: the host-pointer C-ABI call with pinned buffers, copies inside.  One step =
    # one exec_host call on eb fresh c vectors (cfg2's batch of 8 sharing x): the call
    # streams them through the GPU with H2D / transform / D2H overlapped across vectors
    # (a single 2^24 vector cannot overlap: pass 1 needs all of c, pass 2 scatters f).
    def e2e_measure(eb):
        ch = torch.empty(eb, n, dtype=torch.complex128, pin_memory=True)
        for b in range(eb):
            ch[b].copy_(c[b % batch].cpu())
        fh = torch.empty_like(ch).pin_memory()
        plan.execute_host_ptr(ch.data_ptr(), fh.data_ptr(), eb)  # warm
        barrier()
        te = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            plan.execute_host_ptr(ch.data_ptr(), fh.data_ptr(), eb)
            te.append(time.perf_counter() - t0)
        e = torch.tensor([statistics.mean(te)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e, op=dist.ReduceOp.MAX)
        return float(e.item())

    eb = max(1, args.e2e_batch)
    e_s = e2e_measure(eb)
    e2e = {"value": n * eb * world / e_s, "unit": UNIT, "batch": eb,
           "h2d_bytes_per_step": 16 * n * eb, "d2h_bytes_per_step": 16 * n * eb,
           "ms_per_step": e_s * 1e3,
           "api": "nufft_plan2_exec_host (pinned host buffers; batch > 1 pipelines H2D/transform/D2H)"}
    if eb != batch:  # the single-call figure at the device line's batch, for comparison
        e1 = e2e_measure(batch)
        e2e["batch%d" % batch] = {"value": n * batch * world / e1, "ms_per_step": e1 * 1e3}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline_run(args.cpu_sample_n, eps, args.seed, 2, 1)
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as exc:  # the GPU number stands on its own
            cpu = {"value": None, "error": str(exc)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded x iid U[0,1) shared by all ranks; c ~ N(0,1)+iN(0,1) per rank)",
            "config": {"workload": "NUFFT-II N=2^24 eps=1e-14 x iid U[0,1) (cfg2)" if n == 1 << 24
                       else f"NUFFT-II N={n} eps={eps:g}",
                       "n": n, "eps": eps, "rank_K": K, "batch": batch, "mode": args.mode,
                       "parallelism": (f"dp{world} batch-sharded" if scaling == "weak" else f"r-term split over {world} + NCCL reduce"),
                       "l2": "inputs larger than L2 (c 256 MiB, K spectra 5 GiB per transform)",
                       "plan_seconds": plan_s, "path": "fused two-pass" if plan.fused else "generic"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks.summary(),
            "gpu_launches": int(launches),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
