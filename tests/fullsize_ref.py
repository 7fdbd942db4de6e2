"""TEST INFRASTRUCTURE ONLY — the reference's own output at BASELINE.json sizes.

Each BASELINE config gets seeded inputs drawn with the reference's sampler
(nufft::GaussianSampler, proj/include/nufft/random.hpp:14-60: mt19937_64 +
Box-Muller; the C port's sampler is bit-identical to it, tests/test_oracle.py)
and, run as a script, the reference's own plan/exec on those inputs through
oracle/_ref/libnufft_ref.so (the reference headers compiled unmodified):

    cfg2    exec_nufft2,  N = 2^24, eps 1e-14, x iid U[0,1)            transforms.hpp:168-199
            and, on the same plan, 8 further c vectors (the batch-8 config) -> cfg2b8
    cfg3    exec_nufft1,  N = 2^24, eps 1e-12, w_k = clip(k + d_k, 0, N) transforms.hpp:287-289
    cfg4t / cfg4n  exec_nufft3, N = 2^22, eps 1e-9, x iid U[0,1), w iid U[0,N)
            (one seed with bTrivial = true, one with bTrivial = false)   transforms.hpp:382-394
    cfg5    exec_nufft2d2, 4096 x 4096, 2^24 samples, eps 1e-9         transform2d.hpp:107-147

    python tests/fullsize_ref.py <cfg> <outdir> [threads]

writes <outdir>/<cfg>.npy (the output vector; for cfg2b8 shape (8, N)) and
<outdir>/<cfg>.json (timings, rank, bTrivial).  tests/test_gpu_fullsize.py
starts these as background processes at session start (they run on the GPU
box's host cores while the GPU tests proceed) and compares whole vectors.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

N24 = 1 << 24
N22 = 1 << 22
# seeds: cfg4t/cfg4n were chosen so that bTrivial is true / false at N = 2^22
# (a sample with round(N x) = N makes B non-trivial, transforms.hpp:345-350)
SEEDS = {"cfg2": 2024, "cfg3": 3033, "cfg4t": 4041, "cfg4n": 4040, "cfg5": 5055}
EPS = {"cfg2": 1e-14, "cfg2b8": 1e-14, "cfg3": 1e-12, "cfg4t": 1e-9, "cfg4n": 1e-9, "cfg5": 1e-9}
RUNS = ("cfg2", "cfg3", "cfg4t", "cfg4n", "cfg5")  # one process each (cfg2 also writes cfg2b8)


def _sampler(seed: int):
    from oracle import pyoracle
    kind = "reference" if pyoracle.available("reference") else "port"
    return pyoracle.Oracle(kind).sampler(seed)


def inputs(cfg: str) -> dict:
    """The seeded inputs of one config (identical on every host)."""
    if cfg in ("cfg2", "cfg2b8"):
        s = _sampler(SEEDS["cfg2"])
        x = s.uniform_vector(N24, 0.0, 1.0)
        c = s.complex_vector(N24)
        if cfg == "cfg2":
            return {"x": x, "c": c}
        return {"x": x, "cb": np.stack([s.complex_vector(N24) for _ in range(8)])}
    if cfg == "cfg3":
        s = _sampler(SEEDS["cfg3"])
        d = s.uniform_vector(N24, -0.5, 0.5)
        w = np.clip(np.arange(N24, dtype=np.float64) + d, 0.0, float(N24))
        return {"w": w, "c": s.complex_vector(N24)}
    if cfg in ("cfg4t", "cfg4n"):
        s = _sampler(SEEDS[cfg])
        x = s.uniform_vector(N22, 0.0, 1.0)
        w = s.uniform_vector(N22, 0.0, float(N22))
        return {"x": x, "w": w, "c": s.complex_vector(N22)}
    if cfg == "cfg5":
        s = _sampler(SEEDS["cfg5"])
        x = s.uniform_vector(N24, 0.0, 1.0)
        y = s.uniform_vector(N24, 0.0, 1.0)
        C2 = s.complex_vector(N24).reshape(4096, 4096)
        return {"x": x, "y": y, "C": C2}
    raise ValueError(cfg)


def b_trivial(x: np.ndarray) -> bool:
    """bTrivial of plan_nufft3 (transforms.hpp:343-350): no sample rounds to the node N."""
    n = len(x)
    return not bool(np.any(x * n >= n - 0.5))


def run_reference(cfg: str, outdir: str, threads: int) -> None:
    from oracle import pyoracle
    o = pyoracle.Oracle("reference")
    inp = inputs(cfg)
    eps = EPS[cfg]
    info = {"cfg": cfg, "eps": eps, "threads": threads}
    t0 = time.perf_counter()
    if cfg == "cfg2":
        p = o.plan2(inp["x"], eps)
        info["plan_s"] = time.perf_counter() - t0
        info["rank"] = p.rank
        t1 = time.perf_counter()
        f = p.execute(inp["c"], threads=threads)
        info["exec_s"] = time.perf_counter() - t1
        _save(outdir, "cfg2", f, info)
        cb = inputs("cfg2b8")["cb"]
        t1 = time.perf_counter()
        fb = np.stack([p.execute(cb[b], threads=threads) for b in range(len(cb))])
        info = dict(info, cfg="cfg2b8", exec_s=time.perf_counter() - t1)
        _save(outdir, "cfg2b8", fb, info)
        return
    elif cfg == "cfg3":
        p = o.plan1(inp["w"], eps)
        info["plan_s"] = time.perf_counter() - t0
        info["rank"] = p.rank
        t1 = time.perf_counter()
        f = p.execute(inp["c"])
    elif cfg in ("cfg4t", "cfg4n"):
        p = o.plan3(inp["x"], inp["w"], eps)
        info["plan_s"] = time.perf_counter() - t0
        bt, ka, ke, ki = p.info3()
        info.update(bTrivial=bt, rank=ka, effective_rank=ke, inner_rank=ki)
        t1 = time.perf_counter()
        f = p.execute(inp["c"])
    else:
        p = o.plan2d2(inp["x"], inp["y"], 4096, 4096, eps)
        info["plan_s"] = time.perf_counter() - t0
        info["rank"] = list(p.info2d()[:2])
        t1 = time.perf_counter()
        f = p.execute(inp["C"])
    info["exec_s"] = time.perf_counter() - t1
    _save(outdir, cfg, f, info)


def _save(outdir: str, cfg: str, f: np.ndarray, info: dict) -> None:
    tmp = os.path.join(outdir, f".{cfg}.tmp.npy")
    np.save(tmp, f)
    with open(os.path.join(outdir, f"{cfg}.json"), "w") as fh:
        json.dump(info, fh)
    os.replace(tmp, os.path.join(outdir, f"{cfg}.npy"))


if __name__ == "__main__":
    run_reference(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 1)


def runs_for(nodeids) -> tuple:
    """Which reference runs the selected test_gpu_fullsize items need."""
    tags = {"cfg2": ("cfg2_",), "cfg3": ("cfg3_",), "cfg4t": ("cfg4t",), "cfg4n": ("cfg4n",),
            "cfg5": ("cfg5_",)}
    need = tuple(r for r in RUNS if any(any(t in nid for t in tags[r]) for nid in nodeids))
    return need or RUNS


class Runner:
    """Background reference processes, one per entry of RUNS, started at test
    collection (tests/conftest.py) so they run on the host cores while the
    other GPU tests proceed."""

    def __init__(self, outdir: str, threads: int | None = None, runs=RUNS):
        import subprocess
        self.outdir = outdir
        cores = os.cpu_count() or 4
        # cfg2 is the only threaded reference path (transforms.hpp:181); the
        # other four are single-threaded in the reference
        t2 = threads or max(1, cores - 8)  # leave cores for pytest itself
        self.procs = {}
        for cfg in runs:
            log = open(os.path.join(outdir, f"{cfg}.log"), "w")
            self.procs[cfg] = subprocess.Popen(
                [sys.executable, os.path.abspath(__file__), cfg, outdir, str(t2 if cfg == "cfg2" else 1)],
                stdout=log, stderr=subprocess.STDOUT, cwd=ROOT)

    def result(self, cfg: str, timeout: float = 1500.0):
        """(output, info) of one config; waits for its process."""
        run = "cfg2" if cfg == "cfg2b8" else cfg
        if run not in self.procs:
            raise RuntimeError(f"reference run {run} was not started for this session")
        path = os.path.join(self.outdir, f"{cfg}.npy")
        t0 = time.time()
        while not os.path.exists(path):
            rc = self.procs[run].poll()
            if rc is not None and not os.path.exists(path):
                log = open(os.path.join(self.outdir, f"{run}.log")).read()[-2000:]
                raise RuntimeError(f"reference run {run} exited {rc}:\n{log}")
            if time.time() - t0 > timeout:
                raise TimeoutError(f"reference run {run} not done after {timeout:.0f} s")
            time.sleep(0.5)
        with open(os.path.join(self.outdir, f"{cfg}.json")) as fh:
            info = json.load(fh)
        return np.load(path), info

    def close(self) -> None:
        for p in self.procs.values():
            if p.poll() is None:
                p.kill()
                p.wait()
