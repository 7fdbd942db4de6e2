"""Build libnufft_b200.so in-tree: every .cu under csrc/ compiled by nvcc for
sm_100a (-gencode arch=compute_100a,code=sm_100a, -lineinfo), linked into one
shared library exporting the C-ABI of include/nufft_b200.h."""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libnufft_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr", "-I" + os.path.join(HERE, "..", "include")]
# NB_NVCC_EXTRA: extra nvcc flags for experiment builds (e.g. "-Xptxas=-warn-spills")
FLAGS += os.environ.get("NB_NVCC_EXTRA", "").split()


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _headers_digest() -> str:
    h = hashlib.sha1()
    for d in (CSRC, os.path.join(HERE, "..", "include")):
        for f in sorted(os.listdir(d)):
            if f.endswith((".cuh", ".hpp", ".h")):
                h.update(open(os.path.join(d, f), "rb").read())
    return h.hexdigest()[:12]


def _compile(src: str, digest: str, verbose: bool) -> str:
    base = os.path.splitext(os.path.basename(src))[0]
    obj = os.path.join(OBJ, f"{base}.o")
    stamp = obj + ".stamp"
    key = digest + hashlib.sha1(open(src, "rb").read()).hexdigest()[:12] + " ".join(FLAGS)
    if os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read() == key:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-x", "cu", "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    open(stamp, "w").write(key)
    return obj


def build(verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(OBJ, exist_ok=True)
    digest = _headers_digest()
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=jobs or min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, digest, verbose), srcs))
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        tmp = LIB + ".tmp"
        r = subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt",
                            "-lpthread", "-ldl"], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n" + r.stderr)
        os.replace(tmp, LIB)
    _build_example()
    return LIB


CPP_DIR = os.path.join(HERE, "..", "tests", "cpp")
# C++ programs written against the drop-in headers (include/nufft) and linked with
# the library: the usage example / self-check, and the end-to-end timing of
# exec_nufft2(plan, std::vector) that bench.py reports as e2e.dropin_pageable
CPP_PROGRAMS = {"example_dropin": os.path.join(CPP_DIR, "example_dropin.cpp"),
                "bench_dropin": os.path.join(CPP_DIR, "bench_dropin.cpp"),
                # the reference CLI's subcommands / CSV files / exit codes on the GPU
                "nufft": os.path.join(HERE, "tools", "nufft_cli.cpp")}
CLI_BIN = os.path.join(OBJ, "nufft")
EXAMPLE_BIN = os.path.join(OBJ, "example_dropin")
BENCH_DROPIN_BIN = os.path.join(OBJ, "bench_dropin")


def _build_example() -> None:
    for name, src in CPP_PROGRAMS.items():
        exe = os.path.join(OBJ, name)
        hdrs = [os.path.join(HERE, "..", "include", "nufft", h) for h in os.listdir(os.path.join(HERE, "..", "include", "nufft"))]
        if os.path.exists(exe) and os.path.getmtime(exe) >= max([os.path.getmtime(LIB), os.path.getmtime(src)] +
                                                                [os.path.getmtime(h) for h in hdrs]):
            continue
        r = subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(HERE, "..", "include"),
                            src, "-o", exe, "-L" + HERE, "-lnufft_b200",
                            "-Wl,-rpath,$ORIGIN/.."], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"{name} build failed:\n" + r.stderr)


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
