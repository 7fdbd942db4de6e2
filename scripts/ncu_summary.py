#!/usr/bin/env python3
"""Summaries of an `ncu --set full` capture of the type-II kernels for profiles/:
  * a text summary (time, DRAM bytes, FP64 pipe, issue, warps, smem wavefronts, stall totals,
    per-opcode instruction counts, the hottest CUDA source lines),
  * profiles/ncu_traffic.json  (DRAM read+write bytes per launch, the bench's roofline.traffic),
  * profiles/fp64.json         (FP64 thread-instructions per launch and the measured DFMA peak,
                                the bench's roofline.fp64).
Usage: ncu_summary.py REP OUT_TXT [n] [K] [--no-json]   (--no-json: text summary only)"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

write_json = "--no-json" not in sys.argv
argv = [a for a in sys.argv if a != "--no-json"]
rep, out_txt = argv[1], argv[2]
n = int(argv[3]) if len(argv) > 3 else 1 << 24
K = int(argv[4]) if len(argv) > 4 else 20
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second"]
per = defaultdict(list)
for d in data:
    name = d[ix["Kernel Name"]].split("(")[0].split("::")[-1].strip().split("<")[0]
    per[name].append(d)


def val(d, k):
    v = float(d[ix[k]].replace(",", ""))
    u = units[ix[k]]
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "msecond": 1e-3, "usecond": 1e-6,
             "nsecond": 1e-9}.get(u, 1.0)
    return v * scale


lines = []
traffic, fp64, smem = {}, {}, {}
for name, ds in per.items():
    lines.append(f"== {name}  ({len(ds)} launches captured; per-launch means)")
    for k in keys:
        if k in ix:
            v = sum(val(d, k) for d in ds) / len(ds)
            lines.append(f"  {k:65s} {v:.6g} {units[ix[k]] if 'bytes' not in k and 'duration' not in k else ''}")
    t = sum(val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum") for d in ds) / len(ds)
    traffic[name] = t
    if "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum" in ix:
        wf = sum(val(d, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") for d in ds) / len(ds)
        smem[name] = {"lsu_shared_wavefronts": wf, "per_point_term": wf / (n * K)}
    # FP64 thread instructions from the SASS source page
    base = name.split("<")[0].replace("void ", "").strip()
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{base}"],
                         capture_output=True, text=True).stdout
    srows = [r for r in csv.reader(src.splitlines())]
    sh = srows[1]
    si = {h: i for i, h in enumerate(sh)}
    ops = defaultdict(float)
    stalls = defaultdict(float)
    samples = 0.0
    seen = set()
    for r in srows[2:]:
        if len(r) != len(sh) or r[0] == "Address" or r[0] in seen:
            continue  # the view repeats each SASS line once per matching function block
        seen.add(r[0])
        toks = r[si["Source"]].split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        ops[op] += float(r[si["Thread Instructions Executed"]] or 0)
        samples += float(r[si["Warp Stall Sampling (All Samples)"]] or 0)
        for h, i in si.items():
            if h.startswith("stall_") and "Not Issued" not in h:
                stalls[h[6:]] += float(r[i] or 0)
    f64 = sum(ops[o] for o in ("DFMA", "DADD", "DMUL")) / len(ds)
    pipe = sum(val(d, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active") for d in ds) / len(ds)
    fp64[name] = {"fp64_thread_inst": f64, "fp64_pipe_pct": pipe,
                  "per_point_term": f64 / (n * K)}
    lines.append(f"  FP64 thread-instructions per launch {f64:.4g} ({f64 / (n * K):.1f} per point-term at N={n}, K={K}): "
                 + ", ".join(f"{o} {ops[o] / len(ds):.3g}" for o in ("DFMA", "DADD", "DMUL")))
    top = sorted(ops.items(), key=lambda kv: -kv[1])[:12]
    tot = sum(ops.values()) or 1
    lines.append("  thread-instruction mix: " + ", ".join(f"{o} {100 * v / tot:.1f}%" for o, v in top))
    lines.append("  stall samples: " + ", ".join(f"{k} {100 * v / samples:.1f}%" for k, v in
                                               sorted(stalls.items(), key=lambda kv: -kv[1])[:9]))
    hot = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_cuda_lines.py"), rep, base, "14"],
                         capture_output=True, text=True).stdout
    lines.append("  hottest CUDA source lines (share of stall samples, top stall reasons):")
    lines += ["    " + ln for ln in hot.splitlines()[1:]]
open(out_txt, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
if not write_json:
    sys.exit(0)
json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
# shared-memory pipe: one 128-byte wavefront per clock per SM (LDS.128 127.9 B/clk/SM measured,
# scripts/microbench_fft8.cu); the bench divides by the live kernel time
json.dump({"n": n, "K": K, "kernels": smem, "peak_wavefronts_per_s": 148 * 1.965e9,
           "peak_source": "1 shared-memory wavefront (128 B) per clock per SM: LDS.128 127.9 B/clk/SM, STS.128 "
                          "111.9 B/clk/SM measured (scripts/microbench_fft8.cu) x 148 SMs x 1965 MHz",
           "capture": os.path.basename(rep)},
          open(os.path.join(ROOT, "profiles", "smem.json"), "w"), indent=1)
peak_file = os.path.join(ROOT, "profiles", "r2_microbench_pipes.txt")
per_clk, clk = 63.37, 1.965e9
try:
    for ln in open(peak_file):
        if ln.startswith("{"):
            per_clk = json.loads(ln)["dfma_thread_ops_per_clk_sm"]
except OSError:
    pass
json.dump({"n": n, "K": K, "kernels": fp64,
           "peak_fp64_thread_inst_per_s": per_clk * 148 * clk,
           "peak_source": f"measured DFMA issue {per_clk:.2f} thread-ops/clk/SM (scripts/microbench_pipes.cu) x 148 SMs "
                          f"x 1965 MHz (clocks.max.sm)", "capture": os.path.basename(rep)},
          open(os.path.join(ROOT, "profiles", "fp64.json"), "w"), indent=1)
