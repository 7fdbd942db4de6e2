"""Summarize an ncu source page (SASS) by opcode: stall samples and executed instructions."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
kernel = None
agg = {}
hdr = None
for row in csv.reader(out.splitlines()):
    if not row:
        continue
    if row[0] == "Kernel Name":
        kernel = row[1][:60]
        agg[kernel] = defaultdict(lambda: [0, 0])
        continue
    if row[0] == "Address":
        hdr = {h: i for i, h in enumerate(row)}
        continue
    if hdr is None or kernel is None:
        continue
    src = row[hdr["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    try:
        samples = int(row[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        inst = int(row[hdr["Instructions Executed"]] or 0)
    except ValueError:
        continue
    agg[kernel][op][0] += samples
    agg[kernel][op][1] += inst
for k, d in agg.items():
    tot_s = sum(v[0] for v in d.values()) or 1
    tot_i = sum(v[1] for v in d.values()) or 1
    print(f"== {k}  samples={tot_s} inst={tot_i}")
    for op, (s, i) in sorted(d.items(), key=lambda kv: -kv[1][0])[:18]:
        print(f"  {op:10s} stall%={100*s/tot_s:5.1f}  inst%={100*i/tot_i:5.1f}")
