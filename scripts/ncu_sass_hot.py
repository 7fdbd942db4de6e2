#!/usr/bin/env python3
"""Hot SASS lines and per-opcode stall totals of one kernel from an ncu report
(`ncu -i REP --page source --csv` SASS view).  Usage: ncu_sass_hot.py REP REGEX [top]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{rx}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data, _seen = [], set()
for r in rows[2:]:  # the view repeats each SASS line once per matching function block
    if len(r) == len(hdr) and r[0] != "Address" and r[0] not in _seen:
        _seen.add(r[0])
        data.append(r)
S = ix["Warp Stall Sampling (All Samples)"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[S]) for r in data)
byop = defaultdict(lambda: [0.0, 0.0])
for r in data:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    op = op.split(".")[0]
    byop[op][0] += float(r[S])
    byop[op][1] += float(r[ix["Instructions Executed"]] or 0)
print(f"total samples {tot:.0f}")
print("by opcode (samples %, instructions):")
for op, (s, n) in sorted(byop.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"  {op:10s} {100 * s / tot:6.2f}%  {n:14.0f}")
print(f"top {top} lines:")
for k, r in enumerate(sorted(data, key=lambda r: -float(r[S]))[:top]):
    st = sorted(((float(r[ix[h]]), h[6:]) for h in stalls if float(r[ix[h]] or 0) > 0), reverse=True)[:3]
    print(f"  {r[0][-5:]} {100 * float(r[S]) / tot:5.2f}%  {r[ix['Source']].strip()[:60]:60s} " +
          " ".join(f"{n}:{100 * v / tot:.2f}" for v, n in st))
print("stall totals:")
for h in sorted(stalls, key=lambda h: -sum(float(r[ix[h]] or 0) for r in data)):
    v = sum(float(r[ix[h]] or 0) for r in data)
    if v > 0.005 * tot:
        print(f"  {h[6:]:18s} {100 * v / tot:5.1f}%")
