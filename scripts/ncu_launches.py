#!/usr/bin/env python3
"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel
(template arguments kept) total ms, launches and mean ms, in launch order of first
appearance.  Usage: ncu_launches.py FILE.csv"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = OrderedDict()
for r in rows:
    if not r:
        continue
    if r[0] == "ID":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr) or r[hdr["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[hdr["Kernel Name"]].split("(")[0].replace("(anonymous namespace)::", "").replace("nb::", "").strip()
    v = float(r[hdr["Metric Value"]].replace(",", ""))
    unit = r[hdr["Metric Unit"]]
    ms = v * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1e-6)
    a = agg.setdefault(name, [0.0, 0])
    a[0] += ms
    a[1] += 1
tot = sum(v[0] for v in agg.values())
for k, (ms, c) in agg.items():
    print(f"{ms:10.3f} ms {c:5d} x {ms / c:8.4f} ms  {100 * ms / tot:5.1f}%  {k[:90]}")
print(f"{tot:10.3f} ms total")
