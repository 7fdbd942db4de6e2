#!/usr/bin/env python3
"""Per-CUDA-source-line warp-stall samples of one kernel (ncu 'cuda,sass' source view;
needs -lineinfo).  Usage: ncu_cuda_lines.py REP REGEX [top]"""
import csv
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{rx}"], capture_output=True, text=True).stdout
lines, fname, hdr = [], None, None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and r[0] not in ("", "Function Name"):
        ix = {h: i for i, h in enumerate(hdr)}
        try:
            s = float(r[4])
            n = float(r[7] or 0)
        except (ValueError, IndexError):
            continue
        stall = {h: float(r[i] or 0) for h, i in ix.items() if h.startswith("stall_") and "Not" not in h and i < len(r) and r[i] not in ("", "-")}
        lines.append((s, n, fname, r[0], r[1][:70], stall))
tot = sum(x[0] for x in lines) or 1
print(f"total samples {tot:.0f}")
for s, n, f, ln, src, st in sorted(lines, key=lambda x: -x[0])[:top]:
    top3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100 * s / tot:5.2f}% {f}:{ln:>5} {src:70s} " + " ".join(f"{k[6:]}:{100 * v / tot:.1f}" for k, v in top3))
