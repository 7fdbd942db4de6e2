#!/usr/bin/env python3
"""Per-CUDA-source-line shared-memory wavefronts of one kernel (total, ideal, excess = bank
conflicts) from an ncu capture (needs -lineinfo).  Usage: ncu_smem_lines.py REP REGEX [top]"""
import csv
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{rx}"], capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
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
            wf = float(r[ix["L1 Wavefronts Shared"]] or 0)
            ex = float(r[ix["L1 Wavefronts Shared Excessive"]] or 0)
        except (ValueError, IndexError, KeyError):
            continue
        if wf > 0:
            rows.append((wf, ex, fname, r[0], r[1][:80]))
tot = sum(x[0] for x in rows) or 1
print(f"shared wavefronts {tot:.3e}, excess {sum(x[1] for x in rows):.3e} ({100 * sum(x[1] for x in rows) / tot:.1f} %)")
for wf, ex, f, ln, src in sorted(rows, key=lambda x: -x[0])[:top]:
    print(f"{100 * wf / tot:5.1f}% (excess {100 * ex / tot:4.1f}%) {f}:{ln:>5} {src}")
