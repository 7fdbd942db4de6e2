"""List the SASS instructions of one kernel with excess shared-memory wavefronts
(bank conflicts) from an ncu source page export.
usage: ncu -i rep --page source --csv --kernel-name regex:K --print-source sass > src.csv
       python scripts/ncu_conflicts.py src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
out = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        ex = float(r[ix["L1 Wavefronts Shared Excessive"]] or 0)
        wf = float(r[ix["L1 Wavefronts Shared"]] or 0)
        ideal = float(r[ix["L1 Wavefronts Shared Ideal"]] or 0)
    except ValueError:
        continue
    if wf > 0:
        out.append((ex, wf, ideal, r[ix["Address"]], r[ix["Source"]]))
out.sort(reverse=True)
tot = sum(o[1] for o in out)
print(f"shared wavefronts {tot:.3e}, excessive {sum(o[0] for o in out):.3e}")
for ex, wf, ideal, addr, src in out[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{addr:>8} excess {ex:10.3e} wf {wf:10.3e} ideal {ideal:10.3e}  {src[:90]}")
