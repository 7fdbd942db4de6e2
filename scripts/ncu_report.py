"""Write a committed text summary of an ncu --set full capture: per-kernel
duration, DRAM bytes (the roofline `traffic`), throughput, occupancy, FP64
pipe activity, stall breakdown and SASS opcode mix.
usage: python scripts/ncu_report.py gpurun_out/prof.ncu-rep profiles/rN_ncu_full.txt [profiles/ncu_traffic.json]"""
import csv
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
traffic_json = sys.argv[3] if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
keys = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__block_size", "launch__grid_size",
    "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "sm__cycles_elapsed.avg.per_second",
]
stall_prefix = "smsp__pcsamp_warps_issue_stalled_"
lines, traffic = [], {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    short = name.split("<")[0].split("::")[-1] if "<" in name else name.split("(")[0].split("::")[-1]
    lines.append(f"== {name}")
    vals = {}
    for k in keys:
        if k in hdr:
            vals[k] = r[hdr.index(k)]
            lines.append(f"  {k:70s} {r[hdr.index(k)]:>20s} {units[hdr.index(k)]}")
    try:
        rd = float(vals["dram__bytes_read.sum"])
        wr = float(vals["dram__bytes_write.sum"])
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        u_r = units[hdr.index("dram__bytes_read.sum")]
        u_w = units[hdr.index("dram__bytes_write.sum")]
        traffic[short] = rd * scale.get(u_r, 1) + wr * scale.get(u_w, 1)
    except Exception:
        pass
    st = []
    for i, h in enumerate(hdr):
        if h.startswith(stall_prefix) and not h.endswith("not_issued"):
            try:
                st.append((float(r[i]), h[len(stall_prefix):]))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    lines.append("  stall samples: " + ", ".join(f"{n} {100 * v / tot:.1f}%" for v, n in sorted(st, reverse=True)[:8]))
open(out, "w").write("\n".join(lines) + "\n")
if traffic_json:
    json.dump(traffic, open(traffic_json, "w"), indent=1)
print("\n".join(lines))
