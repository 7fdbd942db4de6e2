nvidia-smi topo -m 2>/dev/null | head -8
cat /sys/bus/pci/devices/*/numa_node 2>/dev/null | sort | uniq -c | head
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_e2e_$i.json 2>/dev/null
python - <<PY
import json
d=json.loads(open("gpurun_out/bench_e2e_$i.json").read().strip().splitlines()[-1])
e=d["e2e"]
print(round(d["ms_per_step"],3), round(e["value"]/1e9,3), round(e["ms_per_step"],1), e["host_affinity"], round(e["batch1_pinned"]["ms_per_step"],2), round(e.get("dropin_pageable",{}).get("ms_per_step",0),1))
PY
done
