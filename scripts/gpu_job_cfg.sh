timeout 900 python scripts/bench_configs.py --out gpurun_out/r2_configs_$1.json > gpurun_out/r2_configs_$1.log 2>&1; echo configs_rc=$?
python - <<PY
import json
for e in json.load(open("gpurun_out/r2_configs_$1.json")):
    print(e["config"], round(e["ms_per_exec"],3), e.get("hbm_frac"), e["clocks"]["reasons"], e.get("solve_ms_all"))
PY
