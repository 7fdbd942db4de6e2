timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python scripts/bench_configs.py --only cfg4,cfg3,cfg2 --out gpurun_out/configs_stack.json > gpurun_out/configs_stack.log 2>&1; echo configs_rc=$?
python - <<PY
import json
for e in json.load(open("gpurun_out/configs_stack.json")):
    print(e["config"], round(e["ms_per_exec"],3), e.get("hbm_frac"))
PY
