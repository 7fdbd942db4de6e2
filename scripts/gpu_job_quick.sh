# quick A/B: parity subset + device-timed bench + (optional) every configuration
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_rc=$?
python - <<PY
import json
d=json.load(open("gpurun_out/bench_$TAG.json"))
print("ms_per_step", d["ms_per_step"], "per_pass", d["roofline"]["per_pass_ms"], "frac", d["roofline"]["transform"]["frac"])
PY
if [ "$2" = "configs" ]; then
timeout 900 python scripts/bench_configs.py --out gpurun_out/configs_$TAG.json > gpurun_out/configs_$TAG.log 2>&1; echo configs_rc=$?
python - <<PY
import json
for e in json.load(open("gpurun_out/configs_$TAG.json")):
    print(e["config"], round(e["ms_per_exec"],3), e.get("hbm_frac"))
PY
fi
