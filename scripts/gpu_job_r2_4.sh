set -x
python scripts/e2e_paths.py > gpurun_out/r2_e2e_paths.txt 2>&1; cat gpurun_out/r2_e2e_paths.txt
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-dropin > gpurun_out/r2_bench_ab.json 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2_bench_ab.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], d["roofline"]["per_pass_ms"], "frac", d["roofline"]["transform"]["frac"])
PY
python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -x -q -k "cfg2 or type2 or pow2" > gpurun_out/r2_pytest_j4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pytest_j4.log
