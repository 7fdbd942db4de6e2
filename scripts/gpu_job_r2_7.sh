set -x
python -m pytest tests -m gpu -x -q -k "type3 or nufft3 or cfg4" > gpurun_out/r2_pytest_j7.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_pytest_j7.log
python scripts/bench_configs.py --only cfg4 > gpurun_out/r2_cfg4.log 2>&1; cat gpurun_out/r2_cfg4.log
