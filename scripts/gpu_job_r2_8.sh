set -x
python -m pytest tests -m gpu -x -q -k "2d or cfg5 or guards" --deselect tests/test_gpu_fullsize.py::test_cfg5_2d_vs_reference > gpurun_out/r2_pytest_j8.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2_pytest_j8.log
python scripts/bench_configs.py --only cfg5 > gpurun_out/r2_cfg5.log 2>&1; cat gpurun_out/r2_cfg5.log
