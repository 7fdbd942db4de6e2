# A/B of two library builds on the 2D cfg5 transform (_abtest/libA.so vs libB.so), then the
# 2D parity / guard tests on B.  Usage: bash scripts/ab_2d.sh > gpurun_out/ab_2d.log
for rep in 1 2; do
for lib in A B; do
  NUFFT_B200_LIB=$PWD/_abtest/lib$lib.so python scripts/bench_configs.py --only cfg5 --steps 15 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', 'cfg5 ms %.3f' % d['ms_per_exec'])"
done; done
NUFFT_B200_LIB=$PWD/_abtest/libB.so python -m pytest -q -m gpu tests/test_gpu_guards.py \
  "tests/test_gpu_fullsize.py::test_cfg5_2d_vs_reference" tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_distributed.py -k "2d or guard or cfg5" 2>&1 | tail -3
