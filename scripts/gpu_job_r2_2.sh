# round 2 job 2: type-III restructure (parity + full size), unpermute A/B, pipe microbenchmarks,
# sanitizer timing, config sweep with clocks
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/microbench_pipes scripts/microbench_pipes.cu
scripts/microbench_pipes > gpurun_out/r2_microbench_pipes.txt 2>&1
cat gpurun_out/r2_microbench_pipes.txt
export NUFFT_FULLSIZE_RECORD=gpurun_out/r2_fullsize_t3.jsonl
rm -f $NUFFT_FULLSIZE_RECORD
python -m pytest tests -m gpu -x -q -k "type3 or nufft3 or exec_counts or distributed or sorted or multi or cfg4" > gpurun_out/r2_pytest_t3.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_pytest_t3.log
cat $NUFFT_FULLSIZE_RECORD
python scripts/ab_unpermute.py > gpurun_out/r2_ab_unpermute.txt 2>&1; cat gpurun_out/r2_ab_unpermute.txt
python scripts/bench_configs.py --only cfg4,cfg3,cfg5 --out gpurun_out/r2_configs_t3.json > gpurun_out/r2_configs_t3.log 2>&1; tail -5 gpurun_out/r2_configs_t3.log
( time timeout 900 python -m pytest tests/test_gpu_sanitizer.py -x -q -k "memcheck and type2-" ) > gpurun_out/r2_san1.log 2>&1; tail -5 gpurun_out/r2_san1.log
( time timeout 900 python -m pytest tests/test_gpu_sanitizer.py -x -q -k "racecheck and type2-" ) > gpurun_out/r2_san2.log 2>&1; tail -5 gpurun_out/r2_san2.log
