set -x
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mb5 scripts/microbench_fft5.cu && /tmp/mb5 > gpurun_out/mb5.txt 2>&1
cat gpurun_out/mb5.txt
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_s5_0.json 2> gpurun_out/bench_s5_0.err; echo bench_rc=$?
head -c 1500 gpurun_out/bench_s5_0.json
