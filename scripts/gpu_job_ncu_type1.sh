# one full ncu capture of the transpose-core kernels (type I at 2^24, eps 1e-12)
mkdir -p gpurun_out
CMD="python scripts/bench_configs.py --only cfg3 --steps 2 --warmup 1"
$CMD > gpurun_out/plain_t1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_pass -s 4 -c 2 -o gpurun_out/prof_t1_$1 $CMD > gpurun_out/ncu_t1.log 2>&1
echo ncu_rc=$?
