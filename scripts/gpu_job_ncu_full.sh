# one full ncu capture of the two type-II kernels (second exec, after warm-up)
TAG=${1:-ck}
mkdir -p gpurun_out
BC="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$BC > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_pass -s 2 -c 2 -o gpurun_out/prof_$TAG $BC > gpurun_out/ncu_full.log 2>&1
echo ncu_rc=$?
