set -x
nproc
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider 2>&1 | tail -25
timeout 600 python bench.py --steps 200 --warmup 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench_rc=$?
BC="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$BC > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $BC > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_pass -s 2 -c 2 -o gpurun_out/prof_r1 $BC > gpurun_out/ncu_full.log 2>&1
echo ncu_rc=$?
tail -5 gpurun_out/ncu_full.log
