# checkpoint (one ncu per call): full GPU suite, smoke, full bench (with CPU
# baseline), reference arm, every §8(d) configuration, and the ncu launch list
TAG=${1:-ck}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo ref_rc=$?
timeout 900 python scripts/bench_configs.py --out gpurun_out/configs_$TAG.json > gpurun_out/configs_$TAG.log 2>&1; echo configs_rc=$?
BC="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$BC > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv $BC > gpurun_out/ncu_launch.log 2>&1
echo ncu_rc=$?
