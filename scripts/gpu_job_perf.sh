# perf iteration: parity (type II) -> bench -> ncu full capture of both passes
TAG=${1:-v}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_api.py -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -4
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print(d['ms_per_step'], d['value'], d['roofline']['per_pass_ms'], d['roofline']['frac'], d['clocks'])"
BC="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
$BC > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_pass -s 2 -c 2 -o gpurun_out/prof_$TAG $BC > gpurun_out/ncu_full.log 2>&1
echo ncu_rc=$?
