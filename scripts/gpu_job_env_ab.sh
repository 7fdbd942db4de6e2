# A/B environment switches with a short bench each: ENVS="A=1,B=2 A=0" (comma-separated per case)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -2
i=0
for E in ${ENVS}; do
  i=$((i+1))
  env $(echo $E | tr ',' ' ') timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_$i.json 2>gpurun_out/ab_$i.err
  python -c "import json; d=json.load(open('gpurun_out/ab_$i.json')); print('$E', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['per_pass_ms'].items()}, d['clocks']['sm_mhz'])"
done
