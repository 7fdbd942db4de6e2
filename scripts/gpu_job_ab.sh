# A/B the pass-2 organizations (NUFFT_PASS2_VARIANT) with a short bench each
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -p no:cacheprovider -x 2>&1 | tail -2
for V in ${VARIANTS:-0 1 2 3}; do
  NUFFT_PASS2_VARIANT=$V timeout 300 python bench.py --steps 60 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab_$V.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_$V.json')); print('variant $V', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['per_pass_ms'].items()})"
done
