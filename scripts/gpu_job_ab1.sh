# A/B the pass-1 organizations (NUFFT_PASS1_VARIANT) with a short bench each
mkdir -p gpurun_out
for V in ${VARIANTS:-0 1}; do
  NUFFT_PASS1_VARIANT=$V timeout 300 python bench.py --steps 60 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab1_$V.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab1_$V.json')); print('p1 variant $V', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['per_pass_ms'].items()})"
done
