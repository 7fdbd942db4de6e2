# pass-2 ablation floors (NUFFT_ABLATE bits: 1 no sample math, 2 no FFT, 4 no Y loads)
mkdir -p gpurun_out
for A in 0 1 2 4 3 5 6 7; do
  NUFFT_ABLATE=$A NUFFT_PASS2_CONT=${CONT:-0} timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/abl_$A.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/abl_$A.json')); print('ablate $A', {k: round(v,3) for k,v in d['roofline']['per_pass_ms'].items()})"
done
