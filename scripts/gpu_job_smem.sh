for E in 0 16 32 48 72; do
  NUFFT_FS_EXTRA_SMEM=$E timeout 300 python bench.py --steps 40 --warmup 3 --no-cpu-baseline --e2e-steps 1 --e2e-batch 1 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('extra $E KB', {k: round(v,3) for k,v in d['roofline']['per_pass_ms'].items()})"
done
