for A in 0 256 512 1024 1536 1792; do
  NUFFT_ABLATE=$A NUFFT_TRACE_PASS2=1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2> gpurun_out/trace_$A.txt
  echo "ablate $A: $(grep 'fs S=19' gpurun_out/trace_$A.txt | cut -c1-60)"
  NUFFT_ABLATE=$A timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('   ', {k: round(v,3) for k,v in d['roofline']['per_pass_ms'].items()})"
done
