# A/B two library builds (libnufft_b200_ab.so vs libnufft_b200.so), alternating, short benches
for rep in 1 2 3; do
  for L in ab cur; do
    if [ $L = ab ]; then export NUFFT_B200_LIB=$PWD/paper_1701_04492_b200/libnufft_b200_ab.so; else unset NUFFT_B200_LIB; fi
    timeout 300 python bench.py --steps 60 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$L', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['per_pass_ms'].items()})"
  done
done
