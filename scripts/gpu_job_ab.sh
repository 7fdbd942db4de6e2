# A/B of library variants on the type-II bench: gpu_job_ab.sh "cur A B" [reps] [extra bench_configs --only list]
LIBS=${1:-cur}
REPS=${2:-2}
for rep in $(seq $REPS); do
  for L in $LIBS; do
    if [ $L = cur ]; then unset NUFFT_B200_LIB; else export NUFFT_B200_LIB=$PWD/_abtest/lib$L.so; fi
    timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-dropin --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['roofline']['per_pass_ms'].items()})"
  done
done
if [ -n "$3" ]; then
  for L in $LIBS; do
    if [ $L = cur ]; then unset NUFFT_B200_LIB; else export NUFFT_B200_LIB=$PWD/_abtest/lib$L.so; fi
    timeout 600 python scripts/bench_configs.py --only $3 --out /tmp/cfg_$L.json > /tmp/cfg_$L.log 2>&1
    python -c "
import json
print('$L', {e['config']: round(e['ms_per_exec'],3) for e in json.load(open('/tmp/cfg_$L.json'))})"
  done
fi
unset NUFFT_B200_LIB
