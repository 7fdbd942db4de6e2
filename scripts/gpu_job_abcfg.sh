# A/B of library variants on chosen configurations: gpu_job_abcfg.sh "cur A B" cfg3,cfg4
for rep in 1 2; do
for L in $1; do
  if [ $L = cur ]; then unset NUFFT_B200_LIB; else export NUFFT_B200_LIB=$PWD/_abtest/lib$L.so; fi
  timeout 600 python scripts/bench_configs.py --only $2 --out /tmp/cfg_$L.json > /tmp/cfg_$L.log 2>&1
  python -c "
import json
print('$L', {e['config']: round(e['ms_per_exec'],3) for e in json.load(open('/tmp/cfg_$L.json'))})"
done; done
