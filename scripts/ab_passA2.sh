for rep in 1 2; do
for lib in A B; do
  export NUFFT_B200_LIB=$PWD/_abtest/lib$lib.so
  python scripts/bench_configs.py --only cfg3,cfg2adj,cfg4 > /tmp/c_$lib.log 2>&1
  echo $lib; grep -o '"config": "[a-z0-9]*".*"ms_per_exec": [0-9.]*' /tmp/c_$lib.log | sed 's/"workload.*"points"//'
done; done
