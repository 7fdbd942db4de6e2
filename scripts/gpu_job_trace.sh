export NUFFT_B200_LIB=$PWD/_abtest/lib$1.so
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-dropin --e2e-steps 1 2>&1 | grep -a "trace" | sort | uniq -c | head -20
