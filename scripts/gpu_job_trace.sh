for L in "$@"; do
export NUFFT_B200_LIB=$PWD/_abtest/lib$L.so
echo "== $L"
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-dropin --e2e-steps 1 2>&1 | grep -a "trace" | sort | uniq -c | head -4
done
