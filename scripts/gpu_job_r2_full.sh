# round-2 checkpoint: every GPU test, smoke, both bench arms, the launch list and one ncu --set full
# capture of the type-II kernels of this build
set -x
TAG=${TAG:-ck3}
export NUFFT_FULLSIZE_RECORD=gpurun_out/r2_fullsize_${TAG}.jsonl
rm -f $NUFFT_FULLSIZE_RECORD
( time python -m pytest tests -m gpu -q -rf ) > gpurun_out/r2_pytest_${TAG}.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/r2_pytest_${TAG}.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_${TAG}.json 2> gpurun_out/r2_bench_${TAG}.err; echo "bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_bench_ref_${TAG}.json 2> gpurun_out/r2_bench_ref_${TAG}.err; echo "ref rc=$?"
python scripts/bench_configs.py --out gpurun_out/r2_configs_${TAG}.json > gpurun_out/r2_configs_${TAG}.log 2>&1; echo "configs rc=$?"
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-dropin > gpurun_out/r2_launch_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_${TAG}.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-dropin > gpurun_out/r2_ncu_launch.log 2>&1
echo "ncu launches rc=$?"
python scripts/profile_type2.py 2 2 > gpurun_out/r2_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k2_pass" -s 2 -c 2 -o gpurun_out/r2_prof_type2_${TAG} python scripts/profile_type2.py 2 2 > gpurun_out/r2_ncu_${TAG}.log 2>&1
echo "ncu full rc=$?"
