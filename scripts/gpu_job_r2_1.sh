# round 2: GPU tests (incl. full-size parity vs the reference), smoke, bench both arms
set -x
export NUFFT_FULLSIZE_RECORD=gpurun_out/r2_fullsize.jsonl
rm -f $NUFFT_FULLSIZE_RECORD
( time python -m pytest tests -m gpu -x -q -rA ) > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"
( time python bench.py --steps 20 --warmup 5 ) > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; echo "bench rc=$?"
( time python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/r2_bench1_ref.json 2> gpurun_out/r2_bench1_ref.err; echo "ref rc=$?"
cat gpurun_out/r2_fullsize.jsonl
tail -c 2500 gpurun_out/r2_bench1.json
