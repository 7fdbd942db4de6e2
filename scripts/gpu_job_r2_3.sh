# round 2 job 3: guards, CLI conformance, drop-in e2e with staged copies, then one ncu --set full
# capture of the two type-II kernels of the benched build
set -x
python -m pytest tests -m gpu -x -q -k "guards or dropin or cli" > gpurun_out/r2_pytest_j3.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r2_pytest_j3.log
paper_1701_04492_b200/_build/bench_dropin 16777216 1e-14 20240 5 1 > gpurun_out/r2_dropin.json 2>&1; cat gpurun_out/r2_dropin.json
python scripts/profile_type2.py 2 2 > gpurun_out/r2_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k2_pass" -s 2 -c 2 -o gpurun_out/r2_prof_type2 python scripts/profile_type2.py 2 2 > gpurun_out/r2_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r2_ncu.log
