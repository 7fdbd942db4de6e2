set -x
python scripts/profile_multi.py > gpurun_out/r2_pm_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_multi.csv python scripts/profile_multi.py > gpurun_out/r2_pm_ncu.log 2>&1
echo "ncu rc=$?"
