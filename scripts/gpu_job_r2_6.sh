# launch lists (per-kernel device times) of one type-III (cfg4n inputs) and one 2D (cfg5) exec
set -x
python scripts/profile_type2.py 1 1 3 > gpurun_out/r2_plain3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_t3.csv python scripts/profile_type2.py 1 1 3 > gpurun_out/r2_ncu3.log 2>&1
echo "ncu rc=$?"
