python scripts/profile_type2.py 1 1 1 > gpurun_out/r2_t1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k1_pass" -s 2 -c 2 -o gpurun_out/r2_prof_type1 python scripts/profile_type2.py 1 1 1 > gpurun_out/r2_ncu_t1.log 2>&1
echo "ncu rc=$?"
