python scripts/profile_type2.py 0 1 2d > gpurun_out/r2_2d_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k2d_(rows|cols)" -s 0 -c 2 -o gpurun_out/r2_prof_2d python scripts/profile_type2.py 0 1 2d > gpurun_out/r2_ncu_2d.log 2>&1
echo "ncu rc=$?"
