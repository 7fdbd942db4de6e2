# one full ncu capture of the type-III inner kernels at cfg4 (N = 2^22): the stacked pass A and one pass B
mkdir -p gpurun_out
python scripts/profile_type2.py 1 1 3 > gpurun_out/r2_t3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k1_pass" -s 20 -c 3 -o gpurun_out/r2_prof_type3 python scripts/profile_type2.py 1 1 3 > gpurun_out/r2_ncu_t3.log 2>&1
echo ncu_rc=$?
tail -2 gpurun_out/r2_ncu_t3.log
