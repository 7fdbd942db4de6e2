for E in ${EXTRAS:-0 48}; do
  NUFFT_FS_EXTRA_SMEM=$E NUFFT_TRACE_PASS2=1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2> gpurun_out/trace_e$E.txt
  echo "extra $E"; grep "fs S" gpurun_out/trace_e$E.txt | tail -64 | sed -n "${LINES:-15,24p}"
done
