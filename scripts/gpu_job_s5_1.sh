bash scripts/gpu_job_trace.sh p2trace trD
bash scripts/gpu_job_quick.sh edges
