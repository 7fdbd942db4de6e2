# build + run one microbenchmark source on the GPU box: gpu_job_mb.sh <name> (scripts/<name>.cu)
set -x
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -o /tmp/$1 scripts/$1.cu && /tmp/$1 > gpurun_out/$1.txt 2>&1
cat gpurun_out/$1.txt
