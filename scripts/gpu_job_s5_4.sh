bash scripts/gpu_job_ab.sh "cur noclob" 2 cfg3,cfg4,cfg5
export NUFFT_B200_LIB=$PWD/_abtest/libnoclob.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q -p no:cacheprovider 2>&1 | tail -2
