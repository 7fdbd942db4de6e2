timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "cfg4" 2>&1 | tail -1
bash scripts/gpu_job_abcfg.sh "cur" cfg4
