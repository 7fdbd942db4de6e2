timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -2
bash scripts/gpu_job_ab.sh "cur sw0" 2
