set -x
nproc; free -g; ldconfig -p | grep -i fftw; lscpu | head -20
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench0.json 2> gpurun_out/r2_bench0.err
tail -c 3000 gpurun_out/r2_bench0.json
