# A/B of two library builds: parity subset on B, then alternating short benches
# usage: bash scripts/gpu_ab.sh "<pytest -k expr>" [reps] [extra bench args]
K=${1:-type2}; REPS=${2:-2}; EXTRA=${3:-}
mkdir -p gpurun_out
export NUFFT_B200_LIB=$PWD/_abtest/libB.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -q -x -k "$K" -p no:cacheprovider 2>&1 | tail -3
for rep in $(seq $REPS); do
for lib in A B; do
  export NUFFT_B200_LIB=$PWD/_abtest/lib$lib.so
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-dropin --e2e-steps 1 $EXTRA > /tmp/ab_$lib.json 2>/tmp/ab_$lib.err || tail -5 /tmp/ab_$lib.err
  python - $lib <<'PY'
import json, sys
d = json.loads(open(f"/tmp/ab_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(sys.argv[1], "ms/step %.4f" % d["ms_per_step"], {k: round(v, 4) for k, v in d["roofline"]["per_pass_ms"].items()}, "frac %.4f" % d["roofline"]["transform"]["frac"], d["clocks"]["sm_mhz"])
PY
done; done
