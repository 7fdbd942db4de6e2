for rep in 1 2; do
for lib in A B; do
  export NUFFT_B200_LIB=$PWD/_abtest/lib$lib.so
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-dropin --e2e-steps 2 > /tmp/ab_$lib.json 2>/dev/null
  python - $lib <<'PY'
import json, sys
d = json.loads(open(f"/tmp/ab_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(sys.argv[1], "ms/step %.4f" % d["ms_per_step"], {k: round(v, 4) for k, v in d["roofline"]["per_pass_ms"].items()}, "frac %.4f" % d["roofline"]["transform"]["frac"])
PY
done; done
