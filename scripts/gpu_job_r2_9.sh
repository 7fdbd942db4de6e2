set -x
mkdir -p /tmp/ab
python scripts/ab_split.py A /tmp/ab
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-dropin --e2e-steps 2 > /tmp/b.json 2>/dev/null
python - <<'PY'
import json
d = json.loads(open("/tmp/b.json").read().strip().splitlines()[-1])
print("bench ms/step %.4f" % d["ms_per_step"], {k: round(v, 4) for k, v in d["roofline"]["per_pass_ms"].items()}, "frac %.4f" % d["roofline"]["transform"]["frac"])
PY
python -m pytest tests -m gpu -x -q -k "type1 or type3 or adjoint or g2 or 2048 or pow2 or guards" > /tmp/pt.log 2>&1; echo "pytest rc=$?"; tail -3 /tmp/pt.log
