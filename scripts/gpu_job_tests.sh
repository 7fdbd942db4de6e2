# GPU test pass: full -m gpu suite (parity, API, large-N, reference-suite conformance)
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf 2>&1 | tail -40
for t in fft special lowrank oracle transforms transform2d; do echo "== conf_$t"; ./oracle/_ref/conf_$t 2>&1 | grep -E "FAILED|tests," ; done
