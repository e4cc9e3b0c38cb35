python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for m in 16 1024; do echo "cfg5 a^$m"; python tools/kprof.py cfg5 $m am 2>/dev/null; done
python bench.py --steps 10 --no-e2e --no-cpu-baseline --no-parity | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], [(c['m'], c['ms']) for c in d['per_m']])"
python bench.py --workload cfg5 --steps 5 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['roofline']['frac'], d['parity'], [(c['m'], c['family'], c['ms'], c['hbm_frac']) for c in d['per_m']])"
