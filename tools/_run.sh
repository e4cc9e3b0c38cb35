python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/trace_small.py 1048576 2>/dev/null | grep -v arn | tail -4
python bench.py --workload cfg1 --steps 20 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.load(sys.stdin); print('cfg1', d['value'], d['ms_per_step'], d['parity'])"
python bench.py --workload cfg3 --steps 10 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.load(sys.stdin); print('cfg3', d['value'], d['ms_per_step'], d['parity'])"
free -g | head -2; nproc
