#!/bin/bash
# A/B of dense-output workloads between engine builds (run under gpurun; tools only).
# usage: tools/ab_expand.sh <variant>...   (A = working tree)
for v in "$@"; do
  if [ $v = A ]; then L=paper_1012_2547_b200/libmatchb200.so; else L=build/variants/lib_$v.so; fi
  MB_ENGINE_LIB=$PWD/$L python bench.py --workload cfg5 --steps 10 --no-e2e --no-cpu-baseline --no-parity 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg5', d['value'], d['ms_per_step'], [(x['m'], round(x['ms'],4)) for x in d['per_m']])"
  for c in "2 2" "4 2"; do set -- $c; echo -n "$v cfg2 s=$1 m=$2 "; MB_ENGINE_LIB=$PWD/$L python tools/cell_time.py $1 $2 2>/dev/null | tail -1; done
done
