#!/bin/bash
# A/B of batched config-2 cells and config 5 between a variant build and the
# working tree (run under gpurun; tools only).  usage: tools/ab_cells.sh <rev>
rev=$1
for v in $rev A $rev A; do
  if [ $v = A ]; then L=paper_1012_2547_b200/libmatchb200.so; else L=build/variants/lib_$v.so; fi
  for c in "2 2" "4 2" "2 4" "2 8"; do
    set -- $c
    echo -n "$v cfg2 s=$1 m=$2 "; MB_ENGINE_LIB=$PWD/$L python tools/cell_time.py $1 $2 2>/dev/null | tail -1
  done
  MB_ENGINE_LIB=$PWD/$L python bench.py --workload cfg5 --steps 10 --no-e2e --no-cpu-baseline --no-parity 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg5', d['value'], d['ms_per_step'], [(x['m'], round(x['ms'],4)) for x in d['per_m']])"
done
