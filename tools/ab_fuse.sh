#!/bin/bash
# A/B of list-expansion thresholds on sparse-dense cells (run under gpurun; tools only)
for v in "$@"; do
  if [ $v = A ]; then L=paper_1012_2547_b200/libmatchb200.so; else L=build/variants/lib_$v.so; fi
  for c in "2 8" "4 4" "16 2" "8 2" "32 2"; do set -- $c; echo -n "$v cfg2 s=$1 m=$2 "; MB_ENGINE_LIB=$PWD/$L python tools/cell_time.py $1 $2 2>/dev/null | tail -1; done
done
