#!/bin/bash
# A/B of the duplicate-heavy config-2 cells (replicate_kernel) between a variant
# build and the working tree (run under gpurun; tools only).  usage: tools/ab_repl.sh <rev>
rev=$1
for v in $rev A $rev A; do
  if [ $v = A ]; then L=paper_1012_2547_b200/libmatchb200.so; else L=build/variants/lib_$v.so; fi
  for c in "2 2" "2 4" "4 2" "2 8" "4 4" "16 2"; do
    set -- $c
    echo -n "$v cfg2 s=$1 m=$2 "; MB_ENGINE_LIB=$PWD/$L python tools/cell_time.py $1 $2 2>/dev/null | tail -1
  done
done
