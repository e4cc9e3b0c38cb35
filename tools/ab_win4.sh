for v in HEAD A HEAD A; do
  if [ $v = A ]; then L=paper_1012_2547_b200/libmatchb200.so; else L=build/variants/lib_$v.so; fi
  for c in "2 4" "4 4" "16 4" "256 4"; do
    set -- $c
    echo -n "$v cfg2 s=$1 m=$2 "; MB_ENGINE_LIB=$PWD/$L python tools/cell_time.py $1 $2 2>/dev/null | tail -1
  done
done
tools/ab_bench.sh HEAD run
