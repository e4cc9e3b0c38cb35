#!/bin/bash
# A/B of the headline bench: builds the library at git revision $1 into
# build/variants/lib_<rev>.so, then (run on the GPU box) alternates it with the
# working-tree library.  usage: tools/ab_bench.sh <rev> build   (here)
#                               tools/ab_bench.sh <rev> run     (under gpurun)
set -e
rev=$1; lib=build/variants/lib_$rev.so
if [ "$2" = build ]; then
  rm -rf /tmp/ab_wt; git worktree add -q /tmp/ab_wt "$rev"
  (cd /tmp/ab_wt/paper_1012_2547_b200/csrc && nvcc -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
     -gencode arch=compute_100a,code=sm_100a -shared -o "$OLDPWD/$lib" engine.cu plan.cpp)
  git worktree remove --force /tmp/ab_wt
  exit 0
fi
for l in $lib paper_1012_2547_b200/libmatchb200.so $lib paper_1012_2547_b200/libmatchb200.so; do
  echo -n "$l "; MB_ENGINE_LIB=$l python bench.py --steps 10 --no-e2e --no-cpu-baseline --no-parity | \
    python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['clocks']['sm_mhz'], [(c['m'], c['ms']) for c in d['per_m']])"
done
