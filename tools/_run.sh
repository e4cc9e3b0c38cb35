python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in "4 2" "2 4" "2 2"; do echo "cfg2 $c"; python tools/kprof.py cfg2 $c 2>/dev/null; done
tools/ab_bench.sh HEAD run
