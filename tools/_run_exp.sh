python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in "32 2" "64 2" "95 4" "16 8"; do echo "cfg2 $c"; python tools/kprof.py cfg2 $c 2>/dev/null; done
python bench.py --workload cfg2 --steps 5 > gpurun_out/cfg2.json 2>gpurun_out/cfg2.err
python bench.py --workload cfg3b --steps 5 > gpurun_out/cfg3b.json 2>gpurun_out/cfg3b.err
