# Run the default bench with alternative builds of the engine (MB_ENGINE_LIB); tools only.
for v in ${VARIANTS:-A}; do
  if [ $v = A ]; then L=paper_1012_2547_b200/libmatchb200.so; else L=build/variants/lib_$v.so; fi
  MB_ENGINE_LIB=$PWD/$L python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-parity 2>gpurun_out/var_$v.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'], [(x['m'],x['ms']) for x in d['per_m']])"
done
