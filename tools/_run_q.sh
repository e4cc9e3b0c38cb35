mkdir -p gpurun_out/q
MB_ENGINE_LIB=paper_1012_2547_b200/libmatchb200_trace.so python tools/trace_phases.py 67108864 256 16 > gpurun_out/q/trace64.txt 2>&1
python bench.py --workload cfg3 --steps 10 > gpurun_out/q/bench_cfg3.json 2> gpurun_out/q/e3.txt
python bench.py --workload cfg5 --steps 10 > gpurun_out/q/bench_cfg5.json 2> gpurun_out/q/e5.txt
python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/q/pytest.log 2>&1
