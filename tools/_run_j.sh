mkdir -p gpurun_out/j
python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q -m gpu -k "config2 or config3 or batch" > gpurun_out/j/pytest.log 2>&1
tail -3 gpurun_out/j/pytest.log
for d in "8 2" "12 4" "16 8" "24 12" "40 20"; do set -- $d; MB_PASS_DENS_U=$1 MB_PASS_DENS_U_OV=$2 python bench.py --workload cfg2 --steps 5 > gpurun_out/j/cfg2_d$1_$2.json 2> gpurun_out/j/err_$1_$2.txt; done
MB_PASS_DENS_U=16 MB_PASS_DENS_U_OV=8 python -m pytest tests/test_gpu_configs.py -x -q -m gpu -k "config2" > gpurun_out/j/pytest16.log 2>&1
