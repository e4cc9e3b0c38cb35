mkdir -p gpurun_out/n
(time python -m pytest tests -x -q -m gpu) > gpurun_out/n/pytest.log 2>&1
tail -4 gpurun_out/n/pytest.log
python tools/msigma_sweep.py --check > gpurun_out/n/msigma_sweep_1GiB.jsonl 2> gpurun_out/n/msigma1.err
python tools/msigma_sweep.py --gib 4 > gpurun_out/n/msigma_sweep_4GiB.jsonl 2> gpurun_out/n/msigma4.err
for w in cfg2 cfg3b; do python bench.py --workload $w --steps 5 > gpurun_out/n/bench_${w}_batched.json 2> gpurun_out/n/$w.err; done
python bench.py --workload cfg5 --steps 10 > gpurun_out/n/bench_cfg5.json 2> gpurun_out/n/cfg5.err
