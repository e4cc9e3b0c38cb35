#!/bin/bash
# Re-measure everything profiles/ holds (run under gpurun; outputs in gpurun_out/prof/).
set -x
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench_cfg4_16GiB.json 2> gpurun_out/prof/bench_cfg4.err && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base \
    --csv --log-file gpurun_out/prof/ncu_launches_cfg4_16GiB.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/prof/ncu_l.log 2>&1
python bench.py --text-bytes 2147483648 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/prof/b2g.json 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"scan_kernel" -s 6 -c 1 -o gpurun_out/prof/ncu_full_scan_cfg4_2GiB \
    python bench.py --text-bytes 2147483648 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/prof/ncu_f.log 2>&1
for w in cfg2 cfg3b; do python bench.py --workload $w --steps 5 > gpurun_out/prof/bench_${w}_batched.json 2> gpurun_out/prof/$w.err; done
for w in cfg1 cfg3 cfg5; do python bench.py --workload $w --steps 10 > gpurun_out/prof/bench_${w}.json 2> gpurun_out/prof/$w.err; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/prof/bench_reference_arm.json 2> gpurun_out/prof/ref.err
python tools/one_cell.py 95 16 0 > /dev/null && ncu --set full --import-source on --clock-control none -k regex:"mp_scan|mpb_scan" -s 1 -c 1 \
    -o gpurun_out/prof/ncu_full_mp_cfg3 python tools/kprof.py cfg2 95 16 > gpurun_out/prof/ncu_mp.log 2>&1
python tools/m_sweep.py 4 > gpurun_out/prof/m_sweep_4GiB.jsonl 2> gpurun_out/prof/m_sweep.err
echo done
