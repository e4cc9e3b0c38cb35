#!/bin/bash
# Re-measure everything profiles/r2 holds (run under gpurun; outputs in gpurun_out/prof/).
set -x
mkdir -p gpurun_out/prof
O=gpurun_out/prof
python bench.py > $O/bench_cfg4_16GiB.json 2> $O/bench_cfg4.err && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --print-units base \
    --csv --log-file $O/ncu_launches_cfg4_16GiB.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > $O/ncu_l.log 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_arm.json 2> $O/ref.err
for w in cfg2 cfg3b; do python bench.py --workload $w --steps 5 > $O/bench_${w}_batched.json 2> $O/$w.err; done
for w in cfg1 cfg3 cfg5; do python bench.py --workload $w --steps 10 > $O/bench_${w}.json 2> $O/$w.err; done
cap() {  # name kernel-regex skip -- command...
  local name=$1 rx=$2 skip=$3; shift 3
  if timeout 300 "$@" > $O/$name.plain.log 2>&1; then
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $skip -c 1 \
        -f -o /tmp/$name "$@" > $O/$name.ncu.log 2>&1
    { python tools/ncu_summary.py /tmp/$name.ncu-rep; echo; echo "Top CUDA source lines (stall samples):";
      python tools/ncu_lines_cuda.py /tmp/$name.ncu-rep 0 14; echo; echo "Instruction mix:";
      python tools/ncu_mix.py /tmp/$name.ncu-rep 0; } > $O/ncu_full_${name}_summary.txt 2>&1
    rm -f /tmp/$name.ncu-rep $O/$name.ncu.log $O/$name.plain.log
  else
    echo "plain run failed: $name" >> $O/failed.txt
  fi
}
cap scan_aligned_cfg4_2GiB scan_kernel 6 python bench.py --text-bytes 2147483648 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-parity
cap run1_cfg5_a16        scan_kernel 3 python tools/kprof.py cfg5 16 am
cap expand_cfg5_a16      expand_kernel 3 python tools/kprof.py cfg5 16 am
cap expand_s2_m2         expand_kernel 2 python tools/one_search.py 2 2
cap shiftor_k2_s2_m12    scan_kernel 2 python tools/one_search.py 2 12
cap shiftor_k2_s4_m12    scan_kernel 2 python tools/one_search.py 4 12
echo done
