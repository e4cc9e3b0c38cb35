#!/bin/bash
# Round-2 ncu evidence (run under gpurun): one `--set full` capture per kernel
# the r1 review listed as uncaptured, each after the same command has exited 0
# without ncu.  Reports land in gpurun_out/ncu2/ (summarised into profiles/r2/
# by tools/ncu_summary.py here; the .ncu-rep files stay out of git).
mkdir -p gpurun_out/ncu2
O=gpurun_out/ncu2
cap() {  # name kernel-regex skip -- command...
  local name=$1 rx=$2 skip=$3; shift 3
  if timeout 300 "$@" > $O/$name.plain.log 2>&1; then
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $skip -c 1 \
        -f -o /tmp/$name "$@" > $O/$name.ncu.log 2>&1
    # summaries are made on the box (the reports, ~8 MB each, stay there)
    { python tools/ncu_summary.py /tmp/$name.ncu-rep; echo; echo "Top CUDA source lines (stall samples):";
      python tools/ncu_lines_cuda.py /tmp/$name.ncu-rep 0 14; echo; echo "Instruction mix:";
      python tools/ncu_mix.py /tmp/$name.ncu-rep 0; } > $O/ncu_full_${name}_summary.txt 2>&1
    rm -f /tmp/$name.ncu-rep $O/$name.ncu.log $O/$name.plain.log
  else
    echo "plain run failed: $name" >> $O/failed.txt
  fi
}
# single-pattern scans, 1 GiB text: sigma m family
cap win4_s256_m4      scan_kernel 2 python tools/one_search.py 256 4
cap win4e_s256_m5     scan_kernel 2 python tools/one_search.py 256 5
cap swar3_s256_m3     scan_kernel 2 python tools/one_search.py 256 3
cap gram_s4_m32       scan_kernel 2 python tools/one_search.py 4 32
cap shiftor_s4_m32    scan_kernel 2 python tools/one_search.py 4 32 shiftor
cap aligned2_s4_m12   scan_kernel 2 python tools/one_search.py 4 12
cap swar8_s2_m8       scan_kernel 2 python tools/one_search.py 2 8
cap sampled_s256_m1024 sampled_kernel 2 python tools/one_search.py 256 1024
cap offsets_s256_m8   offsets_kernel 2 python tools/one_search.py 256 8
cap expand_s2_m2      expand_kernel 2 python tools/one_search.py 2 2
cap offsets_s2_m2     offsets_kernel 2 python tools/one_search.py 2 2
# batched: config-2 cell sigma=4 m=2 (replicate), sigma=8 m=4 (mpb pass), config 3 m=16 (mp pass)
cap replicate_cfg2_s4_m2 replicate_kernel 2 python tools/kprof.py cfg2 4 2
cap mpb_cfg2_s8_m4       mpb_scan_kernel 2 python tools/kprof.py cfg2 8 4
cap mp_cfg3_m16          mp_scan_kernel 2 python tools/kprof.py cfg2 95 16
ls -la $O
echo done
