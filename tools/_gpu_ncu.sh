mkdir -p gpurun_out/ncu
for spec in "4 32" "2 64" "8 16" "256 16"; do
  set -- $spec
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:scan_kernel -s 2 -c 1 \
     -o gpurun_out/ncu/scan_s$1_m$2 python tools/one_search.py $1 $2 > gpurun_out/ncu/scan_s$1_m$2.log 2>&1
done
