#!/bin/bash
# K2 (bit-plane Shift-And) survivor-target tuning on the GPU box (tools only)
for t in -10 -12 -14 -16 -18; do
  MB_K2_LOG2=$t python tools/msigma_sweep.py --sigmas 2,4 --lengths 8,12,16,24,48 --family shiftor > gpurun_out/k2_t$t.jsonl 2> gpurun_out/k2_t$t.err
done
