#!/bin/bash
mkdir -p gpurun_out
for sh in k; do for m in 1 32; do for ad in "" "--no-adapters"; do
  echo "######## $sh M=$m $ad"; timeout 120 python tools/trace_linear.py --shape $sh --tokens $m --launches 2 --graph $ad --detail 3
done; done; done > gpurun_out/trace.txt 2>&1
echo done
