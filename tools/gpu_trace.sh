#!/bin/bash
mkdir -p gpurun_out
for sh in k down; do for m in 1 32; do
  echo "######## $sh M=$m"; timeout 120 python tools/trace_linear.py --shape $sh --tokens $m --launches 2 --graph
done; done > gpurun_out/trace.txt 2>&1
echo done
