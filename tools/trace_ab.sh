#!/bin/bash
mkdir -p gpurun_out
for v in A B; do
  echo "######## $v"; SALR_B200_LIB_AB=$PWD/ab/lib$v.so timeout 120 python tools/trace_linear.py --shape gate --tokens 1 --launches 2 --graph --no-adapters --detail 2
done > gpurun_out/trace_ab.txt 2>&1
