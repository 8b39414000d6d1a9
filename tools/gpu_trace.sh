#!/bin/bash
mkdir -p gpurun_out
for m in 3; do
  echo "######## mode $m"; SALR_DEBUG_MODE=$m timeout 120 python tools/trace_linear.py --shape gate --tokens 1 --no-adapters --launches 2
done > gpurun_out/trace.txt 2>&1
echo done
