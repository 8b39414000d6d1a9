#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/stages.jsonl
for rep in 1 2; do for st in 12 8; do
  timeout 300 python tools/bench_linear.py --tokens 1,8,32 --shapes q,k,gate,down --pdl --stages $st 2>&1 | sed "s/^{/{\"stages\": $st, /" >> gpurun_out/stages.jsonl
done; done
