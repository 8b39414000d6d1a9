#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/stages.jsonl
for st in 4 8 12; do
  python tools/bench_linear.py --tokens 1,32 --shapes gate,down --no-adapters --pdl --stages $st 2>&1 | sed "s/^{/{\"stages\": $st, /" >> gpurun_out/stages.jsonl
done
