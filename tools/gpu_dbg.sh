#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/dbg.jsonl
for d in 0 8 1 9; do
  SALR_DEBUG_MODE=$d python tools/bench_linear.py --tokens 1,32 --shapes gate,down --no-adapters --pdl 2>&1 | sed "s/^{/{\"dbg\": $d, /" >> gpurun_out/dbg.jsonl
done
