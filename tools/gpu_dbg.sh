#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/dbg.jsonl
for rep in 1 2; do for d in 0 4; do
  SALR_DEBUG_MODE=$d python tools/bench_linear.py --tokens 16,32 --shapes q,k,o --pdl 2>&1 | sed "s/^{/{\"dbg\": $d, /" >> gpurun_out/dbg.jsonl
done; done
