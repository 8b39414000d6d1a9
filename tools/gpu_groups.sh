#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/groups.jsonl
for rep in 1 2; do for g in 4 2; do
  SALR_DEC_GROUPS=$g timeout 300 python tools/bench_linear.py --tokens 1,8,32 --shapes q,gate,down --pdl 2>&1 | sed "s/^{/{\"g\": $g, /" >> gpurun_out/groups.jsonl
done; done
