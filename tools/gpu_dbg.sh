#!/bin/bash
# Debug-switch bounds (results are wrong by design): 1 skip decode, 2 skip record loads, 8 skip MMAs
mkdir -p gpurun_out
: > gpurun_out/dbg.jsonl
for d in ${DBGS:-0 1 2 3 8}; do
  SALR_DEBUG_MODE=$d timeout 300 python tools/bench_linear.py --tokens ${TOKENS:-1,32} --shapes ${SHAPES:-o,gate} --pdl 2>&1 | sed "s/^{/{\"dbg\": $d, /" >> gpurun_out/dbg.jsonl
done
echo done
