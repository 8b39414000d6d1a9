#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/dbg.jsonl
for d in 0 16 64 128 208; do
  SALR_DEBUG_MODE=$d python tools/bench_linear.py --tokens 1,32 --shapes q,gate,down --pdl 2>&1 | sed "s/^{/{\"dbg\": $d, /" >> gpurun_out/dbg.jsonl
done
python tools/bench_linear.py --tokens 1,32 --shapes q,gate,down --pdl --no-adapters 2>&1 | sed "s/^{/{\"dbg\": \"noad\", /" >> gpurun_out/dbg.jsonl
