#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/pfdbg.jsonl
for d in 0 1 8 9; do
  SALR_DEBUG_MODE=$d timeout 300 python tools/bench_linear.py --tokens 2048 --shapes q,gate --pdl 2>&1 | sed "s/^{/{\"dbg\": $d, /" >> gpurun_out/pfdbg.jsonl
done
for d in 0 1 8; do SALR_DEBUG_MODE=$d python tools/trace_prefill.py --shape q --tokens 512 2>&1 | sed -n "1p;10,12p" | sed "s/^/dbg$d /" >> gpurun_out/pfdbg.jsonl; done
