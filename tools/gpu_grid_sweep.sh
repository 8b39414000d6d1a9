#!/bin/bash
# Per-linear time vs grid size (explicit num_ctas) at decode batch sizes.
mkdir -p gpurun_out
: > gpurun_out/grid.jsonl
for sh in ${SHAPES:-qkv o gateup down}; do for c in ${CTAS:-0 148 128 112 96 74}; do
  timeout 120 python tools/bench_linear.py --tokens ${TOKENS:-32} --shapes $sh --ctas $c --pdl 2>/dev/null \
    | sed "s/^{/{\"ctas_req\": $c, /" >> gpurun_out/grid.jsonl
done; done
echo done
