#!/bin/bash
mkdir -p gpurun_out
for g in 4 2 1; do
  SALR_DEC_GROUPS=$g timeout 300 python tools/bench_linear.py --tokens 1,32 --shapes q,gate --no-adapters --pdl > gpurun_out/bl_g$g.jsonl 2>&1
done
echo done
