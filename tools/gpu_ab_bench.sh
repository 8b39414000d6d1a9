#!/bin/bash
# A/B library builds (ab/lib<VAR>.so) through the full stack bench (magnitude-pruned weights), interleaved.
mkdir -p gpurun_out
: > gpurun_out/ab_bench.jsonl
for rep in 1 2; do for v in ${VARS:-Cur P3 P3b}; do
  SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/lib$v.so timeout 300 python bench.py --no-cpu-baseline --no-nm24 \
    --no-cublas ${EXTRA} 2>/dev/null | tail -1 | sed "s/^{/{\"v\": \"$v\", \"rep\": $rep, /" >> gpurun_out/ab_bench.jsonl
done; done
echo done
