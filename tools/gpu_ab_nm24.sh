#!/bin/bash
# A/B library builds (ab/lib<VAR>.so) on 2:4 weights: TB2 vs NM24 per-linear times, interleaved.
mkdir -p gpurun_out
: > gpurun_out/ab_nm24.jsonl
for rep in 1 2; do for v in ${VARS:-Cur P3}; do
  SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/lib$v.so timeout 300 python tools/nm24_perf.py --shapes ${SHAPES:-q,gate,down} \
    --tokens ${TOKENS:-1,32} 2>&1 | sed "s/^{/{\"v\": \"$v\", \"rep\": $rep, /" >> gpurun_out/ab_nm24.jsonl
done; done
echo done
