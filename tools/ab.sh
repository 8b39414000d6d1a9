#!/bin/bash
# A/B two library builds (ab/libA.so vs ab/libB.so) on the same box, interleaved.
mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
for rep in 1 2; do for v in ${VARS:-A B}; do
  SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/lib$v.so timeout 300 python tools/bench_linear.py --tokens ${TOKENS:-1,8,32} \
    --shapes ${SHAPES:-q,k,gate,down} --pdl $EXTRA 2>&1 | sed "s/^{/{\"v\": \"$v\", \"rep\": $rep, /" >> gpurun_out/ab.jsonl
done; done
echo done
