#!/bin/bash
# A/B/C of ab/libA.so, ab/libB.so, ab/libC.so (interleaved, 2 reps); $C_ENV applies to C
mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
for rep in 1 2; do for v in ${VARS:-A B C}; do
  envs=""
  if [ $v = C ]; then envs="$C_ENV"; fi
  env $envs SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/lib$v.so timeout 300 python tools/bench_linear.py --tokens ${TOKENS:-1,8,32} \
    --shapes ${SHAPES:-q,k,o,gate,down} --pdl $EXTRA 2>&1 | sed "s/^{/{\"v\": \"$v\", \"rep\": $rep, /" >> gpurun_out/ab.jsonl
done; done
echo done
