#!/bin/bash
# Decoder-group count sweep (debug build ab/libD.so honours SALR_DEC_GROUPS).
mkdir -p gpurun_out
for ng in ${NGS:-2 3 4}; do
  echo "## NG=$ng"
  SALR_DEC_GROUPS=$ng SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/libD.so timeout 200 python tools/bench_linear.py --tokens ${TOKENS:-1,32} --shapes ${SHAPES:-q,gate,down} --pdl --copies 4
done > gpurun_out/ng.txt 2>&1
