#!/bin/bash
# Decoder-group count x ring depth sweep on a debug build (SALR_DEC_GROUPS honoured only there).
mkdir -p gpurun_out
for v in ${VARS:-New}; do for ng in 1 2 4; do for st in 8 12 16; do
  echo "## $v NG=$ng stages=$st"
  SALR_DEC_GROUPS=$ng SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/lib$v.so timeout 120 python tools/bench_linear.py --tokens 1,32 --shapes gate --stages $st --pdl --copies 4
done; done; done > gpurun_out/sweep_ng.txt 2>&1
