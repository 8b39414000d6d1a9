#!/bin/bash
# Per-linear timings of alternative builds of the library (ab/lib<VAR>.so).
mkdir -p gpurun_out
for v in ${VARS}; do
  echo "## $v"
  SALR_DEBUG_MODE=${DBG:-0} SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/lib$v.so timeout 120 python tools/bench_linear.py --tokens ${TOKENS:-1,32} --shapes ${SHAPES:-q,gate} --pdl --copies 4 ${EXTRA}
done > gpurun_out/ab_lib.txt 2>&1
