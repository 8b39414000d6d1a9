#!/bin/bash
# Per-linear timings of several library builds (ab/lib_<ver>.so), same box.
mkdir -p gpurun_out
for rep in 1 2; do for v in ${VERS}; do
  echo "## $v"
  SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/lib_$v.so timeout 200 python tools/bench_linear.py --tokens 1,32 --shapes q,gate,down --pdl --copies 4
done; done > gpurun_out/ab_versions.txt 2>&1
