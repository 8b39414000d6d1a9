#!/bin/bash
mkdir -p gpurun_out
for v in ${VARS:-B}; do for ad in ${ADS:---no-adapters}; do
  echo "######## $v $ad"; SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/lib$v.so timeout 120 python tools/trace_linear.py --shape ${SHAPE:-gate} --tokens ${TOK:-1} --launches 2 --graph $ad --detail 2
done; done > gpurun_out/trace_ab.txt 2>&1
