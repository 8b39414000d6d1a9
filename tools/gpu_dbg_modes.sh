#!/bin/bash
# Timing with experiment switches of a debug build: 1 skip decode, 2 skip record
# loads, 8 commit without MMAs, 16 no X tiles (results are wrong by design).
mkdir -p gpurun_out
for v in ${VARS:-New}; do for m in ${MODES:-0 1 8 16 24 9}; do
  echo "## $v dbg=$m"
  SALR_DEBUG_MODE=$m SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/lib$v.so timeout 120 python tools/bench_linear.py --tokens 1,32 --shapes gate --pdl --copies 4 --no-adapters
done; done > gpurun_out/dbg_modes.txt 2>&1
