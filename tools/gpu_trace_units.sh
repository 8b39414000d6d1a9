#!/bin/bash
# Per-unit pipeline timeline of CTA 0 (unit-trace debug build ab/lib<VAR>.so).
mkdir -p gpurun_out
for v in ${VARS:-New}; do for m in ${MODES:-0}; do for t in ${TOKS:-1}; do
  echo "######## $v dbg=$m M=$t"
  SALR_DEBUG_MODE=$m SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/lib$v.so timeout 120 python tools/trace_units.py --shape ${SHAPE:-gate} --tokens $t --units 64 ${EXTRA}
done; done; done > gpurun_out/tu.txt 2>&1
