#!/bin/bash
# Unit timelines of CTA 0, gate: bitmap (TB2) vs 2:4 (NM24) weights (trace build ab/libT.so).
mkdir -p gpurun_out
for nm in "" "--nm24"; do for t in 1 32; do
  echo "######## nm=$nm M=$t"
  SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/libT.so timeout 120 python tools/trace_units.py --shape gate --tokens $t --units 64 $nm
done; done > gpurun_out/tu.txt 2>&1
echo done
