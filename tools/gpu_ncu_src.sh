#!/bin/bash
# ncu --set full with source-level counters of the decode-size kernel (gate, M=32 by default).
mkdir -p gpurun_out
for M in ${MS:-32}; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:salr_linear_kernel -s 2 -c 1 \
  -o gpurun_out/prof_gate${M} -f python tools/profile_linear.py --shape gate --tokens $M --reps 4 > gpurun_out/ncu_full${M}.log 2>&1
done
echo done
