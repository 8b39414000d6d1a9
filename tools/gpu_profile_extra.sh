#!/bin/bash
# Second half of the profile evidence (gpurun_out stays under its 64 MiB limit):
# ncu captures of gate M=1 and of the NM24 (2:4) gate M=32 launch, the sparsity/rank sweep, prefill timings.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:salr_linear_kernel -s 2 -c 1 \
  -o gpurun_out/prof_gate1 python tools/profile_linear.py --shape gate --tokens 1 --reps 4 > gpurun_out/ncu_full1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:salr_linear_kernel -s 2 -c 1 \
  -o gpurun_out/prof_nm24_gate32 python tools/profile_linear.py --shape gate --tokens 32 --reps 4 --nm24 > gpurun_out/ncu_fullnm.log 2>&1
timeout 900 python tools/sweep.py --tokens 1,8,32,2048 > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 600 python tools/bench_linear.py --tokens 128,2048 --shapes q,gate,down --cublas --pdl > gpurun_out/bl_prefill.jsonl 2>&1
echo done
