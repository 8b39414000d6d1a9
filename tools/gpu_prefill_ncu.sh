#!/bin/bash
# Kernel list of one prefill-size call (gate 4096x14336, M=2048, dense path): duration, tensor-pipe and DRAM share.
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor.sum \
  --clock-control none -k regex:"tb2_dense|nvjet|gemm|Gemm|cutlass|Cat|sm100" -c 16 --csv --log-file gpurun_out/prefill_kernels.csv \
  python tools/profile_linear.py --shape gate --tokens 2048 --reps 4 > gpurun_out/prefill_ncu.log 2>&1
echo done
