#!/bin/bash
# ring-depth experiment + timelines of cluster-path linears
mkdir -p gpurun_out
: > gpurun_out/stages.jsonl
for st in 0 12 16; do
  timeout 300 python tools/bench_linear.py --tokens 1,32 --shapes q,o,gate,down --pdl --stages $st 2>&1 | sed "s/^{/{\"stages\": $st, /" >> gpurun_out/stages.jsonl
done
for sh in o down; do
SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/libT.so timeout 120 python tools/trace_linear.py --shape $sh --tokens 32 --graph --launches 2 --detail 2 > gpurun_out/tl_${sh}32.txt 2>&1
SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/libT.so timeout 120 python tools/trace_units.py --shape $sh --tokens 32 > gpurun_out/tu_${sh}32.txt 2>&1
done
SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/libT.so timeout 120 python tools/trace_units.py --shape gate --tokens 32 > gpurun_out/tu_gate32.txt 2>&1
echo done
