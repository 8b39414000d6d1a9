#!/bin/bash
# GPU parity tests of the in-tree build, then an A/B of ab/libA.so vs ab/libB.so, then timelines.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
SHAPES=${SHAPES:-q,k,o,gate,down} bash tools/ab.sh
for sh in ${TRACE:-gate o}; do
SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/libT.so timeout 120 python tools/trace_linear.py --shape $sh --tokens 32 --graph --launches 2 --detail 2 > gpurun_out/tl_${sh}32.txt 2>&1
done
