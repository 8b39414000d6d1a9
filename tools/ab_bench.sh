#!/bin/bash
# bench.py (stack step) with two library builds on the same box
mkdir -p gpurun_out
for v in ${VARS:-A B}; do
  SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/lib$v.so timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cublas \
    > gpurun_out/ab_bench_$v.json 2> gpurun_out/ab_bench_$v.err
done
echo done
