#!/bin/bash
# Quick GPU iteration: tests + per-linear bench (+ optional ncu of one shape).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/bench_linear.py --tokens ${TOKENS:-1,8,32,2048} --shapes ${SHAPES:-q,k,o,gate,down} --cublas > gpurun_out/bench_linear.jsonl 2> gpurun_out/bench_linear.err
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:salr_linear -s 2 -c 1 -o gpurun_out/prof_$NCU python tools/profile_linear.py --shape ${NCU_SHAPE:-gate} --tokens ${NCU_TOKENS:-32} --reps 4 > gpurun_out/ncu_full.log 2>&1
fi
echo done
