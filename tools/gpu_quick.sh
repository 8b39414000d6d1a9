#!/bin/bash
# GPU tests + per-linear timings (quick check after a kernel change).
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/bench_linear.py --tokens ${TOKENS:-1,8,32} --shapes ${SHAPES:-q,k,gate,down} --cublas --pdl > gpurun_out/bl.jsonl 2>&1
echo done
