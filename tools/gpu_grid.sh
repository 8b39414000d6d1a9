#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in 0 1; do
  if [ $v = 1 ]; then export SALR_NO_ALIGNED_GRID=1; fi
  timeout 300 python tools/bench_linear.py --tokens 1,32 --shapes q,k,gate,down --pdl > gpurun_out/bl_grid$v.jsonl 2>&1
done
echo done
