#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/bench_linear.py --tokens ${TOKENS:-1,32} --shapes ${SHAPES:-q,k,gate,down} --no-adapters --pdl > gpurun_out/bl_noad_pdl.jsonl 2>&1
timeout 300 python tools/bench_linear.py --tokens ${TOKENS:-1,32} --shapes ${SHAPES:-q,k,gate,down} --pdl > gpurun_out/bl_ad_pdl.jsonl 2>&1
echo done
