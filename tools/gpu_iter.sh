#!/bin/bash
# iterate: gpu tests, graph-timed per-linear bench (with / without PDL), stack bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/bench_linear.py --tokens ${TOKENS:-1,32} --shapes ${SHAPES:-q,k,gate,down} --no-adapters > gpurun_out/bl_noad.jsonl 2>&1
timeout 300 python tools/bench_linear.py --tokens ${TOKENS:-1,32} --shapes ${SHAPES:-q,k,gate,down} --no-adapters --pdl > gpurun_out/bl_noad_pdl.jsonl 2>&1
timeout 300 python tools/bench_linear.py --tokens ${TOKENS:-1,32} --shapes ${SHAPES:-q,k,gate,down} --cublas --pdl > gpurun_out/bl_ad_pdl.jsonl 2>&1
if [ -n "$BENCH" ]; then timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; fi
echo done
