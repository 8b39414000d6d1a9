#!/bin/bash
# iterate: gpu tests, graph-timed per-linear bench (decoder-group variants), trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for g in ${GROUPS_LIST:-4 2 1}; do
  SALR_DEC_GROUPS=$g timeout 300 python tools/bench_linear.py --tokens ${TOKENS:-1,32} --shapes ${SHAPES:-q,k,gate,down} --no-adapters > gpurun_out/bl_noad_g$g.jsonl 2>&1
done
timeout 300 python tools/bench_linear.py --tokens ${TOKENS:-1,32} --shapes ${SHAPES:-q,k,gate,down} --cublas > gpurun_out/bl_ad.jsonl 2>&1
SALR_DEC_GROUPS=${TRACE_G:-4} timeout 120 python tools/trace_linear.py --shape gate --tokens 1 --no-adapters --launches 2 > gpurun_out/trace.txt 2>&1
echo done
