#!/bin/bash
# timing experiments: normal, skip-decode, skip-loads
mkdir -p gpurun_out
for m in 0 1 2 3; do
  SALR_DEBUG_MODE=$m timeout 300 python tools/bench_linear.py --tokens ${TOKENS:-1,32} --shapes ${SHAPES:-q,k,gate,down} $EXTRA > gpurun_out/exp_$m.jsonl 2>&1
done
timeout 300 python tools/bench_linear.py --tokens ${TOKENS:-1,32} --shapes ${SHAPES:-q,k,gate,down} --cublas --no-adapters > gpurun_out/exp_noad.jsonl 2>&1
echo done
