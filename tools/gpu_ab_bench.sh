#!/bin/bash
# A/B library builds (ab/lib<VAR>.so) through the full stack bench (magnitude-pruned weights), interleaved;
# optional GPU tests of the package build first (TESTS=1).
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
fi
: > gpurun_out/ab_bench.jsonl
for rep in 1 2; do for v in ${VARS:-H X}; do
  SALR_B200_DEBUG=1 SALR_B200_LIB_AB=$PWD/ab/lib$v.so timeout 300 python bench.py --no-cpu-baseline --no-cublas \
    ${EXTRA} 2>/dev/null | tail -1 | sed "s/^{/{\"v\": \"$v\", \"rep\": $rep, /" >> gpurun_out/ab_bench.jsonl
done; done
echo done
