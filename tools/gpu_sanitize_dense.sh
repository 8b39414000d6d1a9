#!/bin/bash
# compute-sanitizer memcheck of the dense prefill path (salr_tb2_decode + GEMM) and the NM24 decode.
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_linear.py -q -x \
  -k "tb2_dense_decode or (dense_prefill_path and 512 and 16)" > gpurun_out/sanitizer_dense.txt 2>&1
echo done
