#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_linear.py -x -q --timeout 120 -k "token_counts or llama" > gpurun_out/pt_prefill.log 2>&1; echo "rc=$?" >> gpurun_out/pt_prefill.log
timeout 600 python tools/bench_linear.py --tokens 512,1024,2048 --shapes q,k,gate,down --pdl > gpurun_out/bl_prefill_new.jsonl 2>&1
SALR_NO_PREFILL=1 timeout 600 python tools/bench_linear.py --tokens 512,1024,2048 --shapes q,k,gate,down --pdl > gpurun_out/bl_prefill_old.jsonl 2>&1
echo done
