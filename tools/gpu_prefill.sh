#!/bin/bash
mkdir -p gpurun_out
timeout 180 python -m pytest tests/test_gpu_linear.py -x -q --timeout 60 -k "prefill or llama" -s > gpurun_out/pt_prefill.log 2>&1; echo "rc=$?" >> gpurun_out/pt_prefill.log
timeout 300 python tools/bench_linear.py --tokens 512,2048 --shapes q,k,gate,down --pdl --cublas > gpurun_out/bl_prefill_new.jsonl 2>&1
SALR_NO_MULTICAST=1 timeout 300 python tools/bench_linear.py --tokens 512,2048 --shapes q,gate,down --pdl > gpurun_out/bl_prefill_old.jsonl 2>&1
echo done
