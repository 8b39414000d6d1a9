#!/bin/bash
# One gpurun call: GPU tests, per-linear bench vs cuBLAS, bench.py, ncu launch list.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/bench_linear.py --tokens 1,8,32,2048 --shapes q,k,o,gate,down --cublas > gpurun_out/bench_linear.jsonl 2> gpurun_out/bench_linear.err
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python tools/profile_linear.py --shape gate --tokens 32 --reps 5 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:salr_linear -s 2 -c 1 -o gpurun_out/prof_gate32 python tools/profile_linear.py --shape gate --tokens 32 --reps 4 > gpurun_out/ncu_full.log 2>&1
echo done
