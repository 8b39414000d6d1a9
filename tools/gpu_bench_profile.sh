#!/bin/bash
# Full bench line + ncu evidence for profiles/ (one gpurun call).
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/nvsmi_pre.csv 2>&1
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
# launch list of the bench workload (1 layer, graph-replayed stack) -- shares, not absolutes
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --layers 1 --no-cpu-baseline --no-cublas --batches 32 > gpurun_out/ncu_launch.log 2>&1
# full capture of the dominant kernel (gate, M=32, adapters)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:salr_linear_kernel -s 2 -c 1 \
  -o gpurun_out/prof_gate32 python tools/profile_linear.py --shape gate --tokens 32 --reps 4 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:salr_linear_kernel -s 2 -c 1 \
  -o gpurun_out/prof_gate1 python tools/profile_linear.py --shape gate --tokens 1 --reps 4 > gpurun_out/ncu_full1.log 2>&1
echo done
