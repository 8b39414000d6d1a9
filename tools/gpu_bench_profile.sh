#!/bin/bash
# Full bench line + ncu evidence for profiles/ (one gpurun call).
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps ${REF_STEPS:-5} --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python tools/bench_linear.py --tokens 1,8,32 --shapes q,k,o,gate,down --cublas --pdl > gpurun_out/bl_all.jsonl 2>&1
# launch list of our kernels in the bench workload (1 layer) -- shares, not absolutes
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"salr_|adapter_u" -c 200 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --layers 1 --no-cpu-baseline --no-cublas --batches 32 > gpurun_out/ncu_launch.log 2>&1
# full capture of the bench's dominant launch (gate|up, M=32), gate at M=32/1 and the prefill kernel
timeout 900 ncu --set full --clock-control none --import-source on -k regex:salr_linear_kernel -s 2 -c 1 \
  -o gpurun_out/prof_gateup32 python tools/profile_linear.py --shape gateup --tokens 32 --reps 4 > gpurun_out/ncu_fullgu.log 2>&1
if [ -n "$PREFILL_NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:salr_prefill_kernel -s 1 -c 1 \
  -o gpurun_out/prof_prefill_gate2048 python tools/profile_linear.py --shape gate --tokens 2048 --reps 3 > gpurun_out/ncu_fullpf.log 2>&1
fi
timeout 900 ncu --set full --clock-control none --import-source on -k regex:salr_linear_kernel -s 2 -c 1 \
  -o gpurun_out/prof_gate32 python tools/profile_linear.py --shape gate --tokens 32 --reps 4 > gpurun_out/ncu_full.log 2>&1
timeout 300 python tools/nm24_perf.py > gpurun_out/nm24_perf.jsonl 2>&1
echo done
