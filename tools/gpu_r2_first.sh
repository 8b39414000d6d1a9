mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python tools/bench_linear.py --tokens 1,8,32 --shapes q,k,o,gate,down --cublas --pdl > gpurun_out/bl_all.jsonl 2>&1
echo done
