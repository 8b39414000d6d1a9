#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck of one small fused-linear
# launch per compute format (TB2 bitmap records, NM24 2:4 records) -- evidence under profiles/.
mkdir -p gpurun_out
for fmt in "" "--nm24"; do
for tool in memcheck racecheck synccheck; do
  echo "### $tool (salr_linear, q 4096x4096, M=8, adapters${fmt:+, NM24 2:4 weights})"
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 python tools/profile_linear.py --shape q --tokens 8 --reps 1 $fmt 2>&1 | head -40
done
done > gpurun_out/sanitizer.txt 2>&1
echo done
