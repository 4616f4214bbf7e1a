#!/bin/bash
# What caps the clock under a sustained GEMM: nvidia-smi power / perf state mid-run.
mkdir -p gpurun_out
nvidia-smi -q -d POWER > gpurun_out/power_idle.txt
for V in tf32 fp16; do
  python scripts/one_gemm.py $V 16384 '{}' 300 > /dev/null 2>&1 &
  P=$!
  sleep 8
  nvidia-smi -q -d POWER,PERFORMANCE,CLOCK > gpurun_out/power_load_$V.txt
  nvidia-smi --query-gpu=clocks.sm,power.draw,power.draw.instant,power.limit,enforced.power.limit,temperature.gpu,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/power_trace_$V.csv &
  Q=$!
  sleep 3
  kill $Q; wait $P
done
python scripts/one_gemm.py tf32 8192 '{}' 1 > /dev/null 2>&1
