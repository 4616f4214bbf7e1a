#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv \
   python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > /dev/null 2>&1; echo "ncu launches rc=$?"
for V in tf32 fp16; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tcec_gemm_pair -s 3 -c 1 -o gpurun_out/prof_r1_$V \
   python bench.py --variant $V --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > /dev/null 2>&1; echo "ncu $V rc=$?"
done
