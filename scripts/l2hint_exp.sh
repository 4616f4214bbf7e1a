#!/bin/bash
rm -f gpurun_out/l2hint.log
for R in 1 2; do
for H in 0 1 2 3 9 6; do
  echo "hint $H" >> gpurun_out/l2hint.log
  TCEC_L2_HINT=$H ITERS=15 timeout 300 python scripts/perf_exp.py >> gpurun_out/l2hint.log 2>&1
done
done
for H in 0 1 2; do
  TCEC_L2_HINT=$H timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:tcec_gemm_pair -c 1 \
    python scripts/one_gemm.py fp16 16384 '{}' 1 2>/dev/null | grep -E "dram__|gpu__time" | sed "s/^/hint $H /" >> gpurun_out/l2hint.log
done
cat gpurun_out/l2hint.log
