#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/ps_time.py 8192,16384 2>&1 | tee gpurun_out/ps_time.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ps_launches.csv \
  python scripts/one_gemm.py fp16 16384 '{"split_mode":2}' 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ps_launches_tf32.csv \
  python scripts/one_gemm.py tf32 16384 '{"split_mode":2}' 2 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:tcec_gemm_ps -s 1 -c 1 -o gpurun_out/ps_fp16 \
  python scripts/one_gemm.py fp16 8192 '{"split_mode":2}' 2 > /dev/null 2>&1; echo "ncu rc=$?"
