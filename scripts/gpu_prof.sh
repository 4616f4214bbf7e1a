#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tcec_gemm_pair -s 2 -c 1 -o gpurun_out/prof_v2c_fp16 \
   env ITERS=1 BNS=256 N=8192 python scripts/perf_exp.py > /dev/null 2>&1; echo "ncu rc=$?"
