#!/bin/bash
mkdir -p gpurun_out
for L in libtcec.so libtcec_exp1.so libtcec_exp2.so libtcec_exp3.so; do
  TCEC_LIB=$PWD/paper_2203_03341_b200/$L timeout 300 python scripts/perf_exp.py >> gpurun_out/exp.log 2>&1
done
cat gpurun_out/exp.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tcec_gemm_pair -s 1 -c 1 -o gpurun_out/prof_v2_fp16 \
   env ITERS=1 BNS=256 python scripts/perf_exp.py > /dev/null 2>&1; echo "ncu rc=$?"
