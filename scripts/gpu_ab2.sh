#!/bin/bash
rm -f gpurun_out/ab2.log
for R in 1 2; do
for L in libtcec_old.so libtcec.so; do
  SPLIT_MODE=${SPLIT_MODE:-0} ITERS=20 TCEC_LIB=$PWD/paper_2203_03341_b200/$L timeout 120 python scripts/perf_exp.py >> gpurun_out/ab2.log 2>&1
done
done
cat gpurun_out/ab2.log
