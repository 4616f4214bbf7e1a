#!/bin/bash
rm -f gpurun_out/exp3.log
for L in libtcec.so libtcec_exp16.so libtcec.so libtcec_exp16.so; do
  TCEC_LIB=$PWD/paper_2203_03341_b200/$L timeout 300 python scripts/perf_exp.py >> gpurun_out/exp3.log 2>&1
done
cat gpurun_out/exp3.log
