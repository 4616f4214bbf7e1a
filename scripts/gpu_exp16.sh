#!/bin/bash
# Half-split ablation (TCEC_EXP=16) vs the real kernel vs no staging at all (12), interleaved.
rm -f gpurun_out/exp16.log
for R in 1 2; do
for L in libtcec.so libtcec_exp32.so libtcec_exp16.so; do
  ITERS=20 TCEC_LIB=$PWD/paper_2203_03341_b200/$L timeout 300 python scripts/perf_exp.py >> gpurun_out/exp16.log 2>&1
done
done
cat gpurun_out/exp16.log
