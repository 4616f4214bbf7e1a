#!/bin/bash
# A/B: current library vs libtcec_old.so, interleaved, 20 launches each.
rm -f gpurun_out/ab.log
for R in 1 2 3; do
for L in libtcec_old.so libtcec.so; do
  ITERS=20 TCEC_LIB=$PWD/paper_2203_03341_b200/$L timeout 300 python scripts/perf_exp.py >> gpurun_out/ab.log 2>&1
done
done
cat gpurun_out/ab.log
