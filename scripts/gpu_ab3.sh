#!/bin/bash
# A/B current vs HEAD library on the default path and the per-tile kernel, interleaved.
rm -f gpurun_out/ab3.log
for R in 1 2 3; do
for L in libtcec_old.so libtcec.so; do
  for KV in 0 4; do
    echo -n "kv=$KV " >> gpurun_out/ab3.log
    KV=$KV ITERS=15 TCEC_LIB=$PWD/paper_2203_03341_b200/$L timeout 120 python scripts/perf_exp.py >> gpurun_out/ab3.log 2>&1
  done
done
done
cat gpurun_out/ab3.log
