#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/exp.log
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest rc=$?"
for L in libtcec.so libtcec_exp1.so libtcec_exp2.so libtcec_exp3.so; do
  TCEC_LIB=$PWD/paper_2203_03341_b200/$L timeout 300 python scripts/perf_exp.py >> gpurun_out/exp.log 2>&1
done
tail -3 gpurun_out/pytest_gpu5.log; cat gpurun_out/exp.log
