#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/diag_tol.py > gpurun_out/diag_tol.log 2>&1; echo "diag rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_v2.log 2>&1; echo "bench rc=$?"
tail -5 gpurun_out/diag_tol.log; tail -3 gpurun_out/bench_v2.log
