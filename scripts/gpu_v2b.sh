#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/diag_tol.py > gpurun_out/diag_tol2.log 2>&1; echo "diag rc=$?"
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x --durations=10 > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_v2b.log 2>&1; echo "bench rc=$?"
grep "bn=256" gpurun_out/diag_tol2.log | grep tf32 | head -12; tail -15 gpurun_out/pytest_gpu2.log; tail -2 gpurun_out/bench_v2b.log
