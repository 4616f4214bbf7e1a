#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/bench_r1c.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --variant fp16 --no-cpu-baseline > gpurun_out/bench_r1c_fp16.log 2>&1; echo "bench16 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
tail -2 gpurun_out/pytest_gpu4.log; tail -1 gpurun_out/bench_r1c.log; tail -1 gpurun_out/bench_r1c_fp16.log; tail -1 gpurun_out/bench_ref.log
