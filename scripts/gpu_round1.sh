#!/bin/bash
# smoke + bench + ncu launch list + ncu full capture of the GEMM kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --variant fp16 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_fp16.log 2>&1; echo "bench16 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-extras > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tcec_gemm -s 1 -c 1 -o gpurun_out/prof_tf32 \
   python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/ncu_tf32.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tcec_gemm -s 1 -c 1 -o gpurun_out/prof_fp16 \
   python bench.py --variant fp16 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/ncu_fp16.log 2>&1; echo "ncu3 rc=$?"
tail -3 gpurun_out/smoke.log; tail -2 gpurun_out/bench.log; tail -2 gpurun_out/bench_fp16.log
