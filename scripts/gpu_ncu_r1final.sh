#!/bin/bash
# Round-1 final profiles: launch list of the bench command, full captures of the
# default pair kernel (TF32 headline, FP16) and of the split-once kernels at 16384^3.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
   python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > /dev/null 2>&1; echo "launches rc=$?"
for V in tf32 fp16; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tcec_gemm_pers -s 2 -c 1 -o gpurun_out/final_pers_$V \
     python scripts/one_gemm.py $V 16384 '{}' 3 > /dev/null 2>&1; echo "pers $V rc=$?"
done
