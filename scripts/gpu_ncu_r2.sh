#!/bin/bash
# Round-2 profiles of the default build: launch list of the bench command
# (TF32-TCEC on ExpRand(-50,50), the headline) and ncu --set full of the
# default persistent kernel for the TF32 headline and FP16, plus the FP16
# split-once GEMM, all at 16384^3.
mkdir -p gpurun_out/ncu2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu2/launches_r02.csv \
   python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extras > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tcec_gemm_pers -s 2 -c 1 -o gpurun_out/ncu2/r02_pers_tf32 \
   python scripts/one_gemm.py tf32 16384 '{}' 3 exprand:-50,50 > /dev/null 2>&1; echo "pers tf32 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tcec_gemm_pers -s 2 -c 1 -o gpurun_out/ncu2/r02_pers_fp16 \
   python scripts/one_gemm.py fp16 16384 '{}' 3 urand > /dev/null 2>&1; echo "pers fp16 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tcec_gemm_ps -s 2 -c 1 -o gpurun_out/ncu2/r02_splitonce_fp16 \
   python scripts/one_gemm.py fp16 16384 '{"split_mode": 2}' 3 urand > /dev/null 2>&1; echo "ps fp16 rc=$?"
