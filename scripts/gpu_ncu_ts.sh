#!/bin/bash
# ncu --set full of the smem pair kernel vs the A-from-TMEM kernel (FP16 and TF32, n=8192)
mkdir -p gpurun_out
for V in fp16 tf32; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:tcec_gemm -s 2 -c 1 -o gpurun_out/ts_pair_$V \
    python scripts/one_gemm.py $V 8192 '{}' 3 > gpurun_out/ncu_pair_$V.log 2>&1; echo "pair $V rc=$?"
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:tcec_gemm -s 2 -c 1 -o gpurun_out/ts_ts_$V \
    python scripts/one_gemm.py $V 8192 '{"block_n":192}' 3 > gpurun_out/ncu_ts_$V.log 2>&1; echo "ts $V rc=$?"
done
