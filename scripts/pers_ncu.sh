#!/bin/bash
for KVG in "0 8" "3 8" "3 16"; do
  set -- $KVG; KV=$1; G=$2
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"tcec_gemm_p" -c 1 \
    python scripts/one_gemm.py tf32 16384 "{\"kernel_variant\":$KV,\"group_m\":$G}" 1 2>/dev/null | grep -E "dram__|gpu__time|hit_rate" | sed "s/^/kv=$KV g=$G /"
done
