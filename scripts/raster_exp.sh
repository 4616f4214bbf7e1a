#!/bin/bash
# Rasterisation group (in 128-row units) vs throughput and DRAM traffic at 16384^3.
rm -f gpurun_out/raster.log
for R in 1 2; do
for G in 2 4 8 12; do
  for V in fp16 tf32; do
    python - $V $G >> gpurun_out/raster.log 2>&1 <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2203_03341_b200 as T
v, g = sys.argv[1], int(sys.argv[2])
s = "corrected3_halfhalf" if v == "fp16" else "corrected3_tf32"
n = 16384
a = torch.rand(n, n, device="cuda") * 2 - 1; b = torch.rand(n, n, device="cuda") * 2 - 1
o = torch.empty(n, n, device="cuda")
for _ in range(3): T.gemm_device(a, b, s, out=o, group_m=g)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(15): T.gemm_device(a, b, s, out=o, group_m=g)
e1.record(); torch.cuda.synchronize()
print(f"{v} group_m={g}: {2*n**3/(e0.elapsed_time(e1)/15)/1e9:.1f} TF/s", flush=True)
PY
  done
done
done
for G in 2 4; do
  timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:tcec_gemm_pair -c 1 \
    python scripts/one_gemm.py fp16 16384 "{\"group_m\":$G}" 1 2>/dev/null | grep -E "dram__|gpu__time|hit_rate" >> gpurun_out/raster.log
done
cat gpurun_out/raster.log
