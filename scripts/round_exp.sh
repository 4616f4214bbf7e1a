#!/bin/bash
# Lock-step rounds inside tiles (persistent kernel, prefetch knob = round length in slices)
for PF in 0 16 8; do
  timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:"tcec_gemm_pers" -c 1 \
    python scripts/one_gemm.py tf32 16384 "{\"kernel_variant\":3,\"prefetch\":$PF}" 1 2>/dev/null | grep -E "dram__|gpu__time" | sed "s/^/round=$PF /"
done
python - <<'PY'
import os, sys, torch
sys.path.insert(0, '.')
import paper_2203_03341_b200 as T
n = 16384
a = torch.rand(n, n, device="cuda") * 2 - 1; b = torch.rand(n, n, device="cuda") * 2 - 1
o = torch.empty(n, n, device="cuda")
ref = T.gemm_device(a, b, "corrected3_tf32", kernel_variant=4)
for sname in ("corrected3_halfhalf", "corrected3_tf32"):
    for rnd in range(3):
        for pf in (0, 16, 8):
            for _ in range(2): T.gemm_device(a, b, sname, out=o, kernel_variant=3, prefetch=pf)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(8): T.gemm_device(a, b, sname, out=o, kernel_variant=3, prefetch=pf)
            e1.record(); torch.cuda.synchronize()
            print(sname, "round", pf, round(2 * n**3 / (e0.elapsed_time(e1) / 8) / 1e9, 1), flush=True)
o2 = T.gemm_device(a, b, "corrected3_tf32", kernel_variant=3, prefetch=8)
print("bit-identical", torch.equal(o2, ref))
PY
