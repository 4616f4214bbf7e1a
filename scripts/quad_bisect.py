"""Bisect the CTA-quad kernel (kernel_variant 5) on small shapes: one process
per case so a fault does not hide the later ones."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2203_03341_b200 as T

m, n, k, var = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
sname = "corrected3_halfhalf" if var == "fp16" else "corrected3_tf32"
g = torch.Generator(device="cuda")
g.manual_seed(1)
A = torch.rand((m, k), generator=g, device="cuda") * 2 - 1
B = torch.rand((k, n), generator=g, device="cuda") * 2 - 1
ref = T.gemm_device(A, B, sname, kernel_variant=4)
torch.cuda.synchronize()
c = T.gemm_device(A, B, sname, kernel_variant=5)
torch.cuda.synchronize()
print(f"{m}x{n}x{k} {var}: identical={torch.equal(c, ref)} maxdiff={(c - ref).abs().max().item():.3e}",
      flush=True)
if not torch.equal(c, ref):
    d = (c - ref).abs()
    for r0 in range(0, m, 64):
        row = [f"{d[r0:r0 + 64, c0:c0 + 128].max().item():.1e}" for c0 in range(0, n, 128)]
        print(f"  rows {r0:4d}+64 by 128-col blocks:", " ".join(row), flush=True)
