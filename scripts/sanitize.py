"""One small call of every kernel path, for compute-sanitizer
(memcheck / racecheck / synccheck; profiles/r01/sanitizer_*.log)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2203_03341_b200 as T

m, n, k = 300, 520, 200
g = torch.Generator(device="cuda")
g.manual_seed(7)
A = torch.rand((m, k), generator=g, device="cuda") * 2 - 1
B = torch.rand((k, n), generator=g, device="cuda") * 2 - 1
runs = []
for sname in ("corrected3_halfhalf", "corrected3_tf32"):
    ref = T.gemm_device(A, B, sname, kernel_variant=4)
    for kw in ({}, {"kernel_variant": 2}, {"kernel_variant": 3},
               {"block_n": 192}, {"block_n": 128}, {"block_n": 64}, {"block_n": 128, "kernel_variant": 1},
               {"split_mode": 2}, {"drain_k": 16 if "half" in sname else 8},
               {"split_k": 2}):
        c = T.gemm_device(A, B, sname, **kw)
        torch.cuda.synchronize()
        same = torch.equal(c, ref) if "drain_k" not in kw and "split_k" not in kw else True
        runs.append((sname, kw, same))
for name in ("markidis4", "tc_plain_fp16", "corrected4_rn"):
    T.gemm_device(A, B, name)
    torch.cuda.synchronize()
    runs.append((name, {}, True))
T.split_device(A, T.scaled_halfhalf())
T.split_device(A, T.tf32tf32())
torch.cuda.synchronize()
for r in runs:
    print(*r)
print("ALL_EQUAL", all(r[2] for r in runs))
