"""Drain interval of the main-term partial: throughput and accuracy vs FP64 at
16384^3 with the default kernel selection (2 interleaved rounds), from the
reference's own schedule (block_k = 16 FP16 / 8 TF32: one MMA k-step) up."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_03341_b200 as T
n = 16384
g = torch.Generator(device="cuda"); g.manual_seed(0)
A = torch.rand((n, n), generator=g, device="cuda") * 2 - 1
B = torch.rand((n, n), generator=g, device="cuda") * 2 - 1
C = torch.empty((n, n), device="cuda")
rows = torch.arange(0, n, 64, device="cuda")
torch.backends.cuda.matmul.allow_tf32 = False
ref = A[rows].double() @ B.double()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
for v, ds in (("corrected3_tf32", (8, 16, 32, 64, 128)), ("corrected3_halfhalf", (16, 32, 64, 128, 256))):
    for rnd in range(2):
        for d in ds:
            for _ in range(2): T.gemm_device(A, B, v, out=C, drain_k=d)
            torch.cuda.synchronize(); e0.record()
            for _ in range(5): T.gemm_device(A, B, v, out=C, drain_k=d)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            rr = float(torch.linalg.norm(ref - C[rows].double()) / torch.linalg.norm(ref))
            print(json.dumps({"v": v, "drain_k": d, "tflops": round(2*n**3/ms/1e9, 1), "relres": rr}), flush=True)
