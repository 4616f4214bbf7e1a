import os, sys, json
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
for v, ds in (("corrected3_tf32", (32, 64, 128)), ("corrected3_halfhalf", (64, 128, 256))):
    for d in ds:
        for kv in (0, 1):
            cfg = T.MmaConfig(block_k=d)
            for _ in range(2): T.gemm_device(A, B, v, cfg=cfg, out=C, kernel_variant=kv)
            torch.cuda.synchronize(); e0.record()
            for _ in range(3): T.gemm_device(A, B, v, cfg=cfg, out=C, kernel_variant=kv)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 3
            rr = float(torch.linalg.norm(ref - C[rows].double()) / torch.linalg.norm(ref))
            print(json.dumps({"v": v, "drain_k": d, "kernel_variant": kv, "tflops": round(2*n**3/ms/1e9, 1), "relres": rr}), flush=True)
