import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_03341_b200 as T
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
for (m, n) in ((8192, 8192),):
    for k in (512, 1024, 2048, 4096, 8192, 16384):
        A = torch.rand((m, k), device="cuda"); B = torch.rand((k, n), device="cuda"); C = torch.empty((m, n), device="cuda")
        out = {"m": m, "n": n, "k": k}
        for v in ("corrected3_halfhalf", "corrected3_tf32"):
            for _ in range(3): T.gemm_device(A, B, v, out=C)
            torch.cuda.synchronize(); e0.record()
            for _ in range(10): T.gemm_device(A, B, v, out=C)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            out[v] = round(2 * m * n * k / ms / 1e9, 1)
        print(json.dumps(out), flush=True)
