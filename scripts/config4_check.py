import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_03341_b200 as T
m, n, k = 2048, 2048, 65536
a = torch.rand(m, k, device="cuda") * 2 - 1
b = torch.rand(k, n, device="cuda") * 2 - 1
out = torch.empty(m, n, device="cuda")
for rnd in range(2):
    for sname in ("corrected3_tf32", "corrected3_halfhalf"):
        for kw in ({}, {"kernel_variant": 3}, {"split_k": 8}):
            f = lambda: T.gemm_device(a, b, sname, out=out, **kw)
            for _ in range(3): f()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(20): f()
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            print(f"{sname} {kw}: {ms:.3f} ms {2*m*n*k/ms/1e9:.1f} TF/s", flush=True)
