"""Sweep rasterisation group and L2 prefetch for the pair kernel at n^3."""
import os, sys, json, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_03341_b200 as T
n = int(os.environ.get("N", "16384"))
g = torch.Generator(device="cuda"); g.manual_seed(0)
A = torch.rand((n, n), generator=g, device="cuda") * 2 - 1
B = torch.rand((n, n), generator=g, device="cuda") * 2 - 1
C = torch.empty((n, n), device="cuda")
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
for v in ("corrected3_halfhalf", "corrected3_tf32"):
    for gm, pf in itertools.product([2, 4, 6, 8, 12, 2, 4, 6, 8, 12], [0]):
        T.gemm_device(A, B, v, out=C, group_m=gm, prefetch=pf)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            T.gemm_device(A, B, v, out=C, group_m=gm, prefetch=pf)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(json.dumps({"v": v, "group_m": gm, "prefetch": pf, "tflops": round(2 * n ** 3 / ms / 1e9, 1)}), flush=True)
