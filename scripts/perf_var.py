"""Time kernel variants at n^3."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_03341_b200 as T
n = int(os.environ.get("N", "16384"))
g = torch.Generator(device="cuda"); g.manual_seed(0)
A = torch.rand((n, n), generator=g, device="cuda") * 2 - 1
B = torch.rand((n, n), generator=g, device="cuda") * 2 - 1
C = torch.empty((n, n), device="cuda")
rows = torch.arange(0, n, 128, device="cuda")
torch.backends.cuda.matmul.allow_tf32 = False
ref = A[rows].double() @ B.double()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
for kv in [int(x) for x in os.environ.get("KVS", "0,1").split(",")]:
    for pf in [int(x) for x in os.environ.get("PFS", "0").split(",")]:
        out = {"kernel_variant": kv, "prefetch": pf}
        for v in ("corrected3_halfhalf", "corrected3_tf32"):
            for _ in range(2): T.gemm_device(A, B, v, out=C, kernel_variant=kv, prefetch=pf)
            torch.cuda.synchronize(); e0.record()
            for _ in range(5): T.gemm_device(A, B, v, out=C, kernel_variant=kv, prefetch=pf)
            e1.record(); torch.cuda.synchronize()
            out[v] = round(2 * n ** 3 / (e0.elapsed_time(e1) / 5) / 1e9, 1)
            out[v + "_relres"] = float(torch.linalg.norm(ref - C[rows].double()) / torch.linalg.norm(ref))
        print(json.dumps(out), flush=True)
