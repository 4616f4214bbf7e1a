"""Time the TCEC kernel at n^3 for the current library (TCEC_LIB selects a measurement build)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_03341_b200 as T
n = int(os.environ.get("N", "16384"))
SM = int(os.environ.get("SPLIT_MODE", "0"))
KV = int(os.environ.get("KV", "0"))
iters = int(os.environ.get("ITERS", "5"))
g = torch.Generator(device="cuda"); g.manual_seed(0)
A = torch.rand((n, n), generator=g, device="cuda") * 2 - 1
B = torch.rand((n, n), generator=g, device="cuda") * 2 - 1
C = torch.empty((n, n), device="cuda")
out = {"lib": os.path.basename(os.environ.get("TCEC_LIB", "libtcec.so")), "n": n}
for v in ("corrected3_halfhalf", "corrected3_tf32"):
    for bn in [int(x) for x in os.environ.get("BNS", "256").split(",")]:
        for _ in range(2):
            T.gemm_device(A, B, v, out=C, block_n=bn, split_mode=SM, kernel_variant=KV)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            T.gemm_device(A, B, v, out=C, block_n=bn, split_mode=SM, kernel_variant=KV)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        out[f"{v}_bn{bn}_tflops"] = round(2 * n ** 3 / ms / 1e9, 1)
print(json.dumps(out), flush=True)
