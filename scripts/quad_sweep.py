"""CTA-quad kernel (kernel_variant 5) timing at n^3 against the default."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2203_03341_b200 as T

nn = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
a = torch.rand(nn, nn, device="cuda") * 2 - 1
b = torch.rand(nn, nn, device="cuda") * 2 - 1
out = torch.empty(nn, nn, device="cuda")
for sname in ("corrected3_halfhalf", "corrected3_tf32"):
    for kv in (0, 5, 0, 5):
        f = lambda: T.gemm_device(a, b, sname, out=out, kernel_variant=kv)
        for _ in range(2):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(5):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"n={nn} {sname} kv={kv} {os.environ.get('TCEC_QUAD_N', '')} "
              f"{os.environ.get('TCEC_QUAD_NOLS', '')}: {ms:.2f} ms {2 * nn**3 / ms / 1e9:.1f} TF/s",
              flush=True)
