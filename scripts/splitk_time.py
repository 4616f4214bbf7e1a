"""Split-K (opts.split_k) timing against the single-pass default: small
squares and the k-heavy BASELINE config 4(ii)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2203_03341_b200 as T

for (m, n, k) in ((1024, 1024, 1024), (1536, 1536, 1536), (2048, 2048, 2048), (2048, 2048, 65536),
                  (1024, 1024, 16384)):
    a = torch.rand(m, k, device="cuda") * 2 - 1
    b = torch.rand(k, n, device="cuda") * 2 - 1
    out = torch.empty(m, n, device="cuda")
    for sname in ("corrected3_halfhalf", "corrected3_tf32"):
        for sk in (0, 2, 3, 4, 6, 8):
            f = lambda: T.gemm_device(a, b, sname, out=out, split_k=sk)
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            reps = 20 if k <= 2048 else 5
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(reps):
                f()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            print(f"{m}x{n}x{k} {sname} split_k={sk}: {ms:.3f} ms {2 * m * n * k / ms / 1e9:.1f} TF/s",
                  flush=True)
