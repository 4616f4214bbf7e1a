"""corrected4_rn (TCEC_SCHEME_INUNIT4_RN) and markidis4 timing at n^3 on device
tensors, by block_k; CUDA events after warm-up."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2203_03341_b200 as T

for nn in (2048, 4096, 8192):
    a = torch.rand(nn, nn, device="cuda") * 2 - 1
    b = torch.rand(nn, nn, device="cuda") * 2 - 1
    out = torch.empty(nn, nn, device="cuda")
    for name, bks in (("markidis4", (16,)), ("corrected4_rn", (16, 32, 64, 128)),
                      ("corrected3_halfhalf", (16,))):
        for bk in bks:
            cfg = T.default_config(T.SCHEMES_BY_NAME[name], block_k=bk)
            f = lambda: T.gemm_device(a, b, name, cfg, out=out)
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(5):
                f()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            print(f"n={nn} {name} block_k={bk}: {ms:.3f} ms {2 * nn**3 / ms / 1e9:.1f} TF/s", flush=True)
