"""Is tcgen05 kind::tf32 blind to the low 13 operand bits?  Compare the default
library with the no-mask build bit for bit, then time both."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2203_03341_b200 as T  # noqa: E402
import paper_2203_03341_b200._native as N  # noqa: E402

res = {}
for lib in ("libtcec.so", "libtcec_nomask.so"):
    N._lib = None
    N.LIB_PATH = os.path.join(os.path.dirname(N.__file__), lib)
    outs = []
    for seed in range(3):
        g = torch.Generator(device="cuda")
        g.manual_seed(seed)
        e = torch.randint(-20, 20, (1024, 2048), generator=g, device="cuda").float()
        A = torch.randn((1024, 2048), generator=g, device="cuda") * torch.exp2(e)
        B = torch.randn((2048, 768), generator=g, device="cuda")
        for rnd in ("rna", "rn", "rz"):
            outs.append(T.gemm_device(A, B, T.corrected3(T.tf32tf32(T.RoundingMode(rnd)))).cpu())
    res[lib] = outs
    n = 16384
    A = torch.rand((n, n), device="cuda")
    B = torch.rand((n, n), device="cuda")
    C = torch.empty((n, n), device="cuda")
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        T.gemm_device(A, B, "corrected3_tf32", out=C)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        T.gemm_device(A, B, "corrected3_tf32", out=C)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"lib": lib, "tf32_tflops": 2 * n ** 3 / (e0.elapsed_time(e1) / 5) / 1e9}),
          flush=True)
    del A, B, C
eq = all(torch.equal(a.view(torch.int32), b.view(torch.int32))
         for a, b in zip(res["libtcec.so"], res["libtcec_nomask.so"]))
print(json.dumps({"bitwise_equal": eq}))
