"""A-from-TMEM pair kernel (block_n=192): bit-identity vs the smem pair kernel
(block_n=256) on ragged shapes, oracle spot check, then timing at large n."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2203_03341_b200 as T
from oracle import oracle as O

SCH = (("corrected3_halfhalf", "fp16", 16, 128), ("corrected3_tf32", "tf32", 8, 64))
ok = True
for (m, n, k) in ((256, 192, 64), (256, 192, 128), (300, 200, 1000), (512, 576, 2048),
                  (1000, 1000, 777), (2048, 2048, 4096)):
    g = torch.Generator().manual_seed(m + n + k)
    a = (torch.rand(m, k, generator=g) * 2 - 1).cuda()
    b = (torch.rand(k, n, generator=g) * 2 - 1).cuda()
    for sname, name, bk, d in SCH:
        f1 = torch.zeros(1, dtype=torch.int32, device="cuda")
        f2 = torch.zeros(1, dtype=torch.int32, device="cuda")
        c256 = T.gemm_device(a, b, sname, block_n=256, flags=f1)
        c192 = T.gemm_device(a, b, sname, block_n=192, flags=f2)
        torch.cuda.synchronize()
        same = torch.equal(c256, c192)
        diff = (c256 - c192).abs().max().item()
        line = f"{m}x{n}x{k} {name}: bit-identical={same} maxdiff={diff:.3e} flags={f1.item()},{f2.item()}"
        if m * n * k <= 2**22:
            oc, _ = O.corrected3(a.cpu().numpy(), b.cpu().numpy(), name, block_k=bk, drain_k=d)
            line += f" vs-oracle={T.relative_residual(c192.cpu().numpy(), oc):.3e}"
        print(line, flush=True)
        ok &= same

if not ok:
    print("MISMATCH: skipping timing")
    sys.exit(1)

def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

for nn in (8192, 16384):
    a = torch.rand(nn, nn, device="cuda") * 2 - 1
    b = torch.rand(nn, nn, device="cuda") * 2 - 1
    out = torch.empty(nn, nn, device="cuda")
    for sname, name, _, _ in SCH:
        for bn in (256, 192):
            ms = timeit(lambda: T.gemm_device(a, b, sname, block_n=bn, out=out), reps=5 if nn > 8192 else 10)
            print(f"n={nn} {name} block_n={bn}: {ms:.2f} ms  {2*nn**3/ms/1e9:.1f} TF/s", flush=True)
