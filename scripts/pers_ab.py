"""Persistent pair kernel (kernel_variant=2) vs the default, interleaved, at several shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_03341_b200 as T

def timeit(fn, reps):
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

for (m, n, k) in ((16384, 16384, 16384), (8192, 8192, 8192)):
    a = torch.rand(m, k, device="cuda") * 2 - 1
    b = torch.rand(k, n, device="cuda") * 2 - 1
    out = torch.empty(m, n, device="cuda")
    reps = max(3, int(2e13 / (2 * m * n * k)) + 3)
    for sname, name in (("corrected3_halfhalf", "fp16"), ("corrected3_tf32", "tf32")):
        for rnd in range(3):
            for kv, gm in ((4, 0), (3, 12), (3, 16), (3, 20)):
                ms = timeit(lambda: T.gemm_device(a, b, sname, out=out, kernel_variant=kv, group_m=gm), reps)
                print(f"{m}x{n}x{k} {name} kv={kv} group_m={gm}: {ms:.3f} ms {2*m*n*k/ms/1e9:.1f} TF/s", flush=True)
    del a, b, out
    torch.cuda.empty_cache()
