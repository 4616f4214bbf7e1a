"""Split-once mode: time the split passes and the GEMM kernel separately
(CUDA events on the current stream; launches through the C ABI)."""
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

for nn in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8192,16384").split(",")]:
    a = torch.rand(nn, nn, device="cuda") * 2 - 1
    b = torch.rand(nn, nn, device="cuda") * 2 - 1
    out = torch.empty(nn, nn, device="cuda")
    for sname, name in (("corrected3_halfhalf", "fp16"), ("corrected3_tf32", "tf32")):
        for rnd in range(3):
            for sm in (0, 2):
                ms = timeit(lambda: T.gemm_device(a, b, sname, out=out, split_mode=sm), 5)
                print(f"n={nn} {name} split_mode={sm}: {ms:.2f} ms {2*nn**3/ms/1e9:.1f} TF/s", flush=True)
