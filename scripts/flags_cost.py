"""Cost of the RunFlags reduction inside the GEMM at 16384^3: gemm_device with
and without a flags tensor (the designated CTAs fold their inputs into the
flags word), interleaved, CUDA events."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_03341_b200 as T
n = int(os.environ.get("FC_N", "16384"))
g = torch.Generator(device="cuda"); g.manual_seed(1)
A = torch.rand((n, n), generator=g, device="cuda") * 2 - 1
B = torch.rand((n, n), generator=g, device="cuda") * 2 - 1
C = torch.empty((n, n), device="cuda")
fl = torch.zeros(1, dtype=torch.int32, device="cuda")
for rnd in range(2):
    for name in ("corrected3_tf32", "corrected3_halfhalf"):
        for use in (False, True):
            kw = {"flags": fl} if use else {}
            for _ in range(3): T.gemm_device(A, B, name, out=C, **kw)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10): T.gemm_device(A, B, name, out=C, **kw)
            e1.record(); torch.cuda.synchronize()
            print(json.dumps({"scheme": name, "flags": use, "tflops": round(2 * n ** 3 / (e0.elapsed_time(e1) / 10) / 1e9, 1)}), flush=True)
