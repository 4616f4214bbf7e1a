"""Time gemm_device at n^3 for both variants with the given kwargs (json), CUDA events.
usage: time_kv.py n '{"kernel_variant": 6}' [label]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_03341_b200 as T  # noqa: E402

n = int(sys.argv[1])
kw = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
label = sys.argv[3] if len(sys.argv) > 3 else os.path.basename(os.environ.get("TCEC_LIB", "libtcec.so"))
g = torch.Generator(device="cuda")
g.manual_seed(1)
A = torch.rand((n, n), generator=g, device="cuda") * 2 - 1
B = torch.rand((n, n), generator=g, device="cuda") * 2 - 1
C = torch.empty((n, n), device="cuda")
out = {"label": label, "n": n, "kw": kw}
for name in ("corrected3_halfhalf", "corrected3_tf32"):
    for _ in range(3):
        T.gemm_device(A, B, name, out=C, **kw)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        T.gemm_device(A, B, name, out=C, **kw)
    e1.record()
    torch.cuda.synchronize()
    out[name] = round(2 * n ** 3 / (e0.elapsed_time(e1) / 10) / 1e9, 1)
print(json.dumps(out), flush=True)
