"""Compare pair-kernel option sets: bit-identity vs the default on ragged
shapes, then device timing at large n (CUDA events, after warm-up).
usage: variant_check.py '<json list of kwargs dicts>' [sizes]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2203_03341_b200 as T

variants = json.loads(sys.argv[1])
sizes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8192, 16384]
SCH = (("corrected3_halfhalf", "fp16"), ("corrected3_tf32", "tf32"))
ok = True
for (m, n, k) in ((256, 192, 64), (300, 200, 1000), (512, 576, 2048), (1000, 1000, 777)):
    g = torch.Generator().manual_seed(m + n + k)
    a = (torch.rand(m, k, generator=g) * 2 - 1).cuda()
    b = (torch.rand(k, n, generator=g) * 2 - 1).cuda()
    for sname, name in SCH:
        ref = T.gemm_device(a, b, sname)
        for kw in variants:
            kw = {kk: vv for kk, vv in kw.items() if not (kk == "drain_k" and isinstance(vv, dict))}
            c = T.gemm_device(a, b, sname, **{kk: (vv[name] if isinstance(vv, dict) else vv) for kk, vv in kw.items()})
            torch.cuda.synchronize()
            same = torch.equal(ref, c)
            if "drain_k" not in kw:
                ok &= same
            print(f"{m}x{n}x{k} {name} {kw}: bit-identical={same} maxdiff={(ref-c).abs().max().item():.3e}", flush=True)
if not ok:
    print("MISMATCH")
    sys.exit(1)


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


for nn in sizes:
    a = torch.rand(nn, nn, device="cuda") * 2 - 1
    b = torch.rand(nn, nn, device="cuda") * 2 - 1
    out = torch.empty(nn, nn, device="cuda")
    for sname, name in SCH:
      for rnd in range(2):
        for kw in [{}] + variants:
            kw2 = {kk: (vv[name] if isinstance(vv, dict) else vv) for kk, vv in kw.items()}
            ms = timeit(lambda: T.gemm_device(a, b, sname, out=out, **kw2), 5 if nn > 8192 else 10)
            print(f"n={nn} {name} {kw2}: {ms:.2f} ms  {2*nn**3/ms/1e9:.1f} TF/s", flush=True)
