"""kernel_variant 6 (split shared through the L2 ring) vs the default fused
kernel: bit-identity on ragged / wide-range shapes, then interleaved timing at
16384^3 (CUDA events, 10 launches after 3 warm-ups)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2203_03341_b200 as T  # noqa: E402

g = torch.Generator(device="cuda")
g.manual_seed(3)


def rnd(m, k, wide=False):
    x = torch.rand((m, k), generator=g, device="cuda") * 2 - 1
    if wide:
        e = torch.randint(-20, 14, (m, k), generator=g, device="cuda").float()
        x = x * torch.exp2(e)
    return x


shapes = [(4096, 4096, 1024), (2560, 3000, 777), (4100, 4500, 520), (8192, 8192, 2048),
          (300, 20000, 200), (20000, 600, 333)]
ok = True
for (m, n, k) in shapes:
    for wide in (False, True):
        A, B = rnd(m, k, wide), rnd(k, n, wide)
        for name in ("corrected3_halfhalf", "corrected3_tf32"):
            f0 = torch.zeros(1, dtype=torch.int32, device="cuda")
            f6 = torch.zeros(1, dtype=torch.int32, device="cuda")
            c0 = T.gemm_device(A, B, name, flags=f0, kernel_variant=4)
            c6 = T.gemm_device(A, B, name, flags=f6, kernel_variant=6)
            torch.cuda.synchronize()
            same = torch.equal(c0.view(torch.int32), c6.view(torch.int32))
            ok &= same and int(f0.item()) == int(f6.item())
            print(json.dumps({"m": m, "n": n, "k": k, "wide": wide, "scheme": name,
                              "bit_identical": same, "flags": [int(f0.item()), int(f6.item())]}),
                  flush=True)
print("ALL_IDENTICAL", ok, flush=True)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A, B = rnd(n, n), rnd(n, n)
C = torch.empty((n, n), device="cuda")
for rep in range(2):
    for name in ("corrected3_halfhalf", "corrected3_tf32"):
        for kv in ((0, 6) if rep == 0 else (6, 0)):
            for _ in range(3):
                T.gemm_device(A, B, name, out=C, kernel_variant=kv)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                T.gemm_device(A, B, name, out=C, kernel_variant=kv)
            e1.record()
            torch.cuda.synchronize()
            print(json.dumps({"n": n, "scheme": name, "kernel_variant": kv,
                              "tflops": round(2 * n ** 3 / (e0.elapsed_time(e1) / 10) / 1e9, 1)}),
                  flush=True)
