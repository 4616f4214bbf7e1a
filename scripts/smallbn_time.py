"""Small products by tile width (block_n 64 / 128 / 192 / 256): time (CUDA
events, 20 launches after 5 warm-ups) and bit-identity with the default."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_03341_b200 as T

shapes = [(1024, 1024, 1024), (512, 1024, 1024), (1024, 512, 2048), (768, 768, 768),
          (1536, 1536, 1536), (2048, 1024, 1024), (1024, 1024, 4096), (2048, 2048, 2048)]
for (m, n, k) in shapes:
    g = torch.Generator(device="cuda"); g.manual_seed(m + n + k)
    A = torch.rand((m, k), generator=g, device="cuda") * 2 - 1
    B = torch.rand((k, n), generator=g, device="cuda") * 2 - 1
    for name in ("corrected3_tf32", "corrected3_halfhalf"):
        ref = T.gemm_device(A, B, name, kernel_variant=4, block_n=256)
        out = {"m": m, "n": n, "k": k, "scheme": name}
        for bn in (0, 64, 128, 192, 256):
            C = T.gemm_device(A, B, name, block_n=bn)
            assert torch.equal(C.view(torch.int32), ref.view(torch.int32)), (m, n, k, name, bn)
            for _ in range(5): T.gemm_device(A, B, name, block_n=bn, out=C)
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            for _ in range(20): T.gemm_device(A, B, name, block_n=bn, out=C)
            e1.record(); torch.cuda.synchronize()
            out[f"bn{bn}"] = round(2 * m * n * k / (e0.elapsed_time(e1) / 20) / 1e9, 1)
        print(json.dumps(out), flush=True)
