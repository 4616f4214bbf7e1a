import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2203_03341_b200 as T
for (m, n, k) in ((1024, 1024, 1024), (1024, 1024, 4096), (512, 512, 8192)):
    g = torch.Generator(device="cuda"); g.manual_seed(1)
    A = torch.rand((m, k), generator=g, device="cuda") * 2 - 1
    B = torch.rand((k, n), generator=g, device="cuda") * 2 - 1
    for name in ("corrected3_tf32", "corrected3_halfhalf"):
        ref = T.gemm_device(A, B, name, kernel_variant=4, block_n=256)
        res = []
        for bn in (64, 128, 256):
            C = T.gemm_device(A, B, name, block_n=bn)
            assert torch.equal(C, ref)
            for _ in range(5): T.gemm_device(A, B, name, block_n=bn, out=C)
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            for _ in range(20): T.gemm_device(A, B, name, block_n=bn, out=C)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            res.append("bn%d %.1f us (%.1f TF/s)" % (bn, ms * 1e3, 2 * m * n * k / ms / 1e9))
        print(os.path.basename(os.environ.get("TCEC_LIB", "cur")), m, n, k, name, " | ".join(res), flush=True)
