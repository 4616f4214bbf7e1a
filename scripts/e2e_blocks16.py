"""e2e through tcec_sgemm_host by blocking and number of compute streams (TCEC_NSC).
Needs a measurement build with HostCtx::kMaxBlk = 16 and four compute streams
(profiles/r02/e2e/README.md); the library clamps blocks to 8 and uses two."""
import ctypes, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2203_03341_b200 import _native as N
n = 16384
hA = torch.empty((n, n), dtype=torch.float32, pin_memory=True).uniform_(-1, 1)
hB = torch.empty((n, n), dtype=torch.float32, pin_memory=True).uniform_(-1, 1)
hC = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
ref = {}
for variant in (1, 0):
    for blocks in ((0, 0), (8, 8), (12, 12), (16, 16), (16, 8), (8, 16), (12, 8)):
        opts = N.make_opts(drain_k=0, host_blocks=blocks)
        fl = ctypes.c_uint32(0)
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            N.check(N.lib().tcec_sgemm_host(variant, n, n, n, hA.data_ptr(), n, hB.data_ptr(), n, hC.data_ptr(), n, ctypes.byref(opts), ctypes.byref(fl), None), "host")
            ts.append((time.perf_counter() - t0) * 1e3)
        if variant not in ref: ref[variant] = hC.clone()
        else: assert torch.equal(ref[variant], hC)
        print("nsc", os.environ.get("TCEC_NSC", "2"), "v", variant, blocks, " ".join("%.1f" % t for t in ts[1:]), flush=True)
