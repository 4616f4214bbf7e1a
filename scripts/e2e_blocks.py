"""e2e (host buffers, pinned) through tcec_sgemm_host for several C blockings."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_03341_b200 import _native as N

n = 16384
hA = torch.empty((n, n), dtype=torch.float32, pin_memory=True).uniform_(-1, 1)
hB = torch.empty((n, n), dtype=torch.float32, pin_memory=True).uniform_(-1, 1)
hC = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
ref = None
for variant, name in ((1, "tf32"), (0, "fp16")):
    for blocks in ((1, 1), (8, 1), (4, 4), (8, 4), (4, 8), (8, 8), (0, 0)):
        opts = N.make_opts(drain_k=0, host_blocks=blocks)
        fl = ctypes.c_uint32(0)
        call = lambda: N.check(N.lib().tcec_sgemm_host(variant, n, n, n, hA.data_ptr(), n, hB.data_ptr(), n,
                                                        hC.data_ptr(), n, ctypes.byref(opts), ctypes.byref(fl), None), "host")
        call()
        if blocks == (1, 1):
            ref = hC.clone()
        else:
            assert torch.equal(hC, ref), blocks
        t0 = time.perf_counter()
        for _ in range(3):
            call()
        dt = (time.perf_counter() - t0) / 3
        print(f"{name} blocks={blocks}: {dt*1e3:.1f} ms  {2*n**3/dt/1e12:.1f} TF/s e2e", flush=True)
