"""First-light check: split + gemm on small shapes vs the CPU oracle (test infra)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2203_03341_b200 as T
from paper_2203_03341_b200 import _native as N
from oracle import oracle as O

print("device", torch.cuda.get_device_name(), flush=True)
# split
x = np.concatenate([O.urand(1, 4096, -1, 1, 3).ravel(), O.exprand(1, 4096, -40, 20, 4).ravel()])
for v, name in ((0, "fp16"), (1, "tf32")):
    xt = torch.from_numpy(x).cuda()
    fl = torch.zeros(1, dtype=torch.int32, device="cuda")
    sch = T.scaled_halfhalf() if v == 0 else T.tf32tf32()
    hi, lo = T.split_device(xt, sch, fl)
    torch.cuda.synchronize()
    ohi, olo = O.split(x, name)
    print(name, "split hi eq", np.array_equal(hi.cpu().numpy().astype(np.float64), ohi),
          "lo eq", np.array_equal(lo.cpu().numpy().astype(np.float64), olo), "flags", int(fl.item()), flush=True)

for (m, n, k) in ((128, 128, 64), (128, 128, 256), (200, 136, 1000), (256, 384, 1024)):
    a = O.urand(m, k, -1, 1, 1)
    b = O.urand(k, n, -1, 1, O.pair_seed(1))
    ref64 = O.fp64_ref(a, b) if m * n * k <= 2**26 else a.astype(np.float64) @ b.astype(np.float64)
    for v, name, sname, bk, d in ((0, "fp16", "corrected3_halfhalf", 16, 64), (1, "tf32", "corrected3_tf32", 8, 32)):
        t0 = time.time()
        run = T.gemm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), sname)
        torch.cuda.synchronize()
        c = run.output.cpu().numpy()
        oc, ofl = O.corrected3(a, b, name, block_k=bk, drain_k=d)
        simt = O.fp32_simt(a, b)
        print(f"{m}x{n}x{k} {name}: relres gpu={T.relative_residual(c, ref64):.3e} oracle={T.relative_residual(oc, ref64):.3e} "
              f"simt={T.relative_residual(simt, ref64):.3e} gpu-vs-oracle={T.relative_residual(c, oc):.3e} "
              f"maxabs={np.abs(c-oc).max():.3e} flags={run.flags} t={time.time()-t0:.2f}s", flush=True)
# numpy host path
a = O.urand(64, 96, -1, 1, 7); b = O.urand(96, 40, -1, 1, 8)
run = T.gemm(a, b, "corrected3_halfhalf")
print("host path relres", T.relative_residual(run.output, O.fp64_ref(a, b)), run.flags)
print("launches", N.launch_count())
