"""The README usage snippet, runnable: host-array gemm(), gemm_device() and the
operator form agree bit for bit (TF32-TCEC host vs op)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_03341_b200 as tcec

a = np.random.default_rng(0).uniform(-1, 1, (4096, 4096)).astype(np.float32)
run = tcec.gemm(a, a, "corrected3_tf32")
print(run.output.dtype, run.flags)
A = torch.from_numpy(a).cuda()
C = tcec.gemm_device(A, A, "corrected3_halfhalf")
C2 = torch.ops.tcec.sgemm(A, A, 1, 0)[0]
torch.cuda.synchronize()
print(C.shape, torch.equal(C2.cpu(), torch.from_numpy(run.output)))
