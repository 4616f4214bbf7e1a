# Needs a measurement build of the 256 x 64 kernel with globaltimer stamps per
# stage (profiles/r02/elect/README.md); prints the per-stage timeline of one CTA.
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2203_03341_b200 as T
m = n = k = 1024
A = torch.rand((m, k), device="cuda"); B = torch.rand((k, n), device="cuda")
T.gemm_device(A, B, os.environ.get("SCH", "corrected3_tf32"), block_n=64); torch.cuda.synchronize()
print("=== second", flush=True)
T.gemm_device(A, B, os.environ.get("SCH", "corrected3_tf32"), block_n=64); torch.cuda.synchronize()
