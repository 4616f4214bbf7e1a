# Needs a measurement build of the persistent kernel with globaltimer stamps per
# operand stage (see profiles/r02/elect/README.md); prints one CTA pair's timeline.
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2203_03341_b200 as T
n = int(os.environ.get("N", "8192"))
A = torch.rand((n, n), device="cuda") * 2 - 1; B = torch.rand((n, n), device="cuda") * 2 - 1
name = os.environ.get("SCH", "corrected3_halfhalf")
for _ in range(3): T.gemm_device(A, B, name)
torch.cuda.synchronize()
print("=== timed", flush=True)
T.gemm_device(A, B, name); torch.cuda.synchronize()
