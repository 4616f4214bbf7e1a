"""One GEMM configuration, a few launches (for ncu captures).
usage: one_gemm.py <fp16|tf32> <n> [json kwargs] [reps] [dist: urand | exprand:a,b]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2203_03341_b200 as T

v, nn = sys.argv[1], int(sys.argv[2])
kw = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
sname = "corrected3_halfhalf" if v == "fp16" else "corrected3_tf32"
from bench import device_matrix, parse_dist

spec = parse_dist(sys.argv[5] if len(sys.argv) > 5 else "urand")
g = torch.Generator(device="cuda")
g.manual_seed(1)
a = device_matrix(spec, nn, nn, g, "cuda")
b = device_matrix(spec, nn, nn, g, "cuda")
out = torch.empty(nn, nn, device="cuda")
for _ in range(reps):
    T.gemm_device(a, b, sname, out=out, **kw)
torch.cuda.synchronize()
print("done", v, nn, kw, spec)
