"""Interleaved A/B of library builds: python scripts/ab_libs.py LIB1 LIB2 ...

Each library is loaded in its own subprocess (TCEC_LIB) and times the default
corrected3 GEMM at 16384^3 (TF32 and FP16, urand inputs, CUDA events, 10
launches after 3 warm-ups); the list is run twice in alternating order so
clock / power drift does not favour one build."""
import json
import os
import subprocess
import sys

CHILD = r'''
import json, os, sys, torch
sys.path.insert(0, os.environ["ROOT"])
import paper_2203_03341_b200 as T
n = int(os.environ.get("AB_N", "16384"))
g = torch.Generator(device="cuda"); g.manual_seed(1)
A = torch.rand((n, n), generator=g, device="cuda") * 2 - 1
B = torch.rand((n, n), generator=g, device="cuda") * 2 - 1
C = torch.empty((n, n), device="cuda")
out = {"lib": os.path.basename(os.environ["TCEC_LIB"])}
kw = json.loads(os.environ.get("AB_KW", "{}"))
for name in ("corrected3_tf32", "corrected3_halfhalf"):
    for _ in range(3):
        T.gemm_device(A, B, name, out=C, **kw)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        T.gemm_device(A, B, name, out=C, **kw)
    e1.record(); torch.cuda.synchronize()
    out[name] = round(2 * n ** 3 / (e0.elapsed_time(e1) / 10) / 1e9, 1)
print(json.dumps(out), flush=True)
'''


def main():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libs = sys.argv[1:]
    for order in (libs, libs[::-1]):
        for lib in order:
            env = dict(os.environ, TCEC_LIB=os.path.abspath(lib), ROOT=root)
            r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
            print(r.stdout.strip() or r.stderr[-400:], flush=True)


if __name__ == "__main__":
    main()
