"""Sustained throughput (power-capped steady state): N back-to-back GEMMs,
CUDA-event time of the last half, for fused vs split-once."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_03341_b200 as T

nn = 16384
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 60
a = torch.rand(nn, nn, device="cuda") * 2 - 1
b = torch.rand(nn, nn, device="cuda") * 2 - 1
out = torch.empty(nn, nn, device="cuda")
for sname, v in (("corrected3_halfhalf", "fp16"), ("corrected3_tf32", "tf32")):
    for sm in (0, 2, 0, 2):
        evs = [torch.cuda.Event(True) for _ in range(reps + 1)]
        evs[0].record()
        for i in range(reps):
            T.gemm_device(a, b, sname, out=out, split_mode=sm)
            evs[i + 1].record()
        torch.cuda.synchronize()
        half = reps // 2
        ms = evs[half].elapsed_time(evs[reps]) / (reps - half)
        first = evs[0].elapsed_time(evs[3]) / 3
        clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader"],
                             capture_output=True, text=True).stdout.strip()
        print(f"{v} split_mode={sm}: first3 {2*nn**3/first/1e9:.1f} TF/s, steady {2*nn**3/ms/1e9:.1f} TF/s "
              f"({ms:.2f} ms) clk-after={clk}", flush=True)
