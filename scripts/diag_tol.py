"""Diagnostics: GPU vs reference goldens in units of 2^-24 * sum|a_eff||b_eff| (split magnitudes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_03341_b200 as T
from oracle import oracle as O
g = np.load("tests/golden/gemm_golden.npz")
for bn in (128, 256):
  for tag in [str(t) for t in g["names"]]:
    a, b = g[f"{tag}__A"], g[f"{tag}__B"]
    for sname, var, s in (("corrected3_halfhalf", "fp16", 11), ("corrected3_tf32", "tf32", 0)):
        fl = torch.zeros(1, dtype=torch.int32, device="cuda")
        c = T.gemm_device(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), sname, flags=fl, block_n=bn).cpu().numpy()
        ref = g[f"{tag}__{sname}__C"]
        ah, al = O.split(a, var); bh, bl = O.split(b, var)
        ah, al, bh, bl = [np.nan_to_num(x, posinf=0, neginf=0) for x in (ah, al, bh, bl)]
        mag = np.abs(ah) @ np.abs(bh) + (np.abs(al) @ np.abs(bh) + np.abs(ah) @ np.abs(bl)) * 2.0 ** -s
        mag0 = np.abs(a.astype(np.float64)) @ np.abs(b.astype(np.float64))
        fin = np.isfinite(ref) & np.isfinite(c)
        d = np.abs(c[fin].astype(np.float64) - ref[fin])
        r1 = np.max(d / np.maximum(mag[fin] * 2.0 ** -24, 1e-300)) if d.size else 0
        r0 = np.max(d / np.maximum(mag0[fin] * 2.0 ** -24, 1e-300)) if d.size else 0
        finpat = np.array_equal(np.isfinite(ref), np.isfinite(c))
        print(f"bn={bn} {tag:28s} {var}: max diff/(u*|a_eff||b_eff|)={r1:9.2f}  /(u*|a||b|)={r0:9.2f} finite_pattern_eq={finpat} flags={int(fl.item())} ref_flags={tuple(g[f'{tag}__{sname}__flags'])}", flush=True)
