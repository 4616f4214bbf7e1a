"""Subsample the B200 accumulator-probe outputs into a committed fixture.

Input: gpurun_out/probe_acc.npz and probe_acc2.npz, written on the B200 by
scripts/probe_accumulator.py (raw operands and the tensor core's outputs).
Output: tests/golden/hw_probe_golden.npz -- for every dataset the first rows
of A, the first columns of B and the matching block of C (16 x 32; 8 x 16 for
k = 256; 4 x 8 for the corrected3 kernel outputs, of which a subset is kept):
rows and columns are independent experiments, so a sub-block is exact.
tests/test_oracle_golden.py checks the oracle's hardware model
(tcec_oracle_hw) against it bit for bit on the CPU.
"""

import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "hw_probe_golden.npz")


def main():
    out = {}
    for fname in ("probe_acc.npz", "probe_acc2.npz"):
        d = np.load(os.path.join(ROOT, "gpurun_out", fname))
        for nm in sorted({k.split("__")[0] for k in d.files}):
            if nm.startswith("c3"):
                if not (nm.endswith("_ovf") or "_d0" in nm or "wide_d16" in nm or "wide_d8" in nm):
                    continue
                r, c = 4, 8
            else:
                r, c = (8, 16) if d[nm + "__A"].shape[1] >= 256 else (16, 32)
            out[nm + "__A"] = np.ascontiguousarray(d[nm + "__A"][:r])
            out[nm + "__B"] = np.ascontiguousarray(d[nm + "__B"][:, :c])
            out[nm + "__C"] = np.ascontiguousarray(d[nm + "__C"][:r, :c])
    np.savez_compressed(OUT, **out)
    print(OUT, os.path.getsize(OUT))


if __name__ == "__main__":
    main()
