"""Probe the tcgen05 MMA accumulator on the B200 (run under gpurun).

Every output element of a GEMM is an independent experiment: C[i, j] is the
tensor core's sum of the products A[i, t] * B[t, j] (t < k).  The inputs are
exactly representable in the MMA's operand format, and the tc_plain schedule
(one TMEM accumulator over all of k, no drain, the raw FP32 accumulator as
output) runs them through `tcgen05.mma.cta_group::2.kind::f16` (K = 16 per
instruction) or `kind::tf32` (K = 8).  k = one instruction isolates the
multi-term adder (enable_input_d = 0); longer k chains instructions through
the accumulator (D = D + A_k B_k).

The raw inputs and outputs are saved to gpurun_out/probe_acc.npz; the model is
fitted offline (scripts/fit_accumulator.py) and then encoded in the oracle's
hardware mode (oracle/tcec_oracle.c, `hw_mma`).
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

OUT = os.path.join(ROOT, "gpurun_out", "probe_acc.npz")


def fp16_values(rng, shape, emin, emax, zero_frac=0.0):
    """Random FP16 values (as float32) with unbiased exponents in [emin, emax]
    (emin < -14 reaches the subnormals: their bit patterns are drawn directly)."""
    n = int(np.prod(shape))
    e = rng.integers(emin, emax + 1, n)
    man = rng.integers(0, 1024, n)
    sign = rng.integers(0, 2, n)
    v = np.where(e >= -14, (1024 + man) * np.exp2(e - 10.0), man * np.exp2(-24.0))
    v = np.where(sign == 1, -v, v)
    if zero_frac > 0:
        v = np.where(rng.random(n) < zero_frac, 0.0, v)
    out = v.astype(np.float16).astype(np.float32).reshape(shape)
    assert np.array_equal(out.astype(np.float64), v.reshape(shape))
    return out


def tf32_values(rng, shape, emin, emax):
    """Random TF32 values (float32 with the low 13 bits zero), exponents in
    [emin, emax] (below -126: FP32 subnormals on the TF32 grid)."""
    n = int(np.prod(shape))
    e = rng.integers(emin, emax + 1, n)
    man = rng.integers(0, 1024, n)
    sign = rng.integers(0, 2, n)
    v = np.where(e >= -126, (1024 + man) * np.exp2(e - 10.0), man * np.exp2(-136.0))
    v = np.where(sign == 1, -v, v)
    out = v.astype(np.float32).reshape(shape)
    assert np.array_equal(out.astype(np.float64), v.reshape(shape))
    assert not np.any(out.view(np.uint32) & 0x1FFF)
    return out


def crafted_fp16(rng, m, k):
    """Rows of A for cancellation / alignment experiments (B = ones or powers of
    two): a big term, its negation at another position, and small terms."""
    rows = []
    for _ in range(m):
        r = np.zeros(k)
        kind = rng.integers(0, 6)
        p, q = rng.choice(k, 2, replace=False)
        big = np.exp2(rng.integers(-2, 15))
        if kind == 0:  # big - big + small at random positions
            r[p], r[q] = big, -big
            for t in rng.choice([t for t in range(k) if t not in (p, q)], rng.integers(1, 4), replace=False):
                r[t] = np.exp2(rng.integers(-24, 14)) * rng.choice([-1, 1]) * (1 + rng.integers(0, 1024) / 1024)
        elif kind == 1:  # 1 + many small terms of one size
            r[p] = big
            e = rng.integers(-24, 0)
            for t in range(k):
                if t != p:
                    r[t] = np.exp2(float(np.log2(big)) + e) * rng.choice([1, -1]) * (1 + rng.integers(0, 8) / 8)
        elif kind == 2:  # one big term, one small term (alignment width)
            r[p] = big * (1 + rng.integers(0, 1024) / 1024)
            r[q] = big * np.exp2(-rng.integers(10, 40)) * rng.choice([-1, 1]) * (1 + rng.integers(0, 1024) / 1024)
        elif kind == 3:  # rounding: big with a tail just at / around the 24th bit
            r[p] = big
            d = rng.integers(20, 30)
            r[q] = rng.choice([-1, 1]) * big * np.exp2(-d) * (1 + rng.integers(0, 4) / 4)
            t = [t for t in range(k) if t not in (p, q)][0]
            r[t] = rng.choice([-1, 1, 0]) * big * np.exp2(-d - rng.integers(1, 6))
        elif kind == 4:  # all equal magnitude, mixed signs
            e = rng.integers(-24, 15)
            r[:] = np.exp2(e) * rng.choice([-1, 1], k) * (1 + rng.integers(0, 1024, k) / 1024)
        else:  # zeros with signs
            r[:] = -0.0 if rng.integers(0, 2) else 0.0
            if rng.integers(0, 2):
                r[p] = np.exp2(rng.integers(-24, 0))
                r[q] = -r[p]
        rows.append(r)
    a = np.array(rows).astype(np.float16).astype(np.float32)
    return a


def run_sets():
    import torch

    import paper_2203_03341_b200 as T

    torch.backends.cuda.matmul.allow_tf32 = False
    rng = np.random.default_rng(20261017)
    sets = {}

    def gemm(name, a, b, scheme):
        A = torch.from_numpy(np.ascontiguousarray(a)).cuda()
        B = torch.from_numpy(np.ascontiguousarray(b)).cuda()
        c = T.gemm_device(A, B, scheme).cpu().numpy()
        sets[name + "__A"] = a
        sets[name + "__B"] = b
        sets[name + "__C"] = c
        print(name, a.shape, b.shape, flush=True)

    M = N = 512
    # ---- FP16, one instruction (k = 16) and chains (k = 32, 64, 256)
    for tag, (lo, hi) in {"narrow": (-1, 1), "mid": (-8, 8), "wide": (-24, 15),
                          "sub": (-24, -10)}.items():
        for k in (16, 32, 64, 256):
            a = fp16_values(rng, (M, k), lo, hi)
            b = fp16_values(rng, (k, N), lo, hi)
            gemm(f"f16_{tag}_k{k}", a, b, "tc_plain_fp16")
    # ones / powers of two in B: the products are A's values (exact FP16)
    for k in (16, 32):
        a = crafted_fp16(rng, M, k)
        b = np.ones((k, N), np.float32)
        b[:, 1::2] = np.exp2(rng.integers(-8, 8, (k, N // 2))).astype(np.float32)
        b[:, 2::4] = -b[:, 2::4]
        gemm(f"f16_crafted_k{k}", a, b, "tc_plain_fp16")
    # ---- TF32, one instruction (k = 8) and chains
    for tag, (lo, hi) in {"narrow": (-1, 1), "mid": (-8, 8), "wide": (-60, 60),
                          "sub": (-140, -110)}.items():
        for k in (8, 16, 32, 256):
            a = tf32_values(rng, (M, k), lo, hi)
            b = tf32_values(rng, (k, N), lo, hi)
            gemm(f"tf32_{tag}_k{k}", a, b, "tc_plain_tf32")
    np.savez_compressed(OUT, **sets)
    print("saved", OUT)


def run_edge_sets():
    """Second round: the edges the random sets do not reach -- FP32-subnormal
    and overflowing sums (TF32), non-finite operands (the FP16 hi of an input
    >= 65520 is inf), negative zeros -- and corrected3 outputs of the full
    kernels for offline comparison with the oracle's hardware mode."""
    import torch

    import paper_2203_03341_b200 as T

    rng = np.random.default_rng(77)
    sets = {}

    def save(name, a, b, c):
        sets[name + "__A"], sets[name + "__B"], sets[name + "__C"] = a, b, c
        print(name, a.shape, b.shape, flush=True)

    def plain(name, a, b, scheme):
        A = torch.from_numpy(np.ascontiguousarray(a)).cuda()
        B = torch.from_numpy(np.ascontiguousarray(b)).cuda()
        save(name, a, b, T.gemm_device(A, B, scheme).cpu().numpy())

    M = N = 256
    # TF32 products landing in the FP32 subnormal range and around the overflow threshold
    for k in (8, 32):
        plain(f"tf32_subout_k{k}", tf32_values(rng, (M, k), -80, -60), tf32_values(rng, (k, N), -80, -60),
              "tc_plain_tf32")
        plain(f"tf32_ovf_k{k}", tf32_values(rng, (M, k), 60, 66), tf32_values(rng, (k, N), 60, 66),
              "tc_plain_tf32")
        # an accumulator in the subnormal range: a large-ish first instruction cancelled later
        a = tf32_values(rng, (M, k), -75, -62)
        b = tf32_values(rng, (k, N), -75, -62)
        plain(f"tf32_subacc_k{k}", a, b, "tc_plain_tf32")
    # non-finite operands: FP16 inf (as an operand value) and zeros, both signs
    for fmt, scheme, big in (("f16", "tc_plain_fp16", np.float32(np.inf)),
                             ("tf32", "tc_plain_tf32", np.float32(np.inf))):
        k = 16 if fmt == "f16" else 8
        vals = fp16_values if fmt == "f16" else tf32_values
        a = vals(rng, (M, k), -4, 4)
        b = vals(rng, (k, N), -4, 4)
        mask = rng.random((M, k)) < 0.05
        a[mask] = big * np.where(rng.random(mask.sum()) < 0.5, -1, 1)
        zmask = rng.random((k, N)) < 0.2
        b[zmask] = np.where(rng.random(zmask.sum()) < 0.5, -0.0, 0.0)
        plain(f"{fmt}_inf_k{k}", a, b, scheme)
        # signed zeros only
        a = np.where(rng.random((M, k)) < 0.5, -0.0, 0.0).astype(np.float32)
        a[:, 0] = vals(rng, (M, 1), -2, 2)[:, 0]
        b = np.where(rng.random((k, N)) < 0.5, -0.0, 0.0).astype(np.float32)
        plain(f"{fmt}_zeros_k{k}", a, b, scheme)
    # corrected3 through the production kernels (default, reference drain, persistent)
    for sname, tag in (("corrected3_halfhalf", "c3f16"), ("corrected3_tf32", "c3tf32")):
        for dist, (lo, hi) in {"urand": (None, None), "exp": (-15, 14), "wide": (-40, 15)}.items():
            m, n, k = 256, 256, 1000
            if lo is None:
                a = rng.uniform(-1, 1, (m, k)).astype(np.float32)
                b = rng.uniform(-1, 1, (k, n)).astype(np.float32)
            else:
                a = (rng.uniform(1, 2, (m, k)) * np.exp2(rng.integers(lo, hi + 1, (m, k)))
                     * rng.choice([-1, 1], (m, k))).astype(np.float32)
                b = (rng.uniform(1, 2, (k, n)) * np.exp2(rng.integers(lo, hi + 1, (k, n)))
                     * rng.choice([-1, 1], (k, n))).astype(np.float32)
            A = torch.from_numpy(a).cuda()
            B = torch.from_numpy(b).cuda()
            for d in (0, 16, 48):
                if d and "tf32" in sname:
                    d //= 2
                c = T.gemm_device(A, B, sname, drain_k=d or None).cpu().numpy()
                save(f"{tag}_{dist}_d{d}", a, b, c)
        # overflow: a few inputs at / above the FP16 hi threshold
        a = rng.uniform(-1, 1, (256, 256)).astype(np.float32)
        b = rng.uniform(-1, 1, (256, 256)).astype(np.float32)
        a[3, 7] = 70000.0
        a[5, :3] = [65520.0, -65536.0, 1e5]
        b[9, 11] = -1e6
        A = torch.from_numpy(a).cuda()
        B = torch.from_numpy(b).cuda()
        save(f"{tag}_ovf", a, b, T.gemm_device(A, B, sname).cpu().numpy())
    out = os.path.join(ROOT, "gpurun_out", "probe_acc2.npz")
    np.savez_compressed(out, **sets)
    print("saved", out)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "edges":
        run_edge_sets()
    else:
        run_sets()
