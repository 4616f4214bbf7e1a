"""Generate golden vectors FROM THE REFERENCE IMPLEMENTATION (build container only).

Run here, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package read-only and writes small .npz fixtures next
to this script.  The fixtures are committed; nothing at test / bench time on the
GPU box reads /root/reference.  Everything is drawn through the reference's own
generators (genmat.py) and computed by the reference's own gemm / split_matrix /
classify_array / round_to_format, so the fixtures pin the C oracle
(oracle/tcec_oracle.c) to the reference bit for bit.
"""

from __future__ import annotations

import os
import sys
from dataclasses import replace

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import tcgemm  # noqa: E402  (the reference)
from tcgemm import schemes as S  # noqa: E402
from tcgemm.formats import FP16, FP32, TF32, RoundingMode  # noqa: E402
from tcgemm.mma import _accumulate_blocks, _sum_round_to_odd, _terminal  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def split_goldens():
    rng = np.random.default_rng(20220307)
    # random bit patterns over the whole finite FP32 range, plus edges
    bits = rng.integers(0, 1 << 32, size=40000, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    x = x[np.isfinite(x)]
    edges = np.array([
        0.0, -0.0, 1.0, -1.0, 65504.0, 65519.0, 65520.0, 65535.9, 65536.0, -65520.0,
        2.0 ** -14, 2.0 ** -24, 2.0 ** -25, 3 * 2.0 ** -26, 2.0 ** -34, 2.0 ** -35,
        2.0 ** -126, 2.0 ** -127, 2.0 ** -149, np.float32(3.4028235e38),
        np.float32(3.4e38), np.float32(-3.4028235e38), 1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11,
    ], dtype=np.float32)
    x = np.concatenate([edges, np.array([0x3F801003], np.uint32).view(np.float32),
                        rng.uniform(-1, 1, 20000).astype(np.float32),
                        tcgemm.generate(tcgemm.MatrixSpec(1, 20000, tcgemm.ExpRand(-40, 20), 7))[0]])
    out = {"x": x}
    for name, sch in (
        ("fp16_rn", tcgemm.scaled_halfhalf(RoundingMode.RN)),
        ("fp16_rz", tcgemm.scaled_halfhalf(RoundingMode.RZ)),
        ("tf32_rna", tcgemm.tf32tf32(RoundingMode.RNA)),
        ("tf32_rn", tcgemm.tf32tf32(RoundingMode.RN)),
        ("tf32_rz", tcgemm.tf32tf32(RoundingMode.RZ)),
    ):
        sm = tcgemm.split_matrix(x.astype(np.float64).reshape(1, -1), sch)
        out[name + "_hi"] = sm.hi.ravel()
        out[name + "_lo"] = sm.lo.ravel()
        out[name + "_class"] = S.classify_array(x.astype(np.float64), sch).astype(np.int8)
    # general rounding kit (formats.py) on float64 residual-like inputs
    r = np.concatenate([rng.standard_normal(5000) * 2.0 ** rng.integers(-40, 20, 5000),
                        np.ldexp(rng.integers(-4096, 4096, 5000).astype(np.float64), -24)])
    out["round_x"] = r
    for fname, fmt in (("fp16", FP16), ("tf32", TF32), ("fp32", FP32)):
        for mname, mode in (("rn", RoundingMode.RN), ("rna", RoundingMode.RNA), ("rz", RoundingMode.RZ)):
            out[f"round_{fname}_{mname}"] = tcgemm.round_to_format(r, fmt, mode)
    np.savez_compressed(os.path.join(OUT, "split_golden.npz"), **out)


def _drain_restatement(A, B, split, bk, drain):
    """SURVEY.md Appendix A restatement composed ONLY of reference primitives.

    Main-term partial takes a terminal RZ per block and is folded into C every
    drain/bk blocks; drain == bk reproduces gemm(corrected3) bit-exactly.
    """
    cfg = S.default_config(S.corrected3(split), block_k=bk)
    Ap, Bp = S._pad_k(A, B, bk)
    s = split.scale_log2
    sa = S.split_matrix(Ap, split)
    sb = S.split_matrix(Bp, split)
    ah, bh = S._to_blocks(sa.hi, sb.hi, bk)
    al, bl = S._to_blocks(sa.lo, sb.lo, bk)
    cfg_rz = replace(cfg, terminal_rounding=RoundingMode.RZ)
    a1 = _accumulate_blocks(al, bh, cfg_rz)
    a2 = _accumulate_blocks(ah, bl, cfg_rz)
    a3 = _accumulate_blocks(ah, bh, cfg_rz)
    shape = (A.shape[0], B.shape[1])
    dc = np.zeros(shape)
    for bi in range(a3.shape[0]):
        dc = _terminal(a1[bi], dc, cfg_rz)
        dc = _terminal(a2[bi], dc, cfg_rz)
    c = np.zeros(shape)
    tmp = np.zeros(shape)
    per = drain // bk
    for bi in range(a3.shape[0]):
        tmp = _terminal(a3[bi], tmp, cfg_rz)
        if (bi + 1) % per == 0 or bi == a3.shape[0] - 1:
            c = S._round32_rn(_sum_round_to_odd(c, tmp))
            tmp = np.zeros(shape)
    c = S._round32_rn(_sum_round_to_odd(c, np.ldexp(dc, -s)))
    return c.astype(np.float32)


def gemm_goldens():
    cases = []
    G = tcgemm.generate
    MS = tcgemm.MatrixSpec
    # (tag, A, B)
    for seed in (0, 1):
        for (m, n, k) in ((16, 16, 64), (8, 24, 200), (16, 16, 1024), (5, 7, 33)):
            a = G(MS(m, k, tcgemm.Urand(-1, 1), seed))
            b = G(MS(k, n, tcgemm.Urand(-1, 1), tcgemm.pair_seed(seed)))
            cases.append((f"urand_s{seed}_{m}x{n}x{k}", a, b))
    for t in (1, 2, 3, 4):
        a, b = tcgemm.type_pair(t, 8, 8, 256, 3)
        cases.append((f"type{t}_8x8x256", a, b))
    a = G(MS(8, 128, tcgemm.ExpRand(-15, 15), 11))
    b = G(MS(128, 8, tcgemm.ExpRand(-15, 15), 12))
    cases.append(("exprand_m15_15_8x8x128", a, b))
    # overflow edge: values >= 65520 overflow the FP16 hi (NaN output + flags)
    a = G(MS(4, 48, tcgemm.ExpRand(14, 16), 21))
    b = G(MS(48, 4, tcgemm.Urand(-1, 1), 22))
    cases.append(("overflow_4x4x48", a, b))
    # single overflowing inputs where the reference returns +-inf, not NaN: B's
    # values have lo != 0 of hi's sign, so A_hi * dB is an infinity of the main
    # term's sign (splitting.py:119-121 sets that row's dA to 0); one zero in B
    # makes inf * 0 = NaN in one column.  Row 1: 70000 overflows FP16 only;
    # row 4: -65520 rounds (RN, ties to even) to -65536 = -inf in FP16; row 5:
    # FLT_MAX overflows both hi formats.
    a = G(MS(6, 40, tcgemm.Urand(-1, 1), 23)).copy()
    a[1, 3], a[4, 10], a[5, 0] = 70000.0, -65520.0, np.float32(3.4028235e38)
    rng = np.random.default_rng(24)
    b = (np.float32(1 + 2.0 ** -13) * np.exp2(rng.integers(-3, 1, (40, 8)))
         * rng.choice([-1, 1], (40, 8))).astype(np.float32)
    b[3, 2] = 0.0
    cases.append(("ovf_inf_6x8x40", a, b))
    # identity: A = I16, B FP16-exact -> output == B
    eye = np.eye(16, dtype=np.float32)
    bexact = (np.round(G(MS(16, 16, tcgemm.Urand(-1, 1), 5)) * 1024) / 1024).astype(np.float32)
    cases.append(("identity_16", eye, bexact))

    out = {}
    names = []
    for tag, a, b in cases:
        names.append(tag)
        out[f"{tag}__A"] = a
        out[f"{tag}__B"] = b
        for sname in ("corrected3_halfhalf", "corrected3_tf32"):
            run = tcgemm.gemm(a, b, tcgemm.SCHEMES_BY_NAME[sname])
            out[f"{tag}__{sname}__C"] = run.output
            out[f"{tag}__{sname}__flags"] = np.array(
                [run.flags.saw_overflow, run.flags.saw_out_of_range], dtype=np.int8)
        out[f"{tag}__fp32_simt__C"] = tcgemm.gemm(a, b, tcgemm.SCHEMES_BY_NAME["fp32_simt"]).output
        out[f"{tag}__fp64_ref__C"] = tcgemm.gemm(a, b, tcgemm.SCHEMES_BY_NAME["fp64_ref"]).output
    # drain-interval restatement goldens (block 16 for FP16 / 8 for TF32)
    a = G(MS(8, 512, tcgemm.Urand(-1, 1), 31))
    b = G(MS(512, 8, tcgemm.Urand(-1, 1), tcgemm.pair_seed(31)))
    out["drain__A"], out["drain__B"] = a, b
    for split_name, split, bk in (("fp16", tcgemm.scaled_halfhalf(), 16), ("tf32", tcgemm.tf32tf32(), 8)):
        for d in (bk, 64, 128):
            c = _drain_restatement(a.astype(np.float64), b.astype(np.float64), split, bk, d)
            out[f"drain__{split_name}__bk{bk}__d{d}"] = c
        if bk == 16:
            ref = tcgemm.gemm(a, b, tcgemm.corrected3(split)).output
            assert np.array_equal(ref, out[f"drain__{split_name}__bk16__d16"])
    # 4-term (dA*dB included) sibling
    a4 = G(MS(6, 96, tcgemm.Urand(-1, 1), 41))
    b4 = G(MS(96, 6, tcgemm.Urand(-1, 1), 42))
    r3, r4, _ = tcgemm.delta_term_ablation(a4, b4)
    out["dd__A"], out["dd__B"], out["dd__C3"], out["dd__C4"] = a4, b4, r3.output, r4.output
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "gemm_golden.npz"), **out)


def generator_goldens():
    out = {
        "urand_s0": tcgemm.generate(tcgemm.MatrixSpec(4, 5, tcgemm.Urand(-1, 1), 0)),
        "urand_pair_s0": tcgemm.generate(tcgemm.MatrixSpec(5, 3, tcgemm.Urand(-1, 1), tcgemm.pair_seed(0))),
        "exprand_s3": tcgemm.generate(tcgemm.MatrixSpec(6, 4, tcgemm.ExpRand(-15, 14), 3)),
    }
    for t in (1, 2, 3, 4):
        a, b = tcgemm.type_pair(t, 3, 4, 5, 9)
        out[f"type{t}_A"], out[f"type{t}_B"] = a, b
    np.savez_compressed(os.path.join(OUT, "genmat_golden.npz"), **out)


def inunit_goldens():
    """The reference's in-unit comparator schemes (schemes.py:343-364), which
    the GPU also runs on the tensor core: pins oracle.inunit bit for bit."""
    G = tcgemm.generate
    MS = tcgemm.MatrixSpec
    cases = []
    for seed in (0, 1):
        a = G(MS(8, 64, tcgemm.Urand(-1, 1), seed))
        b = G(MS(64, 8, tcgemm.Urand(-1, 1), tcgemm.pair_seed(seed)))
        cases.append((f"urand_s{seed}_8x8x64", a, b))
    a = G(MS(6, 1024, tcgemm.Urand(-1, 1), 5))
    b = G(MS(1024, 6, tcgemm.Urand(-1, 1), tcgemm.pair_seed(5)))
    cases.append(("urand_6x6x1024", a, b))
    a = G(MS(8, 128, tcgemm.ExpRand(-15, 15), 11))
    b = G(MS(128, 8, tcgemm.ExpRand(-15, 15), 12))
    cases.append(("exprand_8x8x128", a, b))
    a, b = tcgemm.type_pair(2, 8, 8, 96, 3)
    cases.append(("type2_8x8x96", a, b))
    a = G(MS(4, 40, tcgemm.ExpRand(-40, -20), 13))  # FP16 conversion vanishes
    b = G(MS(40, 4, tcgemm.Urand(-1, 1), 14))
    cases.append(("tiny_4x4x40", a, b))
    a = G(MS(4, 48, tcgemm.ExpRand(14, 16), 21))    # FP16 conversion overflows
    b = G(MS(48, 4, tcgemm.Urand(-1, 1), 22))
    cases.append(("overflow_4x4x48", a, b))
    schemes = {name: tcgemm.SCHEMES_BY_NAME[name] for name in
               ("tc_plain_fp16", "tc_plain_tf32", "markidis4", "corrected4_rn", "corrected4_rz")}
    schemes["markidis4_tf32"] = tcgemm.markidis4(TF32)
    out = {"names": np.array([c[0] for c in cases]), "schemes": np.array(list(schemes))}
    for tag, a, b in cases:
        out[f"{tag}__A"], out[f"{tag}__B"] = a, b
        for sname, sch in schemes.items():
            run = tcgemm.gemm(a, b, sch)
            out[f"{tag}__{sname}__C"] = run.output
            out[f"{tag}__{sname}__flags"] = np.array(
                [run.flags.saw_overflow, run.flags.saw_out_of_range], dtype=np.int8)
    np.savez_compressed(os.path.join(OUT, "inunit_golden.npz"), **out)


def split_stats_goldens():
    """analysis.py exhaustive_length_distribution (split-stats) for RN / RNA / RZ."""
    import json

    from tcgemm.analysis import exhaustive_length_distribution

    out = {}
    for r in ("rn", "rna", "rz"):
        d = exhaustive_length_distribution(RoundingMode.parse(r))
        out[r] = {str(k): [v.numerator, v.denominator] for k, v in d.probabilities.items()}
    with open(os.path.join(OUT, "split_stats_golden.json"), "w") as f:
        json.dump(out, f, indent=0)


if __name__ == "__main__":
    if sys.argv[1:] == ["split-stats"]:
        split_stats_goldens()
        sys.exit(0)
    if sys.argv[1:] == ["inunit"]:
        inunit_goldens()
        sys.exit(0)
    split_goldens()
    generator_goldens()
    gemm_goldens()
    inunit_goldens()
    split_stats_goldens()
    print("wrote", sorted(f for f in os.listdir(OUT) if f.endswith(".npz")))
