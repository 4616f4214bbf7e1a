"""GPU accuracy harness: the reference's `gemm-accuracy` experiment on B200.

Mirrors `tcgemm gemm-accuracy` (reference cli.py:135-170, parser :227-265):
same flags, the same CSV ("m,n,k,scheme,seed,residual,flags" plus an `avg`
row per (m, n, k, scheme)), the same inputs (genmat.py generators, restated
bit-exactly in genmat.py here) and the same metric (Eq. 7, analysis.py:175-192).
The hot path runs on the GPU; the FP64 ground truth is cuBLAS DGEMM on the GPU
(the reference's sequential FP64 sum differs from it at the 1e-16 level).

Schemes: corrected3_halfhalf / corrected3_tf32 (the accelerated path), the
reference's in-unit comparators run on the tensor core (tc_plain_fp16,
tc_plain_tf32, markidis4, corrected4_rz -- the hardware's own accumulator
rounding), and `cublas_sgemm` (FP32 SIMT SGEMM, TF32 disabled) as the SGEMM
baseline.  `ablate-delta` mirrors cli.py:196-214 (three- vs four-term
correction, delta_term_ablation) and `rounding-ablation` is the hardware
analogue of cli.py:173-193: the tensor core's terminal rounding cannot be
switched, so it reports the in-unit four-term scheme (corrected4_rz on the
hardware) against corrected3 (accumulation moved out of the unit) and SGEMM.

    python -m paper_2203_03341_b200.accuracy gemm-accuracy --m 16 --n 16 \
        --k 256,1024,4096 --scheme corrected3_halfhalf,cublas_sgemm --dist urand:-1,1
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

from .genmat import ExpRand, MatrixSpec, Urand, generate, pair_seed, type_pair

GPU_SCHEMES = ("corrected3_halfhalf", "corrected3_tf32", "tc_plain_fp16", "tc_plain_tf32",
               "markidis4", "corrected4_rz", "corrected4_rn", "cublas_sgemm")


def _fmt64(x: float) -> str:
    return format(float(x), ".17g")


def _parse_int_list(text: str) -> list[int]:
    return [int(part) for part in text.split(",") if part != ""]


def parse_dist(text: str):
    """cli.py:58-75: urand:lo,hi | exprand:a,b | type:1..4."""
    kind, _, rest = text.partition(":")
    kind = kind.strip().lower()
    try:
        if kind == "urand":
            lo, hi = (float(p) for p in rest.split(","))
            return Urand(lo, hi)
        if kind == "exprand":
            a, b = (int(p) for p in rest.split(","))
            return ExpRand(a, b)
        if kind == "type":
            type_id = int(rest)
            if not 1 <= type_id <= 4:
                raise ValueError
            return ("type", type_id)
    except (TypeError, ValueError):
        raise ValueError(f"bad distribution spec: {text!r}") from None
    raise ValueError(f"unknown distribution kind: {kind!r}")


def input_pair(dist, m: int, n: int, k: int, seed: int):
    """cli.py:92-97."""
    if isinstance(dist, tuple) and dist[0] == "type":
        return type_pair(dist[1], m, n, k, seed)
    a = generate(MatrixSpec(m, k, dist, seed))
    b = generate(MatrixSpec(k, n, dist, pair_seed(seed)))
    return a, b


def _flags_field(saw_overflow: bool, saw_out_of_range: bool) -> str:
    parts = []
    if saw_overflow:
        parts.append("overflow")
    if saw_out_of_range:
        parts.append("out_of_range")
    return ";".join(parts)


def gemm_accuracy(ms, ns, ks, schemes, dist, seeds, block_k: int = 0) -> list[str]:
    """cmd_gemm_accuracy (cli.py:135-170) with the GEMMs on the GPU."""
    import torch

    from .schemes import gemm

    for name in schemes:
        if name not in GPU_SCHEMES:
            raise ValueError(f"unknown scheme {name!r}; known: {', '.join(GPU_SCHEMES)}")
    if not schemes:
        raise ValueError("no schemes requested")
    prev_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    cfg = _cfg(block_k)
    lines = ["m,n,k,scheme,seed,residual,flags"]
    try:
        for m in ms:
            for n in ns:
                for k in ks:
                    inputs, refs = {}, {}
                    for seed in seeds:
                        a, b = input_pair(dist, m, n, k, seed)
                        A = torch.from_numpy(a).cuda()
                        B = torch.from_numpy(b).cuda()
                        inputs[seed] = (A, B)
                        refs[seed] = A.double() @ B.double()
                    for name in schemes:
                        residuals, fields = [], []
                        for seed in seeds:
                            A, B = inputs[seed]
                            ref = refs[seed]
                            if name == "cublas_sgemm":
                                out = A @ B
                                fl = (bool((~torch.isfinite(out)).any().item()), False)
                            else:
                                run = gemm(A, B, name, cfg)
                                out = run.output
                                fl = (run.flags.saw_overflow, run.flags.saw_out_of_range)
                            den = float(torch.linalg.norm(ref))
                            num = float(torch.linalg.norm(ref - out.double()))
                            res = 0.0 if den == 0.0 and num == 0.0 else num / den
                            residuals.append(res)
                            fields.append(_flags_field(*fl))
                            lines.append(f"{m},{n},{k},{name},{seed},{_fmt64(res)},{fields[-1]}")
                        avg = float(np.mean(residuals))
                        union = ";".join(p for p in ("overflow", "out_of_range")
                                         if any(p in f for f in fields))
                        lines.append(f"{m},{n},{k},{name},avg,{_fmt64(avg)},{union}")
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev_tf32
    return lines


def _cfg(block_k: int):
    """block_k > 0: MmaConfig(block_k), the reference's drain schedule; 0: the
    kernel's tuned default drain interval (no MmaConfig)."""
    from .schemes import MmaConfig

    return MmaConfig(block_k=block_k) if block_k > 0 else None


def _residual(ref, out) -> float:
    """analysis.py:175-192 (Eq. 7) against the FP64 product on the GPU."""
    import torch

    den = float(torch.linalg.norm(ref))
    num = float(torch.linalg.norm(ref - torch.as_tensor(out, device=ref.device).double()))
    return 0.0 if den == 0.0 and num == 0.0 else num / den


def _sizes_seeds(ms, ns, ks, seeds, dist, what):
    if isinstance(dist, tuple):
        raise ValueError(f"{what} takes urand or exprand distributions")
    for m in ms:
        for n in ns:
            for k in ks:
                for seed in seeds:
                    yield m, n, k, seed


def ablate_delta(ms, ns, ks, dist, seeds, block_k: int = 0) -> list[str]:
    """cmd_ablate_delta (cli.py:196-214) on the tensor core."""
    import torch

    from .schemes import delta_term_ablation

    lines = ["m,n,k,seed,residual_3term,residual_4term,max_ulp_diff"]
    for m, n, k, seed in _sizes_seeds(ms, ns, ks, seeds, dist, "ablate-delta"):
        a, b = input_pair(dist, m, n, k, seed)
        ref = torch.from_numpy(a).cuda().double() @ torch.from_numpy(b).cuda().double()
        run3, run4, max_ulp = delta_term_ablation(a, b, cfg=_cfg(block_k))
        lines.append(f"{m},{n},{k},{seed},{_fmt64(_residual(ref, run3.output))},"
                     f"{_fmt64(_residual(ref, run4.output))},{_fmt64(max_ulp)}")
    return lines


def rounding_ablation(ms, ns, ks, dist, seeds, block_k: int = 0) -> list[str]:
    """Hardware analogue of cmd_rounding_ablation (cli.py:173-193): the in-unit
    four-term scheme with the tensor core's own terminal rounding against
    corrected3 (main-term accumulation moved out of the unit, RN adds) and
    cuBLAS SGEMM."""
    import torch

    from .schemes import gemm

    cfg = _cfg(block_k)
    prev_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    lines = ["m,n,k,seed,residual_inunit_hw,residual_corrected3,residual_fp32"]
    try:
        for m, n, k, seed in _sizes_seeds(ms, ns, ks, seeds, dist, "rounding-ablation"):
            a, b = input_pair(dist, m, n, k, seed)
            A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
            ref = A.double() @ B.double()
            r4 = _residual(ref, gemm(A, B, "corrected4_rz", cfg).output)
            r3 = _residual(ref, gemm(A, B, "corrected3_halfhalf", cfg).output)
            r32 = _residual(ref, A @ B)
            lines.append(f"{m},{n},{k},{seed},{_fmt64(r4)},{_fmt64(r3)},{_fmt64(r32)}")
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev_tf32
    return lines


def _dyadic_decimal(fr) -> str:
    """cli.py:42-51: exact decimal of a rational with a power-of-two denominator."""
    num, den = fr.numerator, fr.denominator
    k = den.bit_length() - 1
    if den != 1 << k:
        raise ValueError(f"denominator {den} is not a power of two")
    if k == 0:
        return str(num)
    digits = str(num * 5 ** k).rjust(k + 1, "0")
    return digits[:-k] + "." + digits[-k:]


def split_stats(rounding: str) -> list[str]:
    """cmd_split_stats (cli.py:109-117), the enumeration on the GPU."""
    from .analysis import exhaustive_length_distribution

    if rounding.lower() not in ("rn", "rna", "rz"):
        raise ValueError(f"unknown rounding mode: {rounding!r}")
    dist = exhaustive_length_distribution(rounding.lower())
    lines = ["length,prob_num,prob_den"]
    for length in sorted(dist.probabilities):
        p = dist.probabilities[length]
        lines.append(f"{length},{p.numerator},{p.denominator}")
    lines.append(f"expectation,{_dyadic_decimal(dist.expectation)}")
    return lines


def underflow(e_min: int, e_max: int) -> list[str]:
    """cmd_underflow (cli.py:120-132) with the empirical columns computed
    exhaustively on the GPU (all 2^23 mantissas per exponent) instead of by
    Monte Carlo sampling."""
    from .analysis import exhaustive_underflow, gradual_underflow_probability, underflow_probability

    if e_min > e_max:
        raise ValueError("--e-min must not exceed --e-max")
    lines = ["e_v,p_u_theory,p_ugu_theory,p_u_emp,p_ugu_emp,samples"]
    for e_v in range(e_min, e_max + 1):
        r_u, r_ugu = exhaustive_underflow(e_v)
        lines.append(f"{e_v},{_dyadic_decimal(underflow_probability(e_v))},"
                     f"{_dyadic_decimal(gradual_underflow_probability(e_v))},"
                     f"{_fmt64(float(r_u))},{_fmt64(float(r_ugu))},{1 << 23}")
    return lines


def _add_size_flags(p, default_k: str) -> None:
    p.add_argument("--m", default="16")
    p.add_argument("--n", default="16")
    p.add_argument("--k", default=default_k)
    p.add_argument("--seeds", default="0,1,2,3,4,5,6,7")
    p.add_argument("--block-k", type=int, default=0,
                   help="main-term drain interval, MmaConfig.block_k (0 = the kernel's default)")


def _build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="tcec-accuracy",
                                     description="GPU error-corrected GEMM accuracy (CSV).")
    parser.add_argument("--out", default=None, help="output path (default: stdout)")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("gemm-accuracy", help="relative residuals per scheme")
    _add_size_flags(p, "256,1024,4096")
    p.add_argument("--scheme", default="corrected3_halfhalf,cublas_sgemm")
    p.add_argument("--dist", default="urand:-1,1", help="urand:lo,hi | exprand:a,b | type:1..4")
    p = sub.add_parser("rounding-ablation", help="in-unit (hardware rounding) vs corrected3 vs SGEMM")
    _add_size_flags(p, "16,256,1024,4096")
    p.add_argument("--dist", default="urand:-1,1")
    p = sub.add_parser("ablate-delta", help="three-term vs four-term correction")
    _add_size_flags(p, "16,1024")
    p.add_argument("--dist", default="urand:-1,1")
    p = sub.add_parser("split-stats", help="exact kept-mantissa-length distribution (GPU enumeration)")
    p.add_argument("--rounding", default="rn", help="rn, rna, or rz")
    p = sub.add_parser("underflow", help="residual underflow probabilities (theory + GPU enumeration)")
    p.add_argument("--e-min", type=int, default=-30)
    p.add_argument("--e-max", type=int, default=14)
    return parser


def main(argv: list[str] | None = None) -> int:
    """cli.py:268-281: CSV to stdout or --out; ValueError -> 'error: ...', exit 1."""
    args = _build_parser().parse_args(argv)
    try:
        if args.command == "split-stats":
            lines = split_stats(args.rounding)
        elif args.command == "underflow":
            lines = underflow(args.e_min, args.e_max)
        else:
            sizes = (_parse_int_list(args.m), _parse_int_list(args.n), _parse_int_list(args.k))
        if args.command in ("split-stats", "underflow"):
            pass
        elif args.command == "gemm-accuracy":
            lines = gemm_accuracy(*sizes, [s.strip() for s in args.scheme.split(",") if s.strip()],
                                  parse_dist(args.dist), _parse_int_list(args.seeds), args.block_k)
        elif args.command == "ablate-delta":
            lines = ablate_delta(*sizes, parse_dist(args.dist), _parse_int_list(args.seeds),
                                 args.block_k)
        else:
            lines = rounding_ablation(*sizes, parse_dist(args.dist), _parse_int_list(args.seeds),
                                      args.block_k)
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    text = "\n".join(lines) + "\n"
    if args.out:
        Path(args.out).write_text(text, encoding="utf-8", newline="\n")
    else:
        sys.stdout.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
