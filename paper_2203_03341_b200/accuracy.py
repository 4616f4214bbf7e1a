"""GPU accuracy harness: the reference's `gemm-accuracy` experiment on B200.

Mirrors `tcgemm gemm-accuracy` (reference cli.py:135-170, parser :227-265):
same flags, the same CSV ("m,n,k,scheme,seed,residual,flags" plus an `avg`
row per (m, n, k, scheme)), the same inputs (genmat.py generators, restated
bit-exactly in genmat.py here) and the same metric (Eq. 7, analysis.py:175-192).
The hot path runs on the GPU; the FP64 ground truth is cuBLAS DGEMM on the GPU
(the reference's sequential FP64 sum differs from it at the 1e-16 level).

Schemes: corrected3_halfhalf / corrected3_tf32 (this package's kernels) and
`cublas_sgemm` (FP32 SIMT SGEMM, TF32 disabled) as the SGEMM baseline; the
reference's other CPU comparators are out of scope.

    python -m paper_2203_03341_b200.accuracy gemm-accuracy --m 16 --n 16 \
        --k 256,1024,4096 --scheme corrected3_halfhalf,cublas_sgemm --dist urand:-1,1
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

from .genmat import ExpRand, MatrixSpec, Urand, generate, pair_seed, type_pair

GPU_SCHEMES = ("corrected3_halfhalf", "corrected3_tf32", "cublas_sgemm")


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


def gemm_accuracy(ms, ns, ks, schemes, dist, seeds, block_k: int = 16) -> list[str]:
    """cmd_gemm_accuracy (cli.py:135-170) with the GEMMs on the GPU."""
    import torch

    from .schemes import MmaConfig, gemm

    for name in schemes:
        if name not in GPU_SCHEMES:
            raise ValueError(f"unknown scheme {name!r}; known: {', '.join(GPU_SCHEMES)}")
    if not schemes:
        raise ValueError("no schemes requested")
    prev_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    cfg = MmaConfig(block_k=block_k)
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


def _build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="tcec-accuracy",
                                     description="GPU error-corrected GEMM accuracy (CSV).")
    parser.add_argument("--out", default=None, help="output path (default: stdout)")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("gemm-accuracy", help="relative residuals per scheme")
    p.add_argument("--m", default="16")
    p.add_argument("--n", default="16")
    p.add_argument("--k", default="256,1024,4096")
    p.add_argument("--seeds", default="0,1,2,3,4,5,6,7")
    p.add_argument("--block-k", type=int, default=16, help="drain interval request (MmaConfig.block_k)")
    p.add_argument("--scheme", default="corrected3_halfhalf,cublas_sgemm")
    p.add_argument("--dist", default="urand:-1,1", help="urand:lo,hi | exprand:a,b | type:1..4")
    return parser


def main(argv: list[str] | None = None) -> int:
    """cli.py:268-281: CSV to stdout or --out; ValueError -> 'error: ...', exit 1."""
    args = _build_parser().parse_args(argv)
    try:
        lines = gemm_accuracy(_parse_int_list(args.m), _parse_int_list(args.n),
                              _parse_int_list(args.k),
                              [s.strip() for s in args.scheme.split(",") if s.strip()],
                              parse_dist(args.dist), _parse_int_list(args.seeds), args.block_k)
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
