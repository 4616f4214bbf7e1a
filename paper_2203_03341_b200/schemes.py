"""The drop-in GEMM entry point: gemm(a, b, scheme, cfg) -> GemmRun.

Mirrors the reference's schemes.py (GemmKind :52-59, GemmScheme :62-84,
factories :87-123, SCHEMES_BY_NAME :126-137, RunFlags / GemmRun :140-153,
default_config :156-160, gemm :317-373) for the path this package accelerates:
the three-term corrected scheme (`corrected3`) with the scaled FP16 split
(FP16-TCEC) or the TF32 split (TF32-TCEC).  The compute runs in the sm_100a
kernel behind include/tcec.h; there is no CPU fallback.  The reference's
in-unit comparators (tc_plain, markidis4, corrected4) run on the tensor core
too (resolve_schedule); its CPU baselines (fp64_ref, fp32_simt,
fp32_lsbtrunc) raise NotImplementedError.

Error behaviour follows the reference: ValueError for non-2-D inputs,
mismatched inner dimensions, non-finite inputs and non-FP32 values
(schemes.py:163-171, :327-330); numerical anomalies only set RunFlags
(schemes.py:237-241, :369-371).
"""

from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .formats import FP16, TF32, FloatFormat, RoundingMode
from .splitting import (SplitScheme, markidis_halfhalf, native_split_args, scaled_halfhalf,
                        tf32tf32)


class GemmKind(enum.Enum):
    FP64_REF = "fp64_ref"
    FP32_SIMT = "fp32_simt"
    FP32_LSBTRUNC = "fp32_lsbtrunc"
    TC_PLAIN = "tc_plain"
    MARKIDIS4 = "markidis4"
    CORRECTED4 = "corrected4"
    CORRECTED3 = "corrected3"


@dataclass(frozen=True)
class GemmScheme:
    kind: GemmKind
    split: SplitScheme | None = None
    terminal: RoundingMode | None = None
    conv_format: FloatFormat | None = None

    @property
    def label(self) -> str:
        for name, scheme in SCHEMES_BY_NAME.items():
            if scheme == self:
                return name
        return self.kind.value

    @property
    def input_format(self) -> FloatFormat | None:
        if self.conv_format is not None:
            return self.conv_format
        if self.split is not None:
            return self.split.low_format
        return None


def fp64_ref() -> GemmScheme:
    return GemmScheme(GemmKind.FP64_REF)


def fp32_simt() -> GemmScheme:
    return GemmScheme(GemmKind.FP32_SIMT)


def fp32_lsbtrunc() -> GemmScheme:
    return GemmScheme(GemmKind.FP32_LSBTRUNC)


def tc_plain(fmt: FloatFormat = FP16) -> GemmScheme:
    return GemmScheme(GemmKind.TC_PLAIN, conv_format=fmt)


def markidis4(fmt: FloatFormat = FP16) -> GemmScheme:
    split = markidis_halfhalf() if fmt == FP16 else tf32tf32()
    return GemmScheme(GemmKind.MARKIDIS4, split=split)


def corrected4(terminal: RoundingMode, split: SplitScheme | None = None) -> GemmScheme:
    if split is None:
        split = markidis_halfhalf()
    if split.scale_log2 != 0:
        raise ValueError("corrected4 requires an unscaled split scheme")
    return GemmScheme(GemmKind.CORRECTED4, split=split, terminal=terminal)


def corrected3(split: SplitScheme | None = None) -> GemmScheme:
    if split is None:
        split = scaled_halfhalf()
    return GemmScheme(GemmKind.CORRECTED3, split=split)


SCHEMES_BY_NAME: dict[str, GemmScheme] = {
    "fp64_ref": fp64_ref(),
    "fp32_simt": fp32_simt(),
    "fp32_lsbtrunc": fp32_lsbtrunc(),
    "tc_plain_fp16": tc_plain(FP16),
    "tc_plain_tf32": tc_plain(TF32),
    "markidis4": markidis4(FP16),
    "corrected4_rn": corrected4(RoundingMode.RN),
    "corrected4_rz": corrected4(RoundingMode.RZ),
    "corrected3_halfhalf": corrected3(scaled_halfhalf()),
    "corrected3_tf32": corrected3(tf32tf32()),
}


@dataclass(frozen=True)
class RunFlags:
    saw_overflow: bool = False
    saw_out_of_range: bool = False


@dataclass(frozen=True)
class GemmRun:
    m: int
    n: int
    k: int
    scheme: object
    output: object
    flags: RunFlags


@dataclass(frozen=True)
class MmaConfig:
    """mma.py:26-45.  On the GPU, block_k is the drain interval of the main-term
    partial (schemes.py:300-304): any multiple of the MMA k-step (16 FP16, 8
    TF32).  The accumulator inside one MMA is the tensor core's own, so
    acc_significand_bits must keep the reference's default (25)."""

    input_format: FloatFormat = FP16
    acc_significand_bits: int = 25
    step_rounding: RoundingMode = RoundingMode.RZ
    terminal_rounding: RoundingMode = RoundingMode.RZ
    block_k: int = 16

    def __post_init__(self) -> None:
        if self.block_k < 1:
            raise ValueError("block_k must be >= 1")
        if not 1 <= self.acc_significand_bits <= 53:
            raise ValueError("acc_significand_bits must be in [1, 53]")
        if self.step_rounding is not RoundingMode.RZ:
            raise ValueError("the emulated unit truncates between steps (RZ only)")


def default_config(scheme, block_k: int = 16, acc_bits: int = 25) -> MmaConfig:
    fmt = getattr(scheme, "input_format", None) or FP16
    return MmaConfig(input_format=fmt, acc_significand_bits=acc_bits, block_k=block_k)


STAGE_K = {N.TCEC_FP16: 64, N.TCEC_TF32: 32}
# Default drain interval of the main-term partial when no MmaConfig is given:
# measured on B200 to be both faster and more accurate against FP64 than the
# reference's per-block drain.
DEFAULT_DRAIN_K = {N.TCEC_FP16: 128, N.TCEC_TF32: 64}

MMA_K = {N.TCEC_FP16: 16, N.TCEC_TF32: 8}


def drain_k_for(variant: int, cfg: MmaConfig | None, sched: int = 0) -> int:
    """Drain interval the kernel uses (tcec_opts.drain_k).  cfg=None: the tuned
    default (128 FP16 / 64 TF32; 16 for corrected4_rn, the reference's block).
    An explicit MmaConfig: its block_k, the reference's drain schedule
    (schemes.py:300-304, mma.py:34), which must be a whole number of MMA
    k-steps (16 FP16, 8 TF32)."""
    if cfg is None:
        return 16 if sched == SCHED_INUNIT4_RN else DEFAULT_DRAIN_K[variant]
    if getattr(cfg, "acc_significand_bits", 25) != 25:
        raise NotImplementedError(
            "the tensor core's accumulator is fixed; acc_significand_bits applies to the "
            "reference's emulator only")
    block_k = int(cfg.block_k)
    if block_k % MMA_K[variant]:
        raise NotImplementedError(
            f"block_k={block_k} is not a multiple of the tensor core's k-step ({MMA_K[variant]})")
    return block_k


# Product schedules of the kernel (include/tcec.h TCEC_SCHEME_*).
SCHED_CORRECTED3, SCHED_CORRECTED3_DD, SCHED_TC_PLAIN, SCHED_INUNIT4 = 0, 1, 2, 3
SCHED_INUNIT4_RN = 4


def resolve_scheme(scheme) -> tuple[int, int, int]:
    """(variant, rounding code, scale_log2) for a corrected3 scheme (the
    accelerated path).  Accepts a registry name, this package's GemmScheme, or
    the reference's GemmScheme (duck-typed on .kind.value and .split)."""
    variant, rounding, scale, sched = resolve_schedule(scheme)
    if sched != SCHED_CORRECTED3:
        raise NotImplementedError(f"{getattr(scheme, 'label', scheme)!r} is not a corrected3 scheme")
    return variant, rounding, scale


def resolve_schedule(scheme) -> tuple[int, int, int, int]:
    """(variant, rounding code, scale_log2, product schedule) of any scheme the
    tensor core can run: corrected3 (the accelerated path) and the reference's
    in-unit comparators tc_plain (schemes.py:343-351), markidis4 / corrected4
    with the RZ terminal (schemes.py:352-364, the hardware accumulator's own
    rounding) and corrected4 with the RN terminal (each product's block drained
    and added RN on the CUDA cores, SCHED_INUNIT4_RN).  fp64_ref / fp32_simt / fp32_lsbtrunc are the
    reference's CPU baselines and are not run here."""
    if isinstance(scheme, str):
        if scheme not in SCHEMES_BY_NAME:
            raise ValueError(f"unknown scheme name: {scheme!r}")
        scheme = SCHEMES_BY_NAME[scheme]
    kind = getattr(getattr(scheme, "kind", None), "value", None)
    if kind == GemmKind.CORRECTED3.value:
        return (*native_split_args(scheme.split), SCHED_CORRECTED3)
    if kind == GemmKind.TC_PLAIN.value:
        f = getattr(scheme, "conv_format", None)
        fmt = (getattr(f, "exp_bits", None), getattr(f, "man_bits", None))
        if fmt == (5, 10):  # FP16, converted RN (schemes.py:346)
            return N.TCEC_FP16, N.ROUND_RN, 0, SCHED_TC_PLAIN
        if fmt == (8, 10):  # TF32, converted RNA
            return N.TCEC_TF32, N.ROUND_RNA, 0, SCHED_TC_PLAIN
        raise NotImplementedError(f"tc_plain in {f!r} has no tensor-core kind here")
    if kind in (GemmKind.MARKIDIS4.value, GemmKind.CORRECTED4.value):
        term = getattr(getattr(scheme, "terminal", None), "value", "rz")
        if kind == GemmKind.CORRECTED4.value and term not in ("rz", "rn"):
            raise NotImplementedError(f"corrected4 with terminal {term!r} has no tensor-core form")
        variant, rounding, scale = native_split_args(scheme.split)
        if scale != 0:
            raise ValueError("in-unit four-term schemes require an unscaled split")
        rn = kind == GemmKind.CORRECTED4.value and term == "rn"
        return variant, rounding, 0, SCHED_INUNIT4_RN if rn else SCHED_INUNIT4
    raise NotImplementedError(
        f"scheme kind {kind!r} is a CPU baseline of the reference; the sm_100a path runs "
        "corrected3 (FP16-TCEC / TF32-TCEC) and the in-unit tensor-core comparators")


def _is_torch(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _as_fp32_host(a) -> np.ndarray:
    """schemes.py:163-171 for host inputs.  Finiteness is checked by the kernel
    (its split warps raise TCEC_FLAG_NONFINITE_INPUT) so the host does not make
    an extra pass over float32 data."""
    x = np.asarray(a)
    if x.ndim != 2:
        raise ValueError("gemm expects 2-D matrices")
    if x.dtype == np.float32:
        return x
    x64 = x.astype(np.float64)
    if not np.all(np.isfinite(x64)):
        raise ValueError("gemm requires finite inputs")
    x32 = x64.astype(np.float32)
    if not np.array_equal(x32.astype(np.float64), x64):
        raise ValueError("inputs must hold FP32 values")
    return x32


def _as_fp32_device(t):
    """schemes.py:163-171 for CUDA tensors of another dtype: the values must be
    finite and exactly representable in FP32 (checked on the device, one
    synchronisation); float32 tensors pass through (the kernel flags
    non-finite inputs)."""
    import torch

    if t.dtype == torch.float32:
        return t
    x64 = t.to(torch.float64)
    if not bool(torch.isfinite(x64).all()):
        raise ValueError("gemm requires finite inputs")
    x32 = x64.to(torch.float32)
    if not torch.equal(x32.to(torch.float64), x64):
        raise ValueError("inputs must hold FP32 values")
    return x32


def _flags_to_run(fl: int) -> RunFlags:
    if fl & N.FLAG_NONFINITE_INPUT:
        raise ValueError("gemm requires finite inputs")
    return RunFlags(saw_overflow=bool(fl & N.FLAG_OVERFLOW),
                    saw_out_of_range=bool(fl & N.FLAG_OUT_OF_RANGE))


def _tma_ready(t):
    """A CUDA fp32 tensor view with unit inner stride, a 16-byte aligned base and a
    leading dimension that is a multiple of 4 floats (TMA); copies when needed."""
    import torch

    if t.stride(1) == 1 and t.stride(0) % 4 == 0 and t.stride(0) >= t.shape[1] \
            and t.data_ptr() % 16 == 0:
        return t, t.stride(0)
    rows, cols = t.shape
    ld = max(4, (cols + 3) // 4 * 4)
    buf = torch.empty((rows, ld), dtype=torch.float32, device=t.device)
    buf[:, :cols].copy_(t)
    return buf[:, :cols], ld


def _check_out(out, m: int, n: int, device) -> None:
    import torch

    if not (_is_torch(out) and out.is_cuda and out.device == device):
        raise ValueError("out must be a CUDA tensor on the operands' device")
    if out.dtype != torch.float32 or out.dim() != 2 or tuple(out.shape) != (m, n):
        raise ValueError(f"out must be a float32 tensor of shape ({m}, {n})")
    if not (out.stride(1) == 1 and out.stride(0) % 4 == 0 and out.stride(0) >= max(n, 1)
            and out.data_ptr() % 16 == 0):
        raise ValueError("out must have unit inner stride and a 16-byte aligned leading dimension")


def gemm_device(a, b, scheme="corrected3_halfhalf", cfg: MmaConfig | None = None, out=None,
                flags=None, block_n: int = 0, group_m: int = 0, kernel_variant: int = 0,
                drain_k: int | None = None, split_mode: int = 0, split_k: int = 0):
    """C = A @ B on CUDA float32 tensors, stream-ordered on torch's current stream.

    No host synchronisation: `flags` (int32 CUDA tensor, one element, caller
    zeroed) receives the TCEC_FLAG_* bits.  Returns the output tensor.
    """
    import torch

    variant, rounding, scale, sched = resolve_schedule(scheme)
    if a.dim() != 2 or b.dim() != 2:
        raise ValueError("gemm expects 2-D matrices")
    m, k = a.shape
    kb, n = b.shape
    if kb != k:
        raise ValueError(f"inner dimensions differ: {k} vs {kb}")
    if a.dtype != torch.float32 or b.dtype != torch.float32:
        raise ValueError("inputs must hold FP32 values")
    if not (a.is_cuda and b.is_cuda) or a.device != b.device:
        raise ValueError("gemm_device expects CUDA tensors on one device")
    if flags is not None and not (_is_torch(flags) and flags.is_cuda and flags.device == a.device
                                  and flags.dtype == torch.int32 and flags.numel() >= 1):
        raise ValueError("flags must be an int32 CUDA tensor on the operands' device")
    if out is None:
        ldc = max(4, (n + 3) // 4 * 4)
        out = torch.empty((m, ldc), dtype=torch.float32, device=a.device)[:, :n]
    else:
        _check_out(out, m, n, a.device)
    if m == 0 or n == 0:
        return out
    if k == 0:  # zero blocks: C = 0 exactly (schemes.py:300-307)
        return out.zero_()
    dk = drain_k if drain_k is not None else drain_k_for(variant, cfg, sched)
    opts = N.make_opts(split_rounding=rounding, scale_log2=scale,
                       drain_k=dk, block_n=block_n, group_m=group_m,
                       kernel_variant=kernel_variant, split_mode=split_mode, scheme=sched,
                       split_k=split_k)
    A, lda = _tma_ready(a)
    B, ldb = _tma_ready(b)
    C, ldc = out, out.stride(0)
    stream = torch.cuda.current_stream(a.device).cuda_stream
    N.check(N.lib().tcec_sgemm(variant, m, n, k, A.data_ptr(), lda, B.data_ptr(), ldb,
                               C.data_ptr(), ldc, ctypes.byref(opts),
                               flags.data_ptr() if flags is not None else None, stream),
            "tcec_sgemm")
    return out


def gemm_device_multi(a, b, outs, scheme="corrected3_halfhalf", cfg: MmaConfig | None = None,
                      flags=None):
    """C = A @ B stored into every tensor of `outs` (same shape and leading
    dimension; CUDA memory this GPU can address, e.g. peer buffers of a
    symmetric-memory all-gather) by one kernel: the fused all-gather path
    (tcec_sgemm_multi).  Stream-ordered on torch's current stream."""
    import torch

    variant, rounding, scale = resolve_scheme(scheme)
    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[0]:
        raise ValueError("gemm expects 2-D matrices with matching inner dimensions")
    if a.dtype != torch.float32 or b.dtype != torch.float32:
        raise ValueError("inputs must hold FP32 values")
    if not (a.is_cuda and b.is_cuda) or a.device != b.device:
        raise ValueError("gemm_device_multi expects CUDA tensors on one device")
    outs = list(outs)
    if not 1 <= len(outs) <= 8:
        raise ValueError("1..8 destinations")
    m, k = a.shape
    n = b.shape[1]
    ldc = outs[0].stride(0)
    for o in outs:
        if not _is_torch(o) or not o.is_cuda or tuple(o.shape) != (m, n) or o.stride(0) != ldc \
                or o.stride(1) != 1 or o.dtype != torch.float32 or o.data_ptr() % 16:
            raise ValueError("destinations must be float32 CUDA (m, n) views with one "
                             "16-byte aligned leading dimension")
    if ldc % 4:
        raise ValueError("destination leading dimension must be a multiple of 4")
    opts = N.make_opts(split_rounding=rounding, scale_log2=scale,
                       drain_k=drain_k_for(variant, cfg), kernel_variant=4)
    A, lda = _tma_ready(a)
    B, ldb = _tma_ready(b)
    ptrs = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
    stream = torch.cuda.current_stream(a.device).cuda_stream
    N.check(N.lib().tcec_sgemm_multi(variant, m, n, k, A.data_ptr(), lda, B.data_ptr(), ldb,
                                      ptrs, len(outs), ldc, ctypes.byref(opts),
                                      flags.data_ptr() if flags is not None else None, stream),
            "tcec_sgemm_multi")
    return outs[0]


def gemm(a, b, scheme, cfg: MmaConfig | None = None, out=None) -> GemmRun:
    """schemes.py:317-373 for the corrected3 schemes, on the GPU.

    numpy / array-like inputs: host buffers in, numpy float32 output (copies
    through the C ABI's host entry, tcec_sgemm_host, which pipelines row chunks
    of A and C against the kernel).  CUDA tensors: device buffers, CUDA tensor
    output.  Either way the call synchronises once to read the RunFlags, as the
    reference's GemmRun carries them.  `out` (optional) receives C: a C-contiguous
    float32 ndarray (e.g. in pinned memory) for host inputs, a CUDA tensor for
    device inputs.
    """
    variant, rounding, scale, sched = resolve_schedule(scheme)
    if _is_torch(a) and a.is_cuda:
        import torch

        if not (_is_torch(b) and b.is_cuda):
            raise ValueError("both operands must live on the same kind of memory")
        if a.dim() != 2 or b.dim() != 2:
            raise ValueError("gemm expects 2-D matrices")
        a32 = _as_fp32_device(a)
        b32 = _as_fp32_device(b)
        fl = torch.zeros(1, dtype=torch.int32, device=a.device)
        out = gemm_device(a32, b32, scheme, cfg, out=out, flags=fl)
        m, k = a.shape
        n = b.shape[1]
        return GemmRun(m=m, n=n, k=k, scheme=scheme, output=out,
                       flags=_flags_to_run(int(fl.item())))
    A = _as_fp32_host(a.cpu().numpy() if _is_torch(a) else a)
    B = _as_fp32_host(b.cpu().numpy() if _is_torch(b) else b)
    m, k = A.shape
    kb, n = B.shape
    if kb != k:
        raise ValueError(f"inner dimensions differ: {k} vs {kb}")
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B)
    if out is not None:
        if not (isinstance(out, np.ndarray) and out.dtype == np.float32 and out.shape == (m, n)
                and out.flags["C_CONTIGUOUS"]):
            raise ValueError("out must be a C-contiguous float32 array of shape (m, n)")
        C = out
    else:
        C = np.empty((m, n), dtype=np.float32)
    fl = ctypes.c_uint32(0)
    opts = N.make_opts(split_rounding=rounding, scale_log2=scale,
                       drain_k=drain_k_for(variant, cfg, sched), scheme=sched)
    N.check(N.lib().tcec_sgemm_host(variant, m, n, k, A.ctypes.data, max(k, 1), B.ctypes.data,
                                    max(n, 1), C.ctypes.data, max(n, 1), ctypes.byref(opts),
                                    ctypes.byref(fl), None), "tcec_sgemm_host")
    return GemmRun(m=m, n=n, k=k, scheme=scheme, output=C, flags=_flags_to_run(int(fl.value)))


def _ulp_fp32(x: np.ndarray) -> np.ndarray:
    """schemes.py:412-415."""
    _, e2 = np.frexp(np.abs(x))
    e = np.clip(e2 - 1, -126, 127)
    return np.ldexp(1.0, e - 23)


def delta_term_ablation(a, b, split: SplitScheme | None = None, cfg: MmaConfig | None = None,
                        ) -> tuple[GemmRun, GemmRun, float]:
    """schemes.py:418-451 on the tensor core: the three-term scheme and its
    four-term sibling (the dA*dB chain in a separate accumulator, added last
    with scale 2^-2s) on the same splits.  Returns both runs and the largest
    elementwise difference in FP32 ulps of the four-term output."""
    if split is None:
        split = scaled_halfhalf()
    scheme3 = corrected3(split)
    variant, rounding, scale = native_split_args(split)
    A = _as_fp32_host(a.cpu().numpy() if _is_torch(a) else a)
    B = _as_fp32_host(b.cpu().numpy() if _is_torch(b) else b)
    m, k = A.shape
    kb, n = B.shape
    if kb != k:
        raise ValueError(f"inner dimensions differ: {k} vs {kb}")
    outs = []
    for sched in (SCHED_CORRECTED3, SCHED_CORRECTED3_DD):
        C = np.empty((m, n), dtype=np.float32)
        fl = ctypes.c_uint32(0)
        opts = N.make_opts(split_rounding=rounding, scale_log2=scale,
                           drain_k=drain_k_for(variant, cfg), scheme=sched)
        N.check(N.lib().tcec_sgemm_host(variant, m, n, k, np.ascontiguousarray(A).ctypes.data,
                                        max(k, 1), np.ascontiguousarray(B).ctypes.data, max(n, 1),
                                        C.ctypes.data, max(n, 1), ctypes.byref(opts),
                                        ctypes.byref(fl), None), "tcec_sgemm_host")
        outs.append((C, _flags_to_run(int(fl.value))))
    (c3, f3), (c4, _) = outs
    run3 = GemmRun(m, n, k, scheme3, c3, f3)
    run4 = GemmRun(m, n, k, GemmScheme(GemmKind.CORRECTED4, split=split, terminal=RoundingMode.RZ),
                   c4, f3)
    diff = np.abs(c3.astype(np.float64) - c4.astype(np.float64))
    max_ulp = float(np.max(diff / _ulp_fp32(c4.astype(np.float64)))) if diff.size else 0.0
    return run3, run4, max_ulp
