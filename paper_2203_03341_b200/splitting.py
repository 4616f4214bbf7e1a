"""Split recipes and the GPU split (reference splitting.py).

`SplitScheme` / `scaled_halfhalf` / `tf32tf32` / `markidis_halfhalf` mirror
splitting.py:37-79 so that schemes built with either package select the same
kernel.  `split_matrix` runs the sm_100a split kernel (the same device
arithmetic the fused GEMM runs in its split warps) and returns hi / lo as FP32
values, matching splitting.py:139-147 bit for bit.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

from . import _native as N
from .formats import FP16, TF32, FloatFormat, RoundingMode

# splitting.py:34: mantissa length of FP16 plus the implicit bit.
RESIDUAL_SCALE_LOG2 = FP16.man_bits + 1


class SplitKind(enum.Enum):
    MARKIDIS_HALFHALF = "markidis_halfhalf"
    SCALED_HALFHALF = "scaled_halfhalf"
    TF32TF32 = "tf32tf32"


@dataclass(frozen=True)
class SplitScheme:
    """splitting.py:43-67: target format, residual scale, rounding."""

    kind: SplitKind
    rounding: RoundingMode | None = None

    def __post_init__(self) -> None:
        if self.rounding is None:
            default = RoundingMode.RNA if self.kind is SplitKind.TF32TF32 else RoundingMode.RN
            object.__setattr__(self, "rounding", default)

    @property
    def low_format(self) -> FloatFormat:
        return TF32 if self.kind is SplitKind.TF32TF32 else FP16

    @property
    def scale_log2(self) -> int:
        return RESIDUAL_SCALE_LOG2 if self.kind is SplitKind.SCALED_HALFHALF else 0


def markidis_halfhalf(rounding: RoundingMode = RoundingMode.RN) -> SplitScheme:
    return SplitScheme(SplitKind.MARKIDIS_HALFHALF, rounding)


def scaled_halfhalf(rounding: RoundingMode = RoundingMode.RN) -> SplitScheme:
    return SplitScheme(SplitKind.SCALED_HALFHALF, rounding)


def tf32tf32(rounding: RoundingMode = RoundingMode.RNA) -> SplitScheme:
    return SplitScheme(SplitKind.TF32TF32, rounding)


_ROUND_CODE = {"rn": N.ROUND_RN, "rna": N.ROUND_RNA, "rz": N.ROUND_RZ}


def native_split_args(split) -> tuple[int, int, int]:
    """(variant, rounding code, scale_log2) of a split recipe.

    Accepts this package's SplitScheme or the reference's (duck-typed on
    .kind.value / .rounding.value, the reference's enum values).
    """
    kind = getattr(getattr(split, "kind", None), "value", None)
    rnd = getattr(getattr(split, "rounding", None), "value", None)
    if kind == "tf32tf32":
        variant, scale = N.TCEC_TF32, 0
    elif kind == "scaled_halfhalf":
        variant, scale = N.TCEC_FP16, RESIDUAL_SCALE_LOG2
    elif kind == "markidis_halfhalf":
        variant, scale = N.TCEC_FP16, 0
    else:
        raise ValueError(f"not a split scheme: {split!r}")
    if rnd not in _ROUND_CODE:
        raise ValueError(f"unknown split rounding: {rnd!r}")
    code = _ROUND_CODE[rnd]
    if variant == N.TCEC_FP16 and code == N.ROUND_RNA:
        raise NotImplementedError("FP16 split with RNA rounding has no sm_100 conversion; "
                                  "use RN or RZ")
    return variant, code, scale


@dataclass(frozen=True)
class SplitMatrices:
    """splitting.py:90-103: elementwise split; hi and lo hold low-format values."""

    hi: object
    lo: object
    scale_log2: int

    @property
    def rows(self) -> int:
        return self.hi.shape[0]

    @property
    def cols(self) -> int:
        return self.hi.shape[1]


def split_device(x, split, flags=None):
    """Split a CUDA float32 tensor on the GPU; returns (hi, lo) float32 tensors.

    `flags` (optional int32 CUDA tensor of one element) is OR-ed with the
    TCEC_FLAG_* bits.  Stream-ordered on torch's current stream, no sync.
    """
    import torch

    variant, code, scale = native_split_args(split)
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32):
        raise TypeError("split_device expects a CUDA float32 tensor")
    xc = x.contiguous()
    hi = torch.empty_like(xc)
    lo = torch.empty_like(xc)
    stream = torch.cuda.current_stream(xc.device).cuda_stream
    fptr = flags.data_ptr() if flags is not None else None
    N.check(N.lib().tcec_split(variant, code, scale, xc.data_ptr(), xc.numel(), hi.data_ptr(),
                               lo.data_ptr(), fptr, stream), "tcec_split")
    return hi, lo


def split_matrix(m, scheme: SplitScheme) -> SplitMatrices:
    """splitting.py:139-147 on the GPU.  numpy in -> numpy out; tensor in -> tensor out."""
    import numpy as np
    import torch

    if isinstance(m, torch.Tensor):
        if m.dim() != 2:
            raise ValueError("split_matrix expects a 2-D array")
        x = m if m.is_cuda else m.cuda()
        hi, lo = split_device(x.to(torch.float32), scheme)
        _, _, s = native_split_args(scheme)
        return SplitMatrices(hi, lo, s)
    x = np.asarray(m)
    if x.ndim != 2:
        raise ValueError("split_matrix expects a 2-D array")
    x64 = x.astype(np.float64)
    if not np.all(np.isfinite(x64)):
        raise ValueError("split_matrix requires finite values")
    x32 = x64.astype(np.float32)
    if not np.array_equal(x32.astype(np.float64), x64):
        raise ValueError("inputs must hold FP32 values")
    hi, lo = split_device(torch.from_numpy(np.ascontiguousarray(x32)).cuda(), scheme)
    _, _, s = native_split_args(scheme)
    return SplitMatrices(hi.cpu().numpy().astype(np.float64), lo.cpu().numpy().astype(np.float64), s)
