"""Floating-point format and rounding-mode descriptors (reference formats.py:43-111).

Only the descriptors travel to the GPU path: they select the split recipe of
the kernel.  The arithmetic itself is done by the hardware (cvt / integer
rounding in the split warps, tcgen05 in the MMA stage, FP32 RN adds in the
drain warps); there is no software rounding kit here.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass


class RoundingMode(enum.Enum):
    """formats.py:43-55: nearest ties-to-even, nearest ties-away, toward zero."""

    RN = "rn"
    RNA = "rna"
    RZ = "rz"

    @classmethod
    def parse(cls, name: str) -> "RoundingMode":
        try:
            return cls(name.strip().lower())
        except ValueError:
            raise ValueError(f"unknown rounding mode: {name!r}") from None


@dataclass(frozen=True)
class FloatFormat:
    """formats.py:58-104 (sign, exponent field, stored fraction bits)."""

    exp_bits: int
    man_bits: int
    bias: int
    subnormals_enabled: bool = True

    @property
    def min_normal_exp(self) -> int:
        return 1 - self.bias

    @property
    def max_normal_exp(self) -> int:
        return (1 << self.exp_bits) - 2 - self.bias

    @property
    def max_finite(self) -> float:
        return math.ldexp(2.0 - math.ldexp(1.0, -self.man_bits), self.max_normal_exp)

    @property
    def min_normal(self) -> float:
        return math.ldexp(1.0, self.min_normal_exp)

    @property
    def min_subnormal(self) -> float:
        return math.ldexp(1.0, self.min_normal_exp - self.man_bits)


FP16 = FloatFormat(exp_bits=5, man_bits=10, bias=15)
TF32 = FloatFormat(exp_bits=8, man_bits=10, bias=127)
FP32 = FloatFormat(exp_bits=8, man_bits=23, bias=127)
ACC25 = FloatFormat(exp_bits=8, man_bits=24, bias=127)
