"""Accuracy metric (reference analysis.py:175-192, Eq. 7 of the paper) and the
split statistics of analysis.py:32-172: the closed-form residual-underflow
probabilities (exact dyadic rationals) and their exhaustive GPU counterparts
(every 23-bit mantissa, one thread each, `tcec_split_census`)."""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

import numpy as np

_L_F32, _L_F16, _B_F16 = 23, 10, 15
_MAX_RUN = _L_F32 - _L_F16  # 13
_ENUM = 1 << _L_F32


@dataclass(frozen=True)
class MantissaLengthDistribution:
    """analysis.py:38-50: exact kept-length distribution over all 2^23 mantissas."""

    probabilities: dict

    @property
    def expectation(self) -> Fraction:
        return sum((Fraction(k) * p for k, p in self.probabilities.items()), Fraction(0))


@dataclass(frozen=True)
class UnderflowCurve:
    """analysis.py:53-57: (e_v, p_u, p_u_plus_gu) per unbiased exponent."""

    points: list


def zero_run_probability(n: int) -> Fraction:
    """analysis.py:69-80: geometric zero run below the kept 10 bits, saturating at 13."""
    if n < 0 or n > _MAX_RUN:
        return Fraction(0)
    if n == _MAX_RUN:
        return Fraction(1, 2 ** _MAX_RUN)
    return Fraction(1, 2 ** (n + 1))


def _tail_probability(lower: int) -> Fraction:
    return sum((zero_run_probability(r) for r in range(max(lower, 0), _MAX_RUN + 1)), Fraction(0))


def gradual_underflow_probability(e_v: int) -> Fraction:
    """analysis.py:89-95: residual below the FP16 normal range."""
    return _tail_probability(e_v - _L_F16 + _B_F16 - 2 + 1)


def underflow_probability(e_v: int) -> Fraction:
    """analysis.py:98-100: residual below every FP16 subnormal."""
    return _tail_probability(e_v + _B_F16 - 2 + 1)


def underflow_curve(e_min: int, e_max: int) -> UnderflowCurve:
    """analysis.py:103-113."""
    if e_min > e_max:
        raise ValueError("e_min must not exceed e_max")
    return UnderflowCurve([(e, underflow_probability(e), gradual_underflow_probability(e))
                           for e in range(e_min, e_max + 1)])


def _census(kind: int, rounding: int, e_v: int) -> list:
    import torch

    from . import _native as N

    counts = torch.zeros(24, dtype=torch.int64, device="cuda")
    N.check(N.lib().tcec_split_census(kind, rounding, e_v, counts.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream),
            "tcec_split_census")
    return [int(c) for c in counts.cpu().tolist()]


def exhaustive_length_distribution(split_rounding) -> MantissaLengthDistribution:
    """analysis.py:141-165 on the GPU: every 23-bit mantissa at e_v = 0 through the
    markidis_halfhalf split with `split_rounding` (RoundingMode or 'rn'/'rna'/'rz')."""
    from . import _native as N

    name = getattr(split_rounding, "value", split_rounding)
    code = {"rn": N.ROUND_RN, "rna": N.ROUND_RNA, "rz": N.ROUND_RZ}[str(name).lower()]
    counts = _census(0, code, 0)
    return MantissaLengthDistribution({k: Fraction(c, _ENUM) for k, c in enumerate(counts) if c})


def exhaustive_underflow(e_v: int) -> tuple:
    """Exact residual-underflow rates at exponent e_v over every mantissa (the
    exhaustive form of analysis.py:106-135 empirical_underflow, RZ split):
    (P_u, P_u+gu) as Fractions."""
    from . import _native as N

    counts = _census(1, N.ROUND_RZ, e_v)
    return Fraction(counts[0], _ENUM), Fraction(counts[1], _ENUM)


def relative_residual(c_test, c_ref) -> float:
    """||ref - test||_F / ||ref||_F accumulated in float64; 0/0 reports 0."""
    test = np.asarray(c_test, dtype=np.float64)
    ref = np.asarray(c_ref, dtype=np.float64)
    if test.shape != ref.shape:
        raise ValueError("shapes differ")
    num = float(np.linalg.norm(ref - test))
    den = float(np.linalg.norm(ref))
    if den == 0.0:
        if num == 0.0:
            return 0.0
        raise ValueError("zero reference norm with nonzero residual")
    return num / den
