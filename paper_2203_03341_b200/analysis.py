"""Accuracy metric (reference analysis.py:175-192, Eq. 7 of the paper)."""

from __future__ import annotations

import numpy as np


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
