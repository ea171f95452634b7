"""Parity tolerances shared by the GPU tests, smoke() and bench.py.

Holds no neighborhood-attention arithmetic and imports neither the product
nor the oracle: it only states the bounds of DESIGN.md reading R14.

north_star: max-abs <= 1e-4 for fp32 inputs (TF32 off) and <= 1e-2 on
O/dQ/dK/dV for fp16/bf16 with unit-normal inputs, against the EXACT result
(the oracle's fp64 forward / gradient).  Where the output dtype cannot
represent a value to within the bound -- a bf16 value of magnitude >= 2.56
has a half-ulp above 1e-2 -- the bound is that half-ulp, the error of the
correctly rounded result itself: max(tol, half_ulp(|ref|)), never the sum.
LSE (fp32 output): 1e-4 (fp32 inputs) / 2e-3 (16-bit inputs).
"""
from __future__ import annotations

import numpy as np
import torch

TOL = {torch.float32: 1e-4, torch.float16: 1e-2, torch.bfloat16: 1e-2}
LSE_TOL = {torch.float32: 1e-4, torch.float16: 2e-3, torch.bfloat16: 2e-3}
# significand bits (incl. the implicit one) of each output dtype
_BITS = {torch.float32: 24, torch.float16: 11, torch.bfloat16: 8}


def half_ulp(ref: np.ndarray, dt: torch.dtype) -> np.ndarray:
    """Half the spacing of `dt` at |ref| (normal range; fp16 subnormals use
    the smallest normal exponent)."""
    mag = np.maximum(np.abs(np.asarray(ref, np.float64)), 2.0 ** -14)
    return 2.0 ** (np.floor(np.log2(mag)) - _BITS[dt])


def bound(ref, dt: torch.dtype) -> np.ndarray:
    """Per-element bound max(TOL[dt], half_ulp(|ref|))."""
    return np.maximum(TOL[dt], half_ulp(ref, dt))


def excess(got, ref, dt: torch.dtype) -> float:
    """max over elements of |got - ref| - bound; <= 0 passes."""
    g = np.asarray(got, np.float64)
    r = np.asarray(ref, np.float64)
    return float((np.abs(g - r) - bound(r, dt)).max()) if r.size else -1.0


def max_abs(got, ref) -> float:
    g = np.asarray(got, np.float64)
    r = np.asarray(ref, np.float64)
    return float(np.abs(g - r).max()) if r.size else 0.0
