"""CPU restatement of the per-pixel binned polynomial LUT
(paper_2408_06506_b200/binned.py, csrc/binned.cu) -- TEST INFRASTRUCTURE ONLY.

The stage has no counterpart in the reference (gelsim's
PolyLut, render/lut.py:31-59, is one global polynomial), so parity against
the reference is unpinned; what IS pinned: with one bin this function is
gelsim_oracle.depth_to_rgb (the reference restatement), and the tests check
that.  Gradients follow render/lut.py:25-28 via gelsim_oracle.depth_gradients.
"""
from __future__ import annotations

import numpy as np

from oracle.gelsim_oracle import depth_gradients, monomial_exponents


def bin_index(n: int, bins: int) -> np.ndarray:
    """pixel -> bin along one axis: floor(i * bins / n)."""
    return (np.arange(n, dtype=np.int64) * bins) // n


def depth_to_rgb_binned(values, coeffs, degree):
    """(..., H, W) depth, (bins_y, bins_x, 3, T) coefficients -> (..., H, W, 3)
    float64 in [0, 1]."""
    values = np.asarray(values, dtype=np.float64)
    coeffs = np.asarray(coeffs, dtype=np.float64)
    H, W = values.shape[-2:]
    by, bx = coeffs.shape[:2]
    g_x, g_y = depth_gradients(values)
    per_px = coeffs[bin_index(H, by)[:, None], bin_index(W, bx)[None, :]]  # (H, W, 3, T)
    out = np.zeros(values.shape + (3,), dtype=np.float64)
    for k, (i, j) in enumerate(monomial_exponents(degree)):
        term = np.ones_like(g_x) if (i, j) == (0, 0) else (g_x ** i) * (g_y ** j)
        out += per_px[..., k] * term[..., None]
    return np.clip(out, 0.0, 1.0)
