"""CPU restatement of the smoothing / pyramid stages (paper_2408_06506_b200/
smoothing.py) -- TEST INFRASTRUCTURE ONLY.  These stages have no reference
counterpart (parity unpinned against gelsim); the restatement is checked
against scipy.ndimage.correlate1d(mode='nearest') by tests/test_pyramid.py.
"""
from __future__ import annotations

import numpy as np


def separable_filter(img, taps, step=1):
    """sum_ij w_i w_j img[clamp(s*y+i-R), clamp(s*x+j-R)], float64."""
    img = np.asarray(img, dtype=np.float64)
    taps = np.asarray(taps, dtype=np.float64)
    R = (len(taps) - 1) // 2
    H, W = img.shape[-2:]
    ys = np.arange(0, H, step)
    xs = np.arange(0, W, step)
    tmp = np.zeros(img.shape[:-1] + (len(xs),))
    for j, w in enumerate(taps):
        tmp += w * img[..., np.clip(xs + j - R, 0, W - 1)]
    out = np.zeros(img.shape[:-2] + (len(ys), len(xs)))
    for i, w in enumerate(taps):
        out += w * tmp[..., np.clip(ys + i - R, 0, H - 1), :]
    return out
